mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests.log | grep -E "passed|failed|Error|assert"
summ() { python -c "
import json,sys; d=json.load(open('$1'))
print('$1', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'it', d['iters_per_solve'], 'iter', d['iteration']['us_kernels'], [(k['name'], k['us']) for k in d['iteration']['kernels']])"; }
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; summ gpurun_out/bench.json
FDE_SINE_BODY=3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b3.json 2> gpurun_out/bench_b3.err; summ gpurun_out/bench_b3.json
timeout 600 python tools/sweep.py --quick > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
