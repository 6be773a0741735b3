mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests.log | grep -E "passed|failed|Error|assert"
summ() { python -c "
import json,sys; d=json.load(open('$1'))
print('$1', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'it', d['iters_per_solve'], 'iter', d['iteration']['us_kernels'], [(k['name'], k['us']) for k in d['iteration']['kernels']])"; }
for v in ""; do
FDE_LIB=$PWD/paper_1912_13304_b200/libfde${v}.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench${v}.json 2> gpurun_out/bench${v}.err; summ gpurun_out/bench${v}.json
done
FDE_GRAPH=0 python tools/unit_run.py --reps 1 --pcg > gpurun_out/plain2.log 2>&1 && \
FDE_GRAPH=0 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k_sineop_lines|k_sine_xr" -s 6 -c 3 \
    -o gpurun_out/prof_iter python tools/unit_run.py --reps 1 --pcg > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
