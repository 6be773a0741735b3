summ() { python -c "
import json,sys; d=json.load(open('$1'))
print('$1', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'it', d['iters_per_solve'], 'iter', d['iteration']['us_kernels'], [(k['name'], k['us']) for k in d['iteration']['kernels']])"; }
for v in "" _kd2; do
FDE_LIB=$PWD/paper_1912_13304_b200/libfde${v}.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench$v.json 2> gpurun_out/bench$v.err; summ gpurun_out/bench$v.json
done
FDE_LIB=$PWD/paper_1912_13304_b200/libfde_kd2.so timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q -p no:cacheprovider -k "sine_domain or solver_parity or batch" 2>&1 | tail -2
FDE_LIB=$PWD/paper_1912_13304_b200/libfde_kd2.so timeout 600 python tools/sweep.py --only 1,3,5 > gpurun_out/sweep_kd2.jsonl 2>&1
