mkdir -p gpurun_out
#timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
summ() { python -c "
import json,sys; d=json.load(open('$1'))
print('$1', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'it', d['iters_per_solve'], 'unit_us', d['unit_w']['us'], [(k['name'], k['us']) for k in d['unit_w']['kernels']], 'cold', d['unit_w']['cold_total_us'])"; }
for v in _m3 _kr3m3 _m2; do
  FDE_LIB=$PWD/paper_1912_13304_b200/libfde${v}.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench${v}.json 2> gpurun_out/bench${v}.err; summ gpurun_out/bench${v}.json
done
FDE_LIB=$PWD/paper_1912_13304_b200/libfde_m2.so timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -2
