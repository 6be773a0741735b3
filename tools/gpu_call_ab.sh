#!/bin/bash
# GPU tests, then the unit profile + bench for library variants (FDE_LIB).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for v in "$@"; do
  lib=paper_1912_13304_b200/libfde${v}.so
  FDE_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench${v}.json 2> gpurun_out/bench${v}.err; echo "bench$v rc=$?"
  python -c "
import json,sys; d=json.load(open('gpurun_out/bench${v}.json'))
print('$v', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'unit_us', d['unit_w']['us'], [(k['name'], k['us']) for k in d['unit_w']['kernels']])" 2>&1 | tail -2
done
