#!/bin/bash
# A/B of library variants (FDE_LIB) on the PCG configs: cfg 3/5 sweep lines per variant (two runs each)
# usage: bash tools/gpu_call_pcgab.sh "<variant suffixes; main = libfde.so>"
mkdir -p gpurun_out
for L in $1; do
  [ "$L" = "main" ] && L=""
  for r in 1 2; do
    FDE_LIB=$PWD/paper_1912_13304_b200/libfde$L.so timeout 600 python tools/sweep.py --only 5 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('[$L]', d['cfg'], d['n'], d['batch'], round(d['us_per_iter'], 2), d['iters_per_solve'], {k: round(v, 1) for k, v in d['loop_body_kernels_us'].items()})
"
  done
done | tee gpurun_out/pcgab.txt
