#!/bin/bash
# A/B of library variants (FDE_LIB) on the GMRES configs: cfg 4 and cfg 2 sweep
# lines per variant, the per-step DCGS2 trace, then the gmres parity tests.
# usage: bash tools/gpu_call_gml2.sh "<variant suffixes>" [trace-suffix]
mkdir -p gpurun_out
: > gpurun_out/gml2.txt
for L in $1; do
  [ "$L" = "main" ] && L=""
  for r in 1 2; do
    FDE_LIB=$PWD/paper_1912_13304_b200/libfde$L.so timeout 300 python tools/sweep.py --only 4,2 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('[$L]', d['cfg'], d['n'], round(d['us_per_iter'], 2), d['iters_per_solve'], {k: round(v / 30, 1) for k, v in d['loop_body_kernels_us'].items()})
"
  done
done | tee -a gpurun_out/gml2.txt
if [ -n "$2" ]; then
  FDE_LIB=$PWD/paper_1912_13304_b200/libfde$2.so timeout 200 python tools/gm_trace.py 1023 | awk 'NR%3==1' | tee gpurun_out/gm_trace.txt
fi
[ -n "$3" ] && { timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or matvec or op" > gpurun_out/pytest_gm.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gm.log; }
