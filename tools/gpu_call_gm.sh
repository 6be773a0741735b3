#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cfg4" > gpurun_out/gm_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gm_parity.log
timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q -k "gmres or solver_parity or batch_rhs" > gpurun_out/gm_solvers.log 2>&1; echo "solvers rc=$?"; tail -2 gpurun_out/gm_solvers.log
timeout 300 python tools/sweep.py --only 2,4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print(d['cfg'], d['n'], d['iters_per_solve'], round(d['us_per_iter'],1), {k:round(v,1) for k,v in d['loop_body_kernels_us'].items()})"
