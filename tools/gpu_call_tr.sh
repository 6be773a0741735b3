#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/dbg_batch.py 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cfg5" > gpurun_out/sop_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/sop_parity.log
for tr in 1 0; do FDE_SOP_TR=$tr timeout 600 python tools/sweep.py --only 5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print('TR=$tr', d['n'], d['batch'], d['iters_per_solve'], round(d['us_per_iter'],1), {k:round(v,1) for k,v in d['loop_body_kernels_us'].items()})"; done
