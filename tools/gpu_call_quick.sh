#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ab_sop.py 2>&1 | sed "s/^/main /"
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cfg5" > gpurun_out/sop_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/sop_parity.log
