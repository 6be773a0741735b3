#!/bin/bash
mkdir -p gpurun_out
python tools/dbg_batch.py > gpurun_out/dbg_batch.log 2>&1; cat gpurun_out/dbg_batch.log
for p in 1 2 3; do FDE_LIB=paper_1912_13304_b200/libfde_probe$p.so timeout 300 python tools/ab_sop.py 2>&1 | grep '"n": 1023, "batch": 1,' | sed "s/^/probe$p /"; done
timeout 300 python tools/ab_sop.py 2>&1 | sed "s/^/main /"
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cfg5" > gpurun_out/sop_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/sop_parity.log
