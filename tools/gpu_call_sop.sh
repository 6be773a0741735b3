#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cfg5_n1023" > gpurun_out/sop_parity.log 2>&1; echo "parity rc=$?"; tail -5 gpurun_out/sop_parity.log
timeout 900 python -m pytest tests/test_gpu_solvers.py -x -q -k "sine_domain or batch_rhs or zero_rhs or not_converged or graph_caches" > gpurun_out/sop_solvers.log 2>&1; echo "solvers rc=$?"; tail -5 gpurun_out/sop_solvers.log
timeout 300 python tools/ab_sop.py > gpurun_out/ab_sop1.jsonl 2>&1; echo "ab1 rc=$?"
FDE_SOP=0 timeout 300 python tools/ab_sop.py > gpurun_out/ab_sop0.jsonl 2>&1; echo "ab0 rc=$?"
cat gpurun_out/ab_sop1.jsonl gpurun_out/ab_sop0.jsonl
