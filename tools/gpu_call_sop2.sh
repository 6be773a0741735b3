#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cfg5" > gpurun_out/sop_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/sop_parity.log
timeout 900 python -m pytest tests/test_gpu_solvers.py -x -q -k "sine_domain or batch_rhs or zero_rhs or not_converged or graph_caches" > gpurun_out/sop_solvers.log 2>&1; echo "solvers rc=$?"; tail -3 gpurun_out/sop_solvers.log
timeout 300 python tools/ab_sop.py > gpurun_out/ab_sop1.jsonl 2>&1; echo "ab1 rc=$?"; cat gpurun_out/ab_sop1.jsonl
FDE_GRAPH=0 timeout 300 python tools/unit_run.py --reps 1 --pcg > gpurun_out/plain_sop.log 2>&1 && \
FDE_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sop" -s 2 -c 1 \
    -o gpurun_out/prof_sop4 python tools/unit_run.py --reps 1 --pcg > gpurun_out/ncu_sop.log 2>&1; echo "ncu rc=$?"
