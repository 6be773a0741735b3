#!/bin/bash
# A/B timing + one ncu --set full capture of the sop kernel at n=1023
mkdir -p gpurun_out
timeout 300 python tools/ab_sop.py > gpurun_out/ab_sop1.jsonl 2>&1; echo "ab1 rc=$?"; cat gpurun_out/ab_sop1.jsonl
FDE_GRAPH=0 timeout 300 python tools/unit_run.py --reps 1 --pcg > gpurun_out/plain_sop.log 2>&1 && \
FDE_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sop|k_sine_xr5" -s 4 -c 2 \
    -o gpurun_out/prof_sop python tools/unit_run.py --reps 1 --pcg > gpurun_out/ncu_sop.log 2>&1; echo "ncu rc=$?"
