#!/bin/bash
mkdir -p gpurun_out
FDE_GRAPH=0 timeout 300 python tools/unit_run.py --n 4095 --reps 1 --pcg > gpurun_out/plain_4095.log 2>&1 && \
FDE_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sop|k_sine_xr5" -s 4 -c 2 \
    -o gpurun_out/prof_sop4095 python tools/unit_run.py --n 4095 --reps 1 --pcg > gpurun_out/ncu_4095.log 2>&1; echo "ncu rc=$?"
