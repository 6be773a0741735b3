#!/bin/bash
# One gpurun call: bench, launch list, ncu --set full of the unit kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
python tools/unit_run.py --reps 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(tau|toeplitz|dst)" -c 5 \
    -o gpurun_out/prof_unit python tools/unit_run.py --reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
