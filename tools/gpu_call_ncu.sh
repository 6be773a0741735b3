#!/bin/bash
# ncu --set full (warm cache: --cache-control none) of the unit kernels of one config.
# usage: tools/gpu_call_ncu.sh <tag> [unit_run args...]
tag=$1; shift
mkdir -p gpurun_out
python tools/unit_run.py "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k_(tau|toeplitz|dst)" -s 5 -c 5 \
    -o gpurun_out/prof_$tag python tools/unit_run.py "$@" > gpurun_out/ncu_$tag.log 2>&1; echo "ncu rc=$?"
