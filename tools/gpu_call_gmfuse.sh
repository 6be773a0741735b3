#!/bin/bash
# GMRES with the fused τ-DST + Toeplitz rows operator: parity tests + cfg 1/2/4 sweep lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or smoke or table" > gpurun_out/pytest_gm.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gm.log
timeout 600 python tools/sweep.py --only 1,2,4 > gpurun_out/sweep_gm.jsonl 2> gpurun_out/sweep_gm.err; echo "sweep rc=$?"
