#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
FDE_SOP=0 timeout 300 python tools/sweep.py --only 5 > gpurun_out/sweep_sop0.jsonl 2>&1; echo "sweep0 rc=$?"
