#!/bin/bash
# Round-2 evidence: reference arm, ncu launch list of the bench command
# (FDE_GRAPH=0 so ncu sees the loop-body kernels), one ncu --set full capture
# of the sop operator and the vector step (with source), warm-cache counters.
mkdir -p gpurun_out
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
FDE_GRAPH=0 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
FDE_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
FDE_GRAPH=0 timeout 300 python tools/unit_run.py --reps 1 --pcg > gpurun_out/plain2.log 2>&1 && \
FDE_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sop|k_sine_xr5" -s 4 -c 2 \
    -o gpurun_out/prof_sop_r02 python tools/unit_run.py --reps 1 --pcg > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
bash tools/gpu_call_warmncu.sh
