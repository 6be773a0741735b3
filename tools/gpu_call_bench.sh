#!/bin/bash
# One gpurun call: smoke, bench (JSON line), reference arm, sweep, ncu launch
# list of the bench command (FDE_GRAPH=0 so ncu sees the loop-body kernels),
# ncu --set full of the kernels of one PCG iteration.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
FDE_GRAPH=0 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
FDE_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
FDE_GRAPH=0 python tools/unit_run.py --reps 1 --pcg > gpurun_out/plain2.log 2>&1 && \
FDE_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:"k_sineop|k_sine_xr" -s 6 -c 4 \
    -o gpurun_out/prof_iter python tools/unit_run.py --reps 1 --pcg > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
