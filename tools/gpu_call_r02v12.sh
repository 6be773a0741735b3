#!/bin/bash
# Round-2 evidence: smoke, bench line, reference arm, sweep, ncu launch list of
# the bench command, ncu --set full of one PCG iteration (n=1023) and of the
# cfg4 GMRES operator kernels; summaries produced on the box.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
FDE_GRAPH=0 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
FDE_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
FDE_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:"k_sop|k_sine_xr5" -s 4 -c 2 \
    -o /tmp/prof_iter python tools/unit_run.py --reps 1 --pcg > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
python tools/ncu_summary.py full /tmp/prof_iter.ncu-rep --traffic gpurun_out/traffic_1023.json > gpurun_out/ncu_full_iter.txt 2>&1
python tools/ncu_source.py /tmp/prof_iter.ncu-rep k_sop > gpurun_out/ncu_sop_source.txt 2>&1
FDE_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:"k_toeplitz|k_stau|k_dst_toep" -s 4 -c 4 \
    -o /tmp/prof_cfg4op python tools/unit_run.py --cfg 4 --n 1023 --reps 0 --gmres 4 > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu3 rc=$?"
python tools/ncu_summary.py full /tmp/prof_cfg4op.ncu-rep > gpurun_out/ncu_cfg4_summary.txt 2>&1
