#!/bin/bash
# ncu --set full of the n=4095 sop operator + vector step, and of the cfg4
# standard-basis operator kernels (τ rows/cols DST, variable Toeplitz rows/cols);
# summaries and raw CSV are produced on the box (the .ncu-rep files are too big to bring back)
mkdir -p gpurun_out
FDE_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sop|k_sine_xr5" -s 4 -c 2 \
    -o /tmp/prof_sop4095 python tools/unit_run.py --n 4095 --reps 1 --pcg > gpurun_out/ncu_4095.log 2>&1; echo "ncu4095 rc=$?"
python tools/ncu_summary.py full /tmp/prof_sop4095.ncu-rep > gpurun_out/ncu_4095_summary.txt 2>&1
ncu -i /tmp/prof_sop4095.ncu-rep --page raw --csv > gpurun_out/ncu_4095_raw.csv 2>&1
FDE_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_toeplitz|k_dstm" -s 5 -c 5 \
    -o /tmp/prof_cfg4op python tools/unit_run.py --cfg 4 --n 1023 --reps 2 > gpurun_out/ncu_cfg4.log 2>&1; echo "ncucfg4 rc=$?"
python tools/ncu_summary.py full /tmp/prof_cfg4op.ncu-rep > gpurun_out/ncu_cfg4_summary.txt 2>&1
ncu -i /tmp/prof_cfg4op.ncu-rep --page raw --csv > gpurun_out/ncu_cfg4_raw.csv 2>&1
ls -la gpurun_out
