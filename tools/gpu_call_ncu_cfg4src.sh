#!/bin/bash
# ncu --set full with source of the cfg 4 GMRES operator's Toeplitz passes; per-opcode and top-instruction stall samples
mkdir -p gpurun_out
FDE_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_toeplitz|k_dst_toep" -s 8 -c 2 \
    -o /tmp/prof_cfg4src python tools/unit_run.py --cfg 4 --n 1023 --reps 0 --gmres 8 > gpurun_out/ncu_cfg4src.log 2>&1; echo "ncu rc=$?"
python tools/ncu_source.py /tmp/prof_cfg4src.ncu-rep k_toeplitz_lines 0 40 > gpurun_out/ncu_cfg4_cols_source.txt 2>&1
python tools/ncu_source.py /tmp/prof_cfg4src.ncu-rep k_dst_toep_rows 0 40 > gpurun_out/ncu_cfg4_rows_source.txt 2>&1
ncu -i /tmp/prof_cfg4src.ncu-rep --page source --csv --kernel-name regex:k_toeplitz_lines --launch-count 1 --print-source cuda,sass > gpurun_out/ncu_cfg4_cols_cuda.csv 2>/dev/null
head -30 gpurun_out/ncu_cfg4_cols_source.txt
