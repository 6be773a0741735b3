#!/bin/bash
# sop per-unit phase cycles vs units resident per SM (trace builds; measurement only)
mkdir -p gpurun_out
for v in trace trace3 trace1; do
  FDE_LIB=paper_1912_13304_b200/libfde_$v.so timeout 300 python tools/sop_trace.py 1023 1 > gpurun_out/tr_$v.json 2>&1; echo "$v rc=$?"
done
