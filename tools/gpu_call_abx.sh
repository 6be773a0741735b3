#!/bin/bash
# A/B of library variants (FDE_LIB) on the sine-domain PCG sizes (tools/ab_sop.py).
mkdir -p gpurun_out
for v in "$@"; do
  FDE_LIB=$PWD/paper_1912_13304_b200/libfde${v}.so timeout 300 python tools/ab_sop.py 2>&1 | sed "s/^/[$v] /"
done | tee gpurun_out/abx.txt
