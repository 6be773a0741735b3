bash tools/gpu_call_ncu.sh v2 --reps 3
FDE_LIB=$PWD/paper_1912_13304_b200/libfde_kr3.so bash tools/gpu_call_ncu.sh v2kr3 --reps 3
