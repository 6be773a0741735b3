timeout 1100 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log | grep -E "passed|failed"
timeout 600 python tools/sweep.py --only 1,3,5 > gpurun_out/sweep.jsonl 2>&1
