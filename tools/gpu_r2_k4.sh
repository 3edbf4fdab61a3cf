set -x
timeout 120 python -m pytest tests/test_gpu_half.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/k4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k4_tests.log
timeout 300 python tools/half_check.py cfg1 cfg2 cfg3 cfg4 cfg5 > gpurun_out/k4_ab.log 2>&1
tail -3 gpurun_out/k4_tests.log; cat gpurun_out/k4_ab.log
