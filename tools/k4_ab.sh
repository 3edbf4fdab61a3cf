# K4 A/B: the parity tests that exercise k_pair_half, then stage times of the
# current build (cfg2..cfg5) twice
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_golden_large.py tests/test_gpu_slab.py tests/test_gpu_pencil_half.py -x -q -p no:cacheprovider > gpurun_out/k4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k4_tests.log
timeout 300 python tools/stages.py cfg2 cfg3 cfg4 cfg5 > gpurun_out/k4_st1.log 2>&1
timeout 300 python tools/stages.py cfg5 > gpurun_out/k4_st2.log 2>&1
tail -2 gpurun_out/k4_tests.log; cat gpurun_out/k4_st1.log gpurun_out/k4_st2.log
