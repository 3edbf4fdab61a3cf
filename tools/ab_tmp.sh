#!/bin/bash
mkdir -p gpurun_out
ESP_SPREAD_WARP=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden_large.py tests/test_gpu_tile.py tests/test_gpu_xpass.py -x -q -p no:cacheprovider > gpurun_out/sw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sw_tests.log
tail -3 gpurun_out/sw_tests.log
: > gpurun_out/ab_tmp.log
run() { echo "== $*" >> gpurun_out/ab_tmp.log; env "$@" timeout 300 python tools/stages.py cfg2 cfg3 cfg4 cfg5 2>&1 | cut -c1-170 >> gpurun_out/ab_tmp.log; }
run ESP_SPREAD_WARP=1 ESP_DEBUG_OCC=1
run ESP_SPREAD_WARP=1 ESP_DEBUG_OCC=1 ESP_B200_LIB=libesp_b200_tabs.so
cat gpurun_out/ab_tmp.log
