#!/bin/bash
mkdir -p gpurun_out
ESP_B200_CHECKED=1 ESP_SPREAD_WARP=1 timeout 900 python -m pytest tests/test_gpu_spread_warp.py tests/test_gpu_parity.py tests/test_gpu_golden_large.py tests/test_gpu_xpass.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/sw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sw_tests.log
tail -3 gpurun_out/sw_tests.log; grep -c "ESP_DCHECK failed" gpurun_out/sw_tests.log
: > gpurun_out/ab_tmp.log
run() { echo "== $*" >> gpurun_out/ab_tmp.log; env "$@" timeout 300 python tools/stages.py cfg2 cfg3 cfg4 cfg5 2>&1 | cut -c1-170 >> gpurun_out/ab_tmp.log; }
run ESP_DEBUG_OCC=1
cat gpurun_out/ab_tmp.log
