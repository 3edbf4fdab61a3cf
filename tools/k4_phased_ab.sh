#!/bin/bash
# K4 two-phase targets A/B: parity tests on the default (phased) build path,
# then serialised stage times with ESP_PAIR_PHASED=0 and 1 (cfg2..cfg5)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_golden_large.py tests/test_gpu_slab.py tests/test_gpu_pencil_half.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > gpurun_out/ph_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ph_tests.log
for v in 0 1 0 1; do
  ESP_PAIR_PHASED=$v timeout 300 python tools/stages.py cfg2 cfg3 cfg4 cfg5 >> gpurun_out/ph_stages.log 2>&1
done
tail -3 gpurun_out/ph_tests.log; cat gpurun_out/ph_stages.log
