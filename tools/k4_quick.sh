#!/bin/bash
# K4 quick check: the parity tests that exercise the half-shell kernels, then
# serialised stage times of the current build (env passes through)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_golden_large.py tests/test_gpu_slab.py tests/test_gpu_pencil_half.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > gpurun_out/kq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/kq_tests.log
: > gpurun_out/kq_stages.log
for i in 1 2; do
  timeout 300 python tools/stages.py ${@:-cfg2 cfg3 cfg4 cfg5} >> gpurun_out/kq_stages.log 2>&1
done
tail -3 gpurun_out/kq_tests.log; cat gpurun_out/kq_stages.log
