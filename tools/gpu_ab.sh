# usage: bash tools/gpu_ab.sh "ENV_A" "ENV_B" cfgs... ; quick parity tests first
set -x
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_golden_large.py tests/test_gpu_slab.py tests/test_gpu_family.py -x -q -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
A="$1"; B="$2"; shift 2
env $A timeout 200 python tools/stages.py "$@" > gpurun_out/ab_a.log 2>&1
env $B timeout 200 python tools/stages.py "$@" > gpurun_out/ab_b.log 2>&1
tail -2 gpurun_out/ab_tests.log; cat gpurun_out/ab_a.log gpurun_out/ab_b.log
