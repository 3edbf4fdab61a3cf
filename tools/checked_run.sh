#!/bin/bash
# The GPU test suite and the benchmark workloads on the CHECKED build
# (libesp_b200_checked.so: device-side bounds checks in K4 staging / lists /
# queues, K1 tile and grid indices, K3 field rows, the fused x pass, the
# counting-sort scatter).  A failed check traps -> CUDA error -> test failure.
mkdir -p gpurun_out
export ESP_B200_CHECKED=1
python -c "import paper_2505_09727_b200 as E; print('loaded', E.LIB_PATH)" > gpurun_out/chk_tests.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider >> gpurun_out/chk_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_tests.log
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do
  for x in 0 1; do
    ESP_GRAPH=0 ESP_XPASS=$x timeout 300 python tools/run_eval.py --workload $w --reps 2 >> gpurun_out/chk_runs.log 2>&1
    echo "$w xpass=$x rc=$?" >> gpurun_out/chk_runs.log
  done
done
grep -c "ESP_DCHECK failed" gpurun_out/chk_tests.log gpurun_out/chk_runs.log
tail -3 gpurun_out/chk_tests.log; grep rc= gpurun_out/chk_runs.log
