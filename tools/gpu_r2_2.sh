#!/bin/bash
# Round-2 measurement pass on one B200 (run under gpurun): GPU tests, the
# default bench line (cfg5), the ncu launch list of the bench command and a
# --set full capture of the hot kernels at cfg5.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2c_bench_cfg5.json 2> gpurun_out/r2c_bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2c_launches_cfg5.csv python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline > gpurun_out/r2c_ncu_launch.log 2>&1
ESP_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
  -k "regex:^k_pair_half$|k_spread|k_interp|k_xpass" -s 4 -c 4 -o gpurun_out/r2c_full_cfg5 \
  python tools/run_eval.py --workload cfg5 --reps 2 > gpurun_out/r2c_ncu_full.log 2>&1
tail -3 gpurun_out/r2c_gputest.log
