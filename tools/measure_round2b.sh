#!/bin/bash
# Round-2 closing measurement on one B200 (run under gpurun): GPU tests on the
# product and the checked build, bench lines cfg1-cfg5, the ncu launch list of
# the default bench command and --set full captures (with source) of the hot
# kernels at cfg5 and cfg4.
set -u
R=${1:-r02f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_smi.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${R}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_gputest.log
ESP_B200_CHECKED=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${R}_chk_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_chk_tests.log
for w in cfg4 cfg5; do
  ESP_B200_CHECKED=1 ESP_GRAPH=0 timeout 300 python tools/run_eval.py --workload $w --reps 2 >> gpurun_out/${R}_chk_runs.log 2>&1; echo "$w rc=$?" >> gpurun_out/${R}_chk_runs.log
done
for w in cfg5 cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --workload $w --steps 20 > gpurun_out/${R}_bench_$w.json 2> gpurun_out/${R}_bench_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches_cfg5.csv python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
for w in cfg5 cfg4; do
  ESP_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:^k_pair_half$|^k_pair_tile$|k_spread|k_interp|k_xpass" -s 5 -c 5 -o gpurun_out/${R}_full_$w \
    python tools/run_eval.py --workload $w --reps 2 > gpurun_out/${R}_ncu_full_$w.log 2>&1
done
tail -2 gpurun_out/${R}_gputest.log gpurun_out/${R}_chk_tests.log; grep -c "ESP_DCHECK failed" gpurun_out/${R}_chk_tests.log gpurun_out/${R}_chk_runs.log; cat gpurun_out/${R}_chk_runs.log | grep rc=
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do python - <<P
import json
d=json.loads(open("gpurun_out/${R}_bench_$w.json").read().strip().splitlines()[-1])
print("$w", round(d["ms_per_step"],4), "%.3g"%d["value"], "e2e %.3g"%d["e2e"]["value"], "frac %.3f"%d["roofline"]["frac"], d["stages_ms"])
P
done
