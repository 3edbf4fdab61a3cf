#!/bin/bash
# Round-end measurement on one B200 (run under gpurun):
#   bench lines for every workload, the reference arm, the ncu launch list of
#   the default bench command and --set full captures of K4 (+ K1/K3) per workload.
# Usage: bash tools/measure_round.sh r01
set -u
R=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench_cfg2.json 2> gpurun_out/${R}_bench_cfg2.err || exit 1
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${R}_bench_$w.json 2>/dev/null
done
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_ref_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches_cfg2.csv python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
for w in cfg2 cfg4 cfg5; do
  ESP_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"^k_pair_half$|k_spread|k_interp" -s 3 -c 3 -o gpurun_out/${R}_full_$w \
    python tools/run_eval.py --workload $w --reps 2 > gpurun_out/${R}_ncu_full_$w.log 2>&1
done
echo done
