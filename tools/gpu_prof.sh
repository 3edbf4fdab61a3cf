#!/bin/bash
# One-GPU profiling pass (run under gpurun): ncu launch list of the default
# bench command and --set full captures (with source) of K4/K1/K3 at a workload.
# Usage: bash tools/gpu_prof.sh TAG [workload] [kernel-regex]
set -u
T=${1:-r02}
W=${2:-cfg5}
K=${3:-"regex:^k_pair_half$|k_spread|k_interp"}
mkdir -p gpurun_out
ESP_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
  -k "$K" -s ${SKIP:-3} -c ${COUNT:-3} -o gpurun_out/${T}_full_$W \
  python tools/run_eval.py --workload $W --reps 2 > gpurun_out/${T}_ncu_full_$W.log 2>&1
echo "full rc=$?"
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 \
  --no-cpu-baseline > gpurun_out/${T}_ncu_launch_$W.log 2>&1
echo "launch rc=$?"
fi
