#!/bin/bash
# compute-sanitizer pass on one B200 (run under gpurun), one tool per call:
#   bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
# Evaluations of cfg1 (full-list K4, eight-lane K3) and cfg2 (half-shell K4,
# thread-per-atom K3), and cfg2 with the fused x pass forced (ESP_XPASS=1);
# CUDA graphs off so every kernel launch is checked individually.
T=${1:-memcheck}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for run in "cfg1 0" "cfg2 0" "cfg2 1"; do
  set -- $run
  ESP_GRAPH=0 ESP_XPASS=$2 timeout 1500 $CS --tool $T --error-exitcode 9 --print-limit 50 \
    python tools/run_eval.py --workload $1 --reps 1 > gpurun_out/san_${T}_$1_x$2.log 2>&1
  echo "$T $1 xpass=$2 rc=$?" | tee -a gpurun_out/san_${T}_summary.txt
  tail -3 gpurun_out/san_${T}_$1_x$2.log | tee -a gpurun_out/san_${T}_summary.txt
done
