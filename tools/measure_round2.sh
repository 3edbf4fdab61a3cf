#!/bin/bash
# Round-2 end measurement on one B200 (run under gpurun): bench lines for
# cfg1-cfg4 (cfg5 is the default bench line, see tools/gpu_r2_2.sh), and
# --set full captures of K4/K1/K3 at cfg2 and cfg4.
set -u
R=${1:-r02}
mkdir -p gpurun_out
for w in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --workload $w --steps 20 > gpurun_out/${R}_bench_$w.json 2>gpurun_out/${R}_bench_$w.err
done
for w in cfg2 cfg4; do
  ESP_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"^k_pair_half$|k_spread|k_interp" -s 3 -c 3 -o gpurun_out/${R}_full_$w \
    python tools/run_eval.py --workload $w --reps 2 > gpurun_out/${R}_ncu_full_$w.log 2>&1
done
echo done
