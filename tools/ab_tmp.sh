#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_tmp.log
run() { echo "== $*" >> gpurun_out/ab_tmp.log; env "$@" timeout 300 python tools/stages.py cfg2 cfg3 cfg5 2>&1 | cut -c1-110 >> gpurun_out/ab_tmp.log; }
run A=1
run ESP_HALF_BLOCK=3,8
run ESP_HALF_BLOCK=4,3
run ESP_HALF_BLOCK=4,4
run ESP_HALF_BLOCK=3,3
run ESP_HALF_BLOCK=2,4
run ESP_HALF_BLOCK=2,3
cat gpurun_out/ab_tmp.log
