#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_tmp.log
run() { echo "== $*" >> gpurun_out/ab_tmp.log; env "$@" timeout 300 python tools/stages.py cfg3 cfg5 2>&1 | cut -c1-170 >> gpurun_out/ab_tmp.log; }
run A=1
for v in 1 2 3 4; do run ESP_B200_LIB=libesp_b200_ab$v.so; done
cat gpurun_out/ab_tmp.log
