#!/bin/bash
# A/B of library builds (build.py --variant NAME -D...): stage times per variant
# Usage: bash tools/ab_libs.sh "cfg3 cfg5" default p0 p2 ...
mkdir -p gpurun_out
W=$1; shift
: > gpurun_out/ab_libs.log
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then unset ESP_B200_LIB; else export ESP_B200_LIB=libesp_b200_$v.so; fi
  echo "== $v" >> gpurun_out/ab_libs.log
  timeout 300 python tools/stages.py $W 2>&1 | cut -c1-150 >> gpurun_out/ab_libs.log
done
done
cat gpurun_out/ab_libs.log
