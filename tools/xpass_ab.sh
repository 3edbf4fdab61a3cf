# stage times of the FFT pipeline for the current build (cfg2..cfg5), ESP_XPASS=1
set -x
timeout 200 python tools/stages.py cfg2 cfg3 cfg4 cfg5 > gpurun_out/xp.log 2>&1
cat gpurun_out/xp.log
