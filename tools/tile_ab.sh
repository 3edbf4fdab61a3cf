# K4 cluster-pair checks: the K4 parity tests (cluster kernel auto / forced),
# then stage times: default, forced cluster pairs, column divisor 2 + cluster pairs
set -x
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_half.py tests/test_gpu_golden_large.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/tile_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tile_tests.log
timeout 300 python tools/stages.py ${CFGS:-cfg3 cfg4 cfg5} > gpurun_out/tile_a.log 2>&1
ESP_PAIR_TILE=1 timeout 300 python tools/stages.py cfg3 cfg5 > gpurun_out/tile_b.log 2>&1
ESP_PAIR_TILE=1 ESP_COL_DIV=2 timeout 300 python tools/stages.py cfg3 cfg5 > gpurun_out/tile_c.log 2>&1
ESP_PAIR_TILE=0 ESP_COL_DIV=2 timeout 300 python tools/stages.py cfg5 > gpurun_out/tile_d.log 2>&1
tail -3 gpurun_out/tile_tests.log; cat gpurun_out/tile_a.log gpurun_out/tile_b.log gpurun_out/tile_c.log gpurun_out/tile_d.log
