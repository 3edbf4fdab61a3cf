export ESP_INTERP_TILE_MIN_N=100000
for xh in 1 2 4; do for nt in 128 256; do
  ESP_TILE_XH=$xh ESP_TILE_NT=$nt timeout 200 python tools/stages.py cfg4 cfg5 2>&1 | sed "s/^/xh=$xh nt=$nt /"
done; done
