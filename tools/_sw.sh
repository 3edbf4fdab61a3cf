for c in 1024 1536; do export ESP_PAIR_CAP=$c; echo cap $c; bash tools/quick_bench.sh cfg2 cfg4 cfg5; done
