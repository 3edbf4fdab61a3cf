set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_gputest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest1.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_cfg5.json 2> gpurun_out/r2_bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_cfg5.json 2> gpurun_out/r2_ref_cfg5.err
tail -3 gpurun_out/r2_gputest1.log
