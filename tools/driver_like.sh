#!/bin/bash
# What the driver runs at round end, in order (one B200): GPU tests, smoke(),
# the default bench line, the reference arm with default steps.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/dl_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/dl_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/dl_smoke.log
timeout 900 python bench.py > gpurun_out/dl_bench.json 2> gpurun_out/dl_bench.err; echo "bench rc=$?" >> gpurun_out/dl_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/dl_ref.json 2> gpurun_out/dl_ref.err; echo "ref rc=$?" >> gpurun_out/dl_ref.err
tail -2 gpurun_out/dl_gputest.log; cat gpurun_out/dl_smoke.log; tail -n 1 gpurun_out/dl_bench.err; tail -n 1 gpurun_out/dl_ref.err
