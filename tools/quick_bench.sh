#!/bin/bash
# quick per-workload summary lines (used during development)
for w in "$@"; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 10 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print(d['config']['workload'], round(d['ms_per_step'],3), 'ms', {k:round(v,3) for k,v in d['stages_ms'].items()}, 'frac', round(d['roofline']['frac'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],3))"
done
