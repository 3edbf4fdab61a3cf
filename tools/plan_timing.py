"""Plan build time, host tables vs device tables: median of
5 whole build_plan calls after a warm-up (CUDA context, engine), per config.

    python tools/plan_timing.py"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_09727_b200 as E  # noqa: E402

CASES = [("cfg2", 68.3542, 1e-4, 10.0), ("cfg3", 144.1289, 1e-5, 10.0),
         ("cfg4", 215.4435, 1e-3, 8.0), ("cfg5", 430.6001, 1e-4, 10.0)]
out = {"host_threads": os.cpu_count(), "cases": {}}
E.build_plan([20.0] * 3, "pswf", 1e-4, 5.0, device=0)  # warm-up
for name, L, eps, rc in CASES:
    res = {}
    for mode in ("0", "1"):
        os.environ["ESP_PLAN_DEVICE"] = mode
        E.build_plan([L] * 3, "pswf", eps, rc, device=0)
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            E.build_plan([L] * 3, "pswf", eps, rc, device=0)
            ts.append(time.perf_counter() - t)
        res["device_tables" if mode == "1" else "host_tables"] = statistics.median(ts) * 1e3
    out["cases"][name] = res
    print(name, {k: round(v, 1) for k, v in res.items()}, "ms", flush=True)
print(json.dumps(out))
