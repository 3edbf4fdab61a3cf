"""Serialised stage times (ms, median of 5 timed evaluations after 2
warm-ups) and the overlapped graph-replayed step time for workloads; run it
twice with different ESP_* environment settings for an A/B.

    ESP_SPREAD_PEN=0 python tools/stages.py cfg2 cfg5
"""
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_09727_b200 as E  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402

env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("ESP_"))
for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
    c = S.config(name)
    pos, q, box = c.system()
    plan = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
    s = E.ParticleSystem(box, q, pos)
    ts = [E.evaluate(plan, s).timings for _ in range(7)]
    med = {k: round(statistics.median(t[k] for t in ts[2:]) * 1e3, 4) for k in ts[0]
           if k != "total"}
    d = torch.device("cuda", 0)
    pd, qd = torch.from_numpy(pos).to(d), torch.from_numpy(q).to(d)
    u = torch.empty(q.size, dtype=torch.float64, device=d)
    F = torch.empty(3 * q.size, dtype=torch.float64, device=d)
    e = torch.empty(1, dtype=torch.float64, device=d)
    st = torch.cuda.current_stream()

    def step():
        E.evaluate_device(plan, box, q.size, pd.data_ptr(), qd.data_ptr(), u.data_ptr(),
                          F.data_ptr(), e.data_ptr(), st.cuda_stream)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(st)
    for _ in range(10):
        step()
    ev[1].record(st)
    torch.cuda.synchronize()
    fx = os.path.join(ROOT, "tests", "golden", f"{name}_sub.npz")
    erel = float("nan")
    if os.path.exists(fx):
        ref = float(np.load(fx)["energy"])
        erel = abs(float(e.item()) - ref) / abs(ref)
    print(f"{name} [{env}] step {ev[0].elapsed_time(ev[1]) / 10:.4f} ms  E rel vs ref {erel:.1e}  "
          f"stages {med}", flush=True)
