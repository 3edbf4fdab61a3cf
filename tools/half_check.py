"""A/B check of the K4 variants: half-shell (default) vs full-list.

    python tools/half_check.py cfg2 cfg4 ...
For each workload: real-space parts (local_sum) of both variants compared
(potentials max-rel, forces rel-RMS), pair counts, and the serialised K4 stage
time of a timed evaluation."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_09727_b200 as E  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402


def run(name, half):
    os.environ["ESP_PAIR_HALF"] = "1" if half else "0"
    c = S.config(name)
    pos, q, box = c.system()
    plan = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
    s = E.ParticleSystem(box, q, pos)
    loc = E.local_sum(plan, s)
    npair = plan.last_pair_count()
    ts = []
    for _ in range(6):
        ef = E.evaluate(plan, s, timings=True)
        ts.append(ef.timings["local"])
    return loc, npair, min(ts[2:]), ef.energy


for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg4"]:
    lf, nf, tf, ef = run(name, False)
    lh, nh, th, eh = run(name, True)
    du = np.max(np.abs(lh.u - lf.u)) / np.max(np.abs(lf.u))
    dF = np.sqrt(np.sum((lh.F - lf.F) ** 2) / np.sum(lf.F ** 2))
    print(f"{name}: pairs full={nf} half={nh}  u max-rel={du:.2e} F rel-rms={dF:.2e}  "
          f"E rel={abs(eh - ef) / abs(ef):.2e}  K4 full={tf * 1e3:.3f} ms half={th * 1e3:.3f} ms",
          flush=True)
