"""K4 half-shell block-shape sweep (serialised K4 stage time, timings=True path).

    python tools/half_sweep.py cfg2 "2,3" "2,2" "1,4" ...   (bx,bz; "auto" = heuristic)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_09727_b200 as E  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402

name, shapes = sys.argv[1], sys.argv[2:] or ["auto"]
c = S.config(name)
pos, q, box = c.system()
plan = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
s = E.ParticleSystem(box, q, pos)
ref = None
for sh in shapes:
    if sh == "auto":
        os.environ.pop("ESP_HALF_BLOCK", None)
    else:
        os.environ["ESP_HALF_BLOCK"] = sh
    ts = []
    for _ in range(5):
        ef = E.evaluate(plan, s, timings=True)
        ts.append(ef.timings["local"])
    ref = ref if ref is not None else ef.energy
    print(f"{name} block={sh:6s} cap={os.environ.get('ESP_HALF_CAP', 'def')} K4 min={min(ts[1:]) * 1e3:.3f} ms "
          f"med={sorted(ts[1:])[2] * 1e3:.3f} ms dE={abs(ef.energy - ref) / abs(ref):.1e}", flush=True)
