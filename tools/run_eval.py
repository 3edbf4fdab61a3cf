"""Run a few device-resident evaluations of a workload (profiling driver).

    python tools/run_eval.py --workload cfg4 --reps 3
Used under `ncu` (one GPU) to capture the hot kernels; prints the energy."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--force-method", default="ik")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2505_09727_b200 as E  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402

c = S.config(a.workload)
pos, q, box = c.system()
plan = E.build_plan(box, "pswf", c.eps, c.r_c, E.Overrides(force_method=a.force_method), device=0)
d = torch.device("cuda", 0)
pos_d, q_d = torch.from_numpy(pos).to(d), torch.from_numpy(q).to(d)
u_d = torch.empty(q.size, dtype=torch.float64, device=d)
F_d = torch.empty(3 * q.size, dtype=torch.float64, device=d)
e_d = torch.empty(1, dtype=torch.float64, device=d)
for _ in range(a.reps):
    E.evaluate_device(plan, box, q.size, pos_d.data_ptr(), q_d.data_ptr(), u_d.data_ptr(),
                      F_d.data_ptr(), e_d.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print(a.workload, "energy", float(e_d.item()))
