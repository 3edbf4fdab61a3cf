"""Where the end-to-end time of one host-buffer evaluation goes (cfg2 by
default): the public call, the device-resident call, and the bare copies.

    python tools/e2e_breakdown.py [cfg2]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_09727_b200 as E  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402


def wall(fn, reps=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = S.config(name)
pos, q, box = c.system()
N = q.size
plan = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
pos_h, q_h = pin(pos), pin(q)
u_h, F_h = pin(np.empty(N)), pin(np.empty((N, 3)))
s = E.ParticleSystem(box, q_h, pos_h)
dev = torch.device("cuda", 0)
pos_d, q_d = torch.from_numpy(pos).to(dev), torch.from_numpy(q).to(dev)
u_d, F_d, e_d = (torch.empty(N, dtype=torch.float64, device=dev),
                 torch.empty(3 * N, dtype=torch.float64, device=dev),
                 torch.empty(1, dtype=torch.float64, device=dev))
st = torch.cuda.current_stream()


def dev_eval():
    E.evaluate_device(plan, box, N, pos_d.data_ptr(), q_d.data_ptr(), u_d.data_ptr(),
                      F_d.data_ptr(), e_d.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()


pos_t, q_t = torch.from_numpy(pos_h), torch.from_numpy(q_h)
u_t, F_t = torch.from_numpy(u_h), torch.from_numpy(F_h.reshape(-1))


def copies():
    pos_d.copy_(pos_t, non_blocking=True)
    q_d.copy_(q_t, non_blocking=True)
    u_t.copy_(u_d, non_blocking=True)
    F_t.copy_(F_d, non_blocking=True)
    torch.cuda.synchronize()


res = {
    "public evaluate (host buffers)": wall(lambda: E.evaluate(plan, s, out=(u_h, F_h))),
    "evaluate_device + sync": wall(dev_eval),
    "H2D + D2H copies alone": wall(copies),
    "empty sync": wall(torch.cuda.synchronize),
}
for k, v in res.items():
    print(f"{k:34s} {v:8.3f} ms")
