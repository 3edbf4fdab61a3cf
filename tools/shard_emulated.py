"""Emulated sharded evaluation (esp_shard_evaluate_emulated: every rank's
stages in lockstep on ONE GPU, messages as device copies) timed with CUDA
events: the total over ranks / G is the mean per-rank compute of the
sharded step (the NCCL transfers themselves are not included -- they need
real peers).  Prints one JSON line per G.

    python tools/shard_emulated.py cfg5 2 4 8
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_09727_b200 as E  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402


def main():
    name = sys.argv[1]
    ranks = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    c = S.config(name)
    pos, q, box = c.system()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    # single-GPU reference step (graph path)
    p1 = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
    pd, qd = torch.from_numpy(pos).to(dev), torch.from_numpy(q).to(dev)
    u = torch.empty(q.size, dtype=torch.float64, device=dev)
    F = torch.empty(3 * q.size, dtype=torch.float64, device=dev)
    e = torch.empty(1, dtype=torch.float64, device=dev)

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    t1 = timed(lambda: E.evaluate_device(p1, box, q.size, pd.data_ptr(), qd.data_ptr(),
                                         u.data_ptr(), F.data_ptr(), e.data_ptr(),
                                         st.cuda_stream))
    print(json.dumps({"workload": name, "G": 1, "ms": t1}), flush=True)
    del p1
    for G in ranks:
        plans = [E.build_plan(box, "pswf", c.eps, c.r_c, device=0) for _ in range(G)]
        own = E.shard_owner(plans[0], G, pos)
        idx = [np.nonzero(own == r)[0] for r in range(G)]
        nmax = max(i.size for i in idx)
        shards = [E.Shard(plans[r], r, G, nmax) for r in range(G)]
        P = [torch.from_numpy(np.ascontiguousarray(pos[i])).to(dev) for i in idx]
        Q = [torch.from_numpy(q[i]).to(dev) for i in idx]
        U = [torch.empty(i.size, dtype=torch.float64, device=dev) for i in idx]
        Fo = [torch.empty((i.size, 3), dtype=torch.float64, device=dev) for i in idx]
        Eo = [torch.empty(1, dtype=torch.float64, device=dev) for _ in idx]

        def step():
            E.evaluate_sharded_emulated(shards, box, [i.size for i in idx],
                                        [t.data_ptr() for t in P], [t.data_ptr() for t in Q],
                                        [t.data_ptr() for t in U], [t.data_ptr() for t in Fo],
                                        [t.data_ptr() for t in Eo], st.cuda_stream)

        tG = timed(step)
        for s in shards:
            s.check()
        print(json.dumps({"workload": name, "G": G, "ms_all_ranks": tG,
                          "mean_rank_ms": tG / G, "efficiency_vs_1gpu": t1 / tG,
                          "own_atoms": [int(i.size) for i in idx],
                          "ghost_capacity": shards[0].info["ghost_capacity"]}), flush=True)
        del shards, plans


if __name__ == "__main__":
    main()
