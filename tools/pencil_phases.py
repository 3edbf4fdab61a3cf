"""Per-rank compute time of the distributed-FFT evaluation, measured on ONE
GPU with the ranks emulated in lockstep (dist.evaluate_pencil_emulated's
phases, each rank timed alone with CUDA events), plus the bytes each rank
moves per evaluation.  This is the compute side of a strong-scaling
projection -- the exchanges themselves need real NVLink peers and are not
timed here.

    python tools/pencil_phases.py cfg5 2 4 8            # replicated inputs
    python tools/pencil_phases.py cfg5 2 4 8 --local    # own atoms + ghosts per rank
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
from paper_2505_09727_b200.dist import (PencilBuffers, PencilLayout, _Lib,  # noqa: E402
                                        atom_owner, evaluate_pencil_emulated, fold_positions,
                                        ghost_masks, pencil_half_enabled)


def main():
    name = sys.argv[1]
    local = "--local" in sys.argv
    ranks = [int(x) for x in sys.argv[2:] if not x.startswith("--")] or [2, 4, 8]
    c = S.config(name)
    pos, q, box = c.system()
    N = q.size
    dev = torch.device("cuda", 0)
    pos_d = torch.from_numpy(pos).to(dev)
    q_d = torch.from_numpy(q).to(dev)
    st = torch.cuda.current_stream()
    s = st.cuda_stream
    plan1 = E.build_plan(box, "pswf", c.eps, c.r_c, device=0)
    u = torch.empty(N, dtype=torch.float64, device=dev)
    F = torch.empty(3 * N, dtype=torch.float64, device=dev)
    e = torch.empty(1, dtype=torch.float64, device=dev)

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    single = timed(lambda: E.evaluate_device(plan1, box, N, pos_d.data_ptr(), q_d.data_ptr(),
                                             u.data_ptr(), F.data_ptr(), e.data_ptr(), s))
    res = {"workload": name, "N": N, "nf": list(plan1.nf), "single_gpu_ms": single,
           "inputs": "local (own + ghosts)" if local else "replicated", "ranks": {}}
    for G in ranks:
        plans = [E.build_plan(box, "pswf", c.eps, c.r_c, device=0) for _ in range(G)]
        lay = PencilLayout.of(plans[0], G)
        if local:
            posf = fold_positions(pos, box)
            own = atom_owner(lay, posf[:, 0])
            masks = [ghost_masks(lay, r, posf[:, 0], box[0], c.r_c) for r in range(G)]
            Ns, poss, qs, nown = [], [], [], []
            for r in range(G):
                lft, rgt = lay.neighbours(r)
                mine = np.nonzero(own == r)[0]
                gh = ((own == lft) & masks[lft][1] | (own == rgt) & masks[rgt][0]) & (own != r)
                loc = np.concatenate([mine, np.nonzero(gh)[0]])
                Ns.append(loc.size)
                nown.append(mine.size)
                poss.append(torch.from_numpy(np.ascontiguousarray(posf[loc]).ravel()).to(dev))
                qs.append(torch.from_numpy(q[loc]).to(dev))
        else:
            Ns, poss, qs, nown = [N] * G, [pos_d] * G, [q_d] * G, [None] * G
        bufs = [PencilBuffers(lay, r, Ns[r], dev) for r in range(G)]
        evaluate_pencil_emulated(plans, box, Ns if local else N, poss if local else pos_d,
                                 qs if local else q_d, bufs, lay, s)  # fills the buffers
        per = []
        for r in range(G):
            b, p = bufs[r], plans[r]
            o = b.out
            Nr, pos_r, q_r = Ns[r], poss[r], qs[r]
            t = {
                "phase_a": timed(lambda: _Lib.pencil_phase_a(p, box, Nr, pos_r, q_r, r, G, b.slab, s)),
                "forward": timed(lambda: _Lib.pencil_forward(p, r, G, b.slab, b.send, s)),
                # solve clobbers recv: time it on a scratch copy
                "solve": timed(lambda: (b.A.copy_(b.recv), _Lib.pencil_solve(p, r, G, b.A, b.A, b.B, s))),
                "backward": timed(lambda: _Lib.pencil_backward(p, r, G, b.A2, b.B2, b.fslab, s)),
                "phase_b": timed(lambda: _Lib.pencil_phase_b(p, r, G, b.fslab, o[:Nr], o[Nr:4 * Nr],
                                                             o[4 * Nr:], s)),
            }
            t["total"] = sum(t.values())
            pl = lay.plane(1) * 8
            halo_bytes = 2 * lay.halo * pl * (1 + lay.nfields)          # out: slab + field halos
            a2a = 8 * (sum(lay.fwd_send_splits(r)) - lay.fwd_send_splits(r)[r]) * \
                (1 + (2 if lay.nfields == 4 else 1))                    # fwd + A (+B), off-rank
            if local:  # ghosts out (32 B each, about the ghosts received) + energy;
                # half-shell K4: plus the ghost rows' partner terms returned (32 B each)
                back = 32 * (Nr - nown[r]) if pencil_half_enabled() else 0
                t["bytes_out"] = halo_bytes + a2a + 32 * (Nr - nown[r]) + back + 8
                t["atoms_own"], t["atoms_ghost"] = nown[r], Nr - nown[r]
            else:      # + output all-reduce
                t["bytes_out"] = halo_bytes + a2a + 8 * (4 * N + 1)
            per.append(t)
        res["ranks"][G] = {"per_rank": per,
                           "max_total_ms": max(t["total"] for t in per),
                           "max_bytes_out": max(t["bytes_out"] for t in per)}
        print(G, json.dumps(res["ranks"][G]["max_total_ms"]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
