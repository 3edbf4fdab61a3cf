"""Multi-process path of bench.py (replicas + max-over-ranks timing) on CPU
with the gloo backend, world_size 2."""
import os

import numpy as np
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_09727_b200 import systems as S
    from paper_2505_09727_b200.dist import env, max_over_ranks, replica_seed, weak_scaling_value
    r, w, lr = env()
    base = S.config("cfg1")
    c = S.Config(base.name, base.kind, base.N, base.L, base.r_c, base.eps,
                 seed=replica_seed(base.seed, r))
    pos, q, box = c.system()
    ms = [1.0 + r, 10.0 - r]  # per-rank "step times"
    mx = max_over_ranks(ms)
    out[r] = (r, w, lr, float(pos[0, 0]), mx, weak_scaling_value(q.size, w, mx[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_and_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert (r0[0], r0[1], r0[2]) == (0, 2, 0) and (r1[0], r1[1], r1[2]) == (1, 2, 1)
    assert r0[3] != r1[3]                       # replicas are distinct systems
    assert r0[4] == r1[4] == [2.0, 10.0]        # element-wise max over ranks
    assert r0[5] == pytest.approx(1000 * 2 / 2e-3)


def test_single_process_identity():
    from paper_2505_09727_b200.dist import max_over_ranks, replica_seed
    assert max_over_ranks([1.5, 2.5]) == [1.5, 2.5]
    assert replica_seed(1, 0) == 1 and replica_seed(1, 3) == 4


class _OracleEngine:
    """CPU stand-in for the per-rank C-ABI phases (test infrastructure): slabs
    are index ranges, the physics is the numpy oracle."""

    def __init__(self, oplan, pos, q):
        from oracle import esp_oracle as O
        self.O, self.p, self.pos, self.q = O, oplan, pos, q

    def _own(self, rank, nranks):
        N = self.q.size
        return slice(N * rank // nranks, N * (rank + 1) // nranks)

    def phase_a(self, plan, box, N, pos, q, rank, nranks, grid, stream):
        own = self._own(rank, nranks)
        g = self.O.spread(self.p, self.O.fold(self.pos[own], box), self.q[own])
        grid.copy_(torch.from_numpy(g.ravel()))
        ul, Fl = self.O.local_sum(self.p, self.pos, self.q)
        self.ul = np.zeros_like(ul)
        self.Fl = np.zeros_like(Fl)
        self.ul[own], self.Fl[own] = ul[own], Fl[own]

    def phase_b(self, plan, rank, nranks, grid, u, F, e, stream):
        own = self._own(rank, nranks)
        us, Fs = self.O.spectral_from_grid(self.p, grid.numpy(), self.pos, self.q)
        uu = self.ul.copy()
        FF = self.Fl.copy()
        uu[own] += us[own] - self.O.self_correction(self.p, self.q)[own]
        FF[own] += Fs[own]
        u.copy_(torch.from_numpy(uu))
        F.copy_(torch.from_numpy(FF.ravel()))
        e.fill_(0.5 * float(np.dot(self.q, uu)))


def _slab_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import esp_oracle as O
    from paper_2505_09727_b200.dist import evaluate_slab
    box = (10.0, 10.0, 10.0)
    pos, q = O.random_system(300, box, 3)
    p = O.build_plan(box, "pswf", 1e-3, 1.0)
    N = q.size
    res = torch.empty(4 * N + 1, dtype=torch.float64)
    grid = torch.empty(int(np.prod(p.nf)), dtype=torch.float64)
    evaluate_slab(p, box, N, None, None, res, grid, rank, world,
                  engine=_OracleEngine(p, pos, q))
    out[rank] = res.numpy().copy()
    dist.destroy_process_group()


def test_slab_decomposition_plumbing_gloo():
    """Two ranks: partial grids and partial outputs summed by all-reduce
    reproduce the single-process evaluation."""
    import numpy as np  # noqa: F811
    from oracle import esp_oracle as O
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    box = (10.0, 10.0, 10.0)
    pos, q = O.random_system(300, box, 3)
    E, u, F = O.evaluate(O.build_plan(box, "pswf", 1e-3, 1.0), pos, q)
    N = q.size
    for r in range(world):
        res = out[r]
        assert np.allclose(res[:N], u, rtol=0, atol=1e-12 * np.abs(u).max())
        assert np.allclose(res[N:4 * N].reshape(N, 3), F, rtol=0, atol=1e-12 * np.abs(F).max())
        assert abs(res[4 * N] - E) <= 1e-12 * abs(E)
