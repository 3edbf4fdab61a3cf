"""Multi-process path of bench.py (replicas + max-over-ranks timing) on CPU
with the gloo backend, world_size 2."""
import os
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
