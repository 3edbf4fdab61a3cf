"""Slab decomposition over ranks, emulated sequentially on one GPU: each
emulated rank has its own plan (as on separate GPUs); grids and outputs are
summed on the device like the NCCL all-reduces would.  The sum must equal the
single-GPU evaluation."""
import numpy as np
import pytest
import torch

from conftest import max_rel, rel_rms

pytestmark = pytest.mark.gpu


def _slab(esp, box, pos, q, eps, r_c, nranks):
    dev = torch.device("cuda", 0)
    N = q.size
    pos_d = torch.from_numpy(pos).to(dev)
    q_d = torch.from_numpy(q).to(dev)
    plans = [esp.build_plan(box, "pswf", eps, r_c, device=0) for _ in range(nranks)]
    M = esp.grid_size(plans[0])
    grids = [torch.empty(M, dtype=torch.float64, device=dev) for _ in range(nranks)]
    outs = [torch.empty(4 * N + 1, dtype=torch.float64, device=dev) for _ in range(nranks)]
    st = torch.cuda.current_stream().cuda_stream
    for r in range(nranks):
        esp.eval_phase_a(plans[r], box, N, pos_d.data_ptr(), q_d.data_ptr(), r, nranks,
                         grids[r].data_ptr(), st)
    gsum = sum(grids)
    for r in range(nranks):
        o = outs[r]
        esp.eval_phase_b(plans[r], r, nranks, gsum.data_ptr(), o[:N].data_ptr(),
                         o[N:4 * N].data_ptr(), o[4 * N:].data_ptr(), st)
    tot = sum(outs).cpu().numpy()
    return tot[:N], tot[N:4 * N].reshape(N, 3), float(tot[4 * N])


@pytest.mark.parametrize("name,nranks", [("cfg2", 2), ("cfg2", 3), ("cfg4", 4)])
def test_slab_sum_equals_single_gpu(esp, gpu, name, nranks):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    full = esp.evaluate(esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu),
                        esp.ParticleSystem(box, q, pos))
    u, F, E = _slab(esp, box, pos, q, c.eps, c.r_c, nranks)
    assert abs(E - full.energy) <= 1e-12 * abs(full.energy)
    assert rel_rms(F, full.F) <= 1e-12
    assert max_rel(u, full.u) <= 1e-12


def test_slab_all_pairs_fallback(esp, gpu):
    """Small box (nc < 3): the real-space slab is a range of targets."""
    from oracle import esp_oracle as O
    box = (10.0, 10.0, 10.0)
    pos, q = O.random_system(64, box, 17)
    full = esp.evaluate(esp.build_plan(box, "pswf", 1e-3, 3.4, device=gpu),
                        esp.ParticleSystem(box, q, pos))
    u, F, E = _slab(esp, box, pos, q, 1e-3, 3.4, 3)
    assert abs(E - full.energy) <= 1e-12 * abs(full.energy)
    assert rel_rms(F, full.F) <= 1e-12
