"""Distributed FFT with the half-shell K4 (the default; ESP_PENCIL_HALF=0 selects
full lists; read when a plan is built): targets filtered by grid-plane ownership, every pair evaluated on
the rank owning its base atom (same-cell pairs based by position, which all
ranks see identically).  Replicated inputs: partner terms on other ranks'
atoms are summed with the outputs.  Local inputs: the ghost rows carry partner
terms owed to their owners (dist.return_ghost_terms); the emulation adds them
by global index.  Both must equal the single-GPU evaluation."""
import numpy as np
import pytest
import torch

from conftest import max_rel, rel_rms
from test_gpu_pencil import _pencil_local

pytestmark = pytest.mark.gpu


def _emulated_replicated(esp, box, pos, q, eps, r_c, nranks):
    from paper_2505_09727_b200.dist import PencilBuffers, PencilLayout, evaluate_pencil_emulated
    dev = torch.device("cuda", 0)
    plans = [esp.build_plan(box, "pswf", eps, r_c, device=0) for _ in range(nranks)]
    layout = PencilLayout.of(plans[0], nranks)
    N = q.size
    bufs = [PencilBuffers(layout, r, N, dev) for r in range(nranks)]
    pos_d = torch.from_numpy(np.ascontiguousarray(pos).ravel()).to(dev)
    q_d = torch.from_numpy(q).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    out = evaluate_pencil_emulated(plans, box, N, pos_d, q_d, bufs, layout, st).cpu().numpy()
    pairs = sum(p.last_pair_count() for p in plans)
    return out[:N], out[N:4 * N].reshape(N, 3), float(out[4 * N]), pairs


@pytest.mark.parametrize("name,nranks,local", [("cfg2", 2, False), ("cfg2", 4, False),
                                               ("cfg4", 2, False), ("cfg4", 4, False),
                                               ("cfg2", 2, True), ("cfg2", 3, True),
                                               ("cfg4", 4, True), ("cfg4", 8, True)])
def test_pencil_half_equals_single_gpu(esp, gpu, monkeypatch, name, nranks, local):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    p1 = esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu)
    full = esp.evaluate(p1, esp.ParticleSystem(box, q, pos))
    esp.local_sum(p1, esp.ParticleSystem(box, q, pos))
    n1 = p1.last_pair_count()
    monkeypatch.setenv("ESP_PENCIL_HALF", "1")
    if local:
        u, F, E = _pencil_local(esp, box, pos, q, c.eps, c.r_c, nranks, half=True)
    else:
        u, F, E, pairs = _emulated_replicated(esp, box, pos, q, c.eps, c.r_c, nranks)
        assert pairs == n1  # every pair exactly once over the ranks
    assert abs(E - full.energy) <= 1e-12 * abs(full.energy)
    assert rel_rms(F, full.F) <= 1e-12
    assert max_rel(u, full.u) <= 1e-12


@pytest.mark.parametrize("local", [False, True])
def test_pencil_full_lists_still_match(esp, gpu, monkeypatch, local):
    """ESP_PENCIL_HALF=0 (full-list K4 in the distributed FFT) stays correct."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    full = esp.evaluate(esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu),
                        esp.ParticleSystem(box, q, pos))
    monkeypatch.setenv("ESP_PENCIL_HALF", "0")
    if local:
        u, F, E = _pencil_local(esp, box, pos, q, c.eps, c.r_c, 3, half=False)
    else:
        u, F, E, _ = _emulated_replicated(esp, box, pos, q, c.eps, c.r_c, 2)
    assert abs(E - full.energy) <= 1e-12 * abs(full.energy)
    assert rel_rms(F, full.F) <= 1e-12
    assert max_rel(u, full.u) <= 1e-12
