"""Deterministic mode (esp_plan_set_deterministic): the reference's results
are bit-identical for any thread count (README.md:87-94, test_cli.cpp:174-188);
the default GPU path is not (atomic counting-sort ranks, partner-term REDs,
tile flushes with REDs).  In deterministic mode repeated evaluations -- same
plan, a fresh plan, the graph-replayed device path and the serialised host
path -- must be BITWISE identical, and still match the compiled reference to
the stated tolerances."""
import numpy as np
import pytest
import torch

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu

E_TOL, F_TOL, U_TOL = 1e-11, 1e-10, 1e-10


def _sys(esp, name):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    return esp.ParticleSystem(box, q, pos), c


def _device_eval(esp, plan, s):
    d = torch.device("cuda", 0)
    pos, q = torch.from_numpy(s.pos).to(d), torch.from_numpy(s.q).to(d)
    u = torch.empty(s.size(), dtype=torch.float64, device=d)
    F = torch.empty(3 * s.size(), dtype=torch.float64, device=d)
    e = torch.empty(1, dtype=torch.float64, device=d)
    st = torch.cuda.current_stream()
    for _ in range(3):  # warm-up, graph capture, replays
        esp.evaluate_device(plan, s.box, s.size(), pos.data_ptr(), q.data_ptr(), u.data_ptr(),
                            F.data_ptr(), e.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    return float(e.item()), u.cpu().numpy(), F.cpu().numpy().reshape(-1, 3)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_bitwise_reproducible(esp, gpu, name):
    s, c = _sys(esp, name)
    plan = esp.build_plan(s.box, "pswf", c.eps, c.r_c, device=gpu)
    plan.set_deterministic(True)
    assert plan.deterministic
    a = esp.evaluate(plan, s)
    b = esp.evaluate(plan, s)
    assert a.energy == b.energy and np.array_equal(a.u, b.u) and np.array_equal(a.F, b.F)
    p2 = esp.build_plan(s.box, "pswf", c.eps, c.r_c, device=gpu)
    p2.set_deterministic(True)
    e2, u2, F2 = _device_eval(esp, p2, s)  # overlapped CUDA-graph path, another engine
    assert e2 == a.energy and np.array_equal(u2, a.u) and np.array_equal(F2, a.F)
    g = golden("cfg1.npz" if name == "cfg1" else f"{name}_sub.npz")
    idx = g["idx"] if "idx" in g else np.arange(s.size())
    assert abs(a.energy - float(g["energy"])) <= E_TOL * abs(float(g["energy"]))
    assert rel_rms(a.F[idx], g["F"]) <= F_TOL
    assert max_rel(a.u[idx], g["u"]) <= U_TOL
    # back to the default mode: same results to roundoff
    plan.set_deterministic(False)
    assert not plan.deterministic
    d = esp.evaluate(plan, s)
    assert abs(d.energy - a.energy) <= 1e-13 * abs(a.energy)
    assert rel_rms(d.F, a.F) <= 1e-13


def test_parts_bitwise_reproducible(esp, gpu):
    s, c = _sys(esp, "cfg2")
    plan = esp.build_plan(s.box, "pswf", c.eps, c.r_c, device=gpu)
    plan.set_deterministic(True)
    l1, l2 = esp.local_sum(plan, s), esp.local_sum(plan, s)
    assert np.array_equal(l1.u, l2.u) and np.array_equal(l1.F, l2.F)
    s1, s2 = esp.spectral_sum(plan, s), esp.spectral_sum(plan, s)
    assert np.array_equal(s1.u, s2.u) and np.array_equal(s1.F, s2.F)
    g1, g2 = esp.spread(plan, s), esp.spread(plan, s)
    assert np.array_equal(g1, g2)


def test_noncubic_odd_P_bitwise(esp, gpu):
    from oracle import esp_oracle as O
    box = (10.0, 12.5, 15.0)
    pos, q = O.random_system(600, box, 7)
    s = esp.ParticleSystem(box, q, pos)
    plan = esp.build_plan(box, "pswf", 1e-4, 1.0, esp.Overrides(P=7), device=gpu)
    plan.set_deterministic(True)
    a, b = esp.evaluate(plan, s), esp.evaluate(plan, s)
    assert np.array_equal(a.u, b.u) and np.array_equal(a.F, b.F) and a.energy == b.energy
    o = O.build_plan(box, "pswf", 1e-4, 1.0, P_ov=7)
    Eo, uo, Fo = O.evaluate(o, pos, q)
    assert abs(a.energy - Eo) <= E_TOL * abs(Eo)
    assert rel_rms(a.F, Fo) <= F_TOL
