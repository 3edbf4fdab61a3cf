"""Device construction of the plan's O(n_f^3) tables (
csrc/plan_device.cu): the chihat octant of every grid-inflation step and the
influence half spectrum (gridder.hpp:162-210, ewald.hpp:110-143) computed on
the plan's GPU must give the host path's plan -- the same n_f, P, c1 and E_A
-- and the same influence multipliers to roundoff.  ESP_PLAN_DEVICE=0 (read
when a plan is built) selects the host path."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # (family, box, eps, r_c, nf override)
    ("pswf", (10.0, 10.0, 10.0), 1e-4, 1.0, 0),       # cfg1
    ("pswf", (68.3542,) * 3, 1e-4, 10.0, 0),           # cfg2
    ("pswf", (144.1289,) * 3, 1e-5, 10.0, 0),          # cfg3
    ("pswf", (215.4435,) * 3, 1e-3, 8.0, 0),           # cfg4
    ("pswf", (430.6001,) * 3, 1e-4, 10.0, 0),          # cfg5
    ("pswf", (10.0, 10.0, 15.0), 1e-4, 1.0, 0),        # test_ewald.cpp:62-68 box
    ("pswf", (16.0, 16.0, 16.0), 1e-4, 2.0, 32),       # nf pinned
    ("gaussian", (68.3542,) * 3, 1e-4, 10.0, 0),
    ("gaussian", (10.0, 12.0, 14.0), 1e-3, 1.5, 0),
]


def _build(esp, monkeypatch, on_device, fam, box, eps, rc, nf, gpu):
    monkeypatch.setenv("ESP_PLAN_DEVICE", "1" if on_device else "0")
    ov = esp.Overrides(nf=nf) if nf else None
    t = time.perf_counter()
    p = esp.build_plan(np.array(box), fam, eps, rc, ov, device=gpu)
    return p, time.perf_counter() - t


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1][0]}-{c[2]}")
def test_device_plan_matches_host(esp, gpu, monkeypatch, case):
    fam, box, eps, rc, nf = case
    ph, th = _build(esp, monkeypatch, False, fam, box, eps, rc, nf, gpu)
    pd, td = _build(esp, monkeypatch, True, fam, box, eps, rc, nf, gpu)
    assert pd.nf == ph.nf and pd.P == ph.P
    assert pd.c1 == ph.c1 or (np.isnan(pd.c1) and np.isnan(ph.c1))
    assert pd.stats.E_A == pytest.approx(ph.stats.E_A, rel=1e-12)
    ih, idv = ph.influence, pd.influence
    assert ih.shape == idv.shape
    # device sin/cos/exp differ from the host's by an ulp; the window
    # deconvolution 1/phihat^2 amplifies that at the largest |k| (the host table
    # itself agrees with the reference's to ~1e-12)
    scale = np.max(np.abs(ih))
    assert np.max(np.abs(idv - ih)) <= 1e-11 * scale
    print(f"{fam} box={box} nf={pd.nf}: host plan {th * 1e3:.1f} ms, device plan {td * 1e3:.1f} ms")


def test_device_plan_evaluates_like_host(esp, gpu, monkeypatch):
    """An evaluation on the device-built plan equals one on the host-built plan."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    sysm = esp.ParticleSystem(box, q, pos)
    ph, _ = _build(esp, monkeypatch, False, "pswf", box, c.eps, c.r_c, 0, gpu)
    pd, _ = _build(esp, monkeypatch, True, "pswf", box, c.eps, c.r_c, 0, gpu)
    a, b = esp.evaluate(ph, sysm), esp.evaluate(pd, sysm)
    assert abs(a.energy - b.energy) <= 1e-13 * abs(a.energy)
    num = np.sqrt(np.sum((a.F - b.F) ** 2) / np.sum(a.F ** 2))
    assert num <= 1e-13
