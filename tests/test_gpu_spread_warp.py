"""Warp-per-bin spreading (k_spread_warp: one warp owns a spread bin and its
shared-memory tile, a second warp prepares the next 32 atoms' window weights)
against the reference's grid (gridder.hpp:215-241, golden fixture) and against
the CTA-per-bin kernel k_spread, for every window order the kernel is compiled
for (P = 5..8: one or two footprint-pair passes, packed leftovers), non-cubic
boxes, clustered atoms (long runs in one cell) and bins with no atoms.

ESP_SPREAD_WARP (read when a plan is built): -1 / unset = warp-per-bin for
N >= 2^14, 0 = never, 1 = whenever P is in [5, 8]."""
import numpy as np
import pytest

from conftest import golden, max_rel

pytestmark = pytest.mark.gpu


def _plan(esp, monkeypatch, mode, box, eps, r_c, gpu, **kw):
    monkeypatch.setenv("ESP_SPREAD_WARP", str(mode))
    return esp.build_plan(box, "pswf", eps, r_c, device=gpu, **kw)


def test_warp_spread_matches_reference_grid(esp, gpu, monkeypatch):
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg1")
    pos, q, box = c.system()
    g = golden("grid_cfg1.npz")
    sub = esp.ParticleSystem(box, q[:200], pos[:200])
    plan = _plan(esp, monkeypatch, 1, box, c.eps, c.r_c, gpu)
    grid = esp.spread(plan, sub)
    assert plan.spread_kernel == "warp"
    assert max_rel(grid, g["spread"]) <= 1e-13
    cta = _plan(esp, monkeypatch, 0, box, c.eps, c.r_c, gpu)
    grid0 = esp.spread(cta, sub)
    assert cta.spread_kernel == "cta"
    assert max_rel(grid, grid0) <= 1e-13


@pytest.mark.parametrize("eps,P_expect", [(1e-3, 5), (1e-4, 6), (1e-5, 8), (5e-5, 7)])
def test_warp_spread_equals_cta_spread(esp, gpu, monkeypatch, eps, P_expect):
    """Both kernels on the same random ions in a non-cubic box: node for node."""
    from paper_2505_09727_b200 import systems as S
    box = (31.0, 27.5, 35.25)
    pos, q = S.generate_system("random", 6000, box, 5)
    sysm = esp.ParticleSystem(box, q, pos)
    warp = _plan(esp, monkeypatch, 1, box, eps, 6.0, gpu)
    if warp.P != P_expect:
        pytest.skip(f"parameter selection gave P = {warp.P}")
    gw = esp.spread(warp, sysm)
    assert warp.spread_kernel == "warp"
    cta = _plan(esp, monkeypatch, 0, box, eps, 6.0, gpu)
    gc = esp.spread(cta, sysm)
    assert cta.spread_kernel == "cta"
    assert max_rel(gw, gc) <= 1e-13
    # total charge on the grid: sum of the window's partition of unity
    assert abs(gw.sum() - gc.sum()) <= 1e-10 * np.abs(gc).sum()


def test_warp_spread_clustered_and_empty_bins(esp, gpu, monkeypatch):
    """All atoms in a few cells (runs of hundreds of atoms with one tile
    offset, most bins empty), chunk tails of every length."""
    box = (40.0, 40.0, 40.0)
    rng = np.random.default_rng(11)
    for n in (1, 31, 32, 33, 65, 700):
        centres = rng.uniform(0.0, 40.0, (3, 3))
        pos = (centres[rng.integers(0, 3, n)] + rng.uniform(-0.4, 0.4, (n, 3))) % 40.0
        q = rng.uniform(-1.0, 1.0, n)
        sysm = esp.ParticleSystem(box, q, pos)
        warp = _plan(esp, monkeypatch, 1, box, 1e-4, 8.0, gpu)
        gw = esp.spread(warp, sysm)
        assert warp.spread_kernel == "warp"
        cta = _plan(esp, monkeypatch, 0, box, 1e-4, 8.0, gpu)
        gc = esp.spread(cta, sysm)
        assert max_rel(gw, gc) <= 1e-13, n


def test_warp_spread_selected_automatically(esp, gpu, monkeypatch):
    from paper_2505_09727_b200 import systems as S
    monkeypatch.delenv("ESP_SPREAD_WARP", raising=False)
    for name, want in (("cfg1", "cta"), ("cfg2", "warp")):
        c = S.config(name)
        pos, q, box = c.system()
        plan = esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu)
        assert plan.spread_kernel == "none"
        esp.evaluate(plan, esp.ParticleSystem(box, q, pos))
        assert plan.spread_kernel == want, name


def test_warp_spread_evaluate_cfg2_matches_reference(esp, gpu, monkeypatch):
    from paper_2505_09727_b200 import systems as S
    from conftest import rel_rms
    c = S.config("cfg2")
    pos, q, box = c.system()
    g = golden("cfg2_sub.npz")
    plan = _plan(esp, monkeypatch, 1, box, c.eps, c.r_c, gpu)
    ef = esp.evaluate(plan, esp.ParticleSystem(box, q, pos))
    assert plan.spread_kernel == "warp"
    idx = g["idx"]
    assert abs(ef.energy - g["energy"]) <= 1e-11 * abs(g["energy"])
    assert rel_rms(ef.F[idx], g["F"]) <= 1e-10
    assert max_rel(ef.u[idx], g["u"]) <= 1e-10
