"""Cluster-pair K4 (k_pair_tile: a warp evaluates 2 targets x 16 partners with
out-of-range lanes masked) against the reference's golden outputs and the
full-list kernel (k_pair, both orders as in ewald.hpp:473-509), including the
overflow path, non-uniform and non-cubic systems (odd target counts per
column, clusters of one target), and the automatic selection.

ESP_PAIR_TILE (read when a plan is built): -1 / unset = cluster pairs when
the cell columns are r_c/2 wide (~200 in-range pairs per atom, e.g. cfg4),
0 = never, 1 = whenever the half-shell form runs."""
import numpy as np
import pytest

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu


def _plan(esp, monkeypatch, half, tile, box, eps, r_c, gpu, family="pswf"):
    monkeypatch.setenv("ESP_PAIR_HALF", str(half))
    monkeypatch.setenv("ESP_PAIR_TILE", str(tile))
    return esp.build_plan(box, family, eps, r_c, device=gpu)


def _compare_to_full(esp, monkeypatch, gpu, sysm, eps, r_c, tol=1e-12, family="pswf"):
    full = _plan(esp, monkeypatch, 0, 0, sysm.box, eps, r_c, gpu, family)
    lf = esp.local_sum(full, sysm)
    nf = full.last_pair_count()
    assert full.pair_kernel == "full"
    tile = _plan(esp, monkeypatch, 2, 1, sysm.box, eps, r_c, gpu, family)
    lt = esp.local_sum(tile, sysm)
    assert tile.pair_kernel == "tile"
    assert tile.last_pair_count() == nf > 0
    assert max_rel(lt.u, lf.u) <= tol
    assert rel_rms(lt.F, lf.F) <= tol
    return tile, full


def test_tile_cfg1_matches_reference(esp, gpu, monkeypatch):
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg1")
    pos, q, box = c.system()
    sysm = esp.ParticleSystem(box, q, pos)
    g = golden("cfg1.npz")
    plan = _plan(esp, monkeypatch, 2, 1, box, c.eps, c.r_c, gpu)
    loc = esp.local_sum(plan, sysm)
    assert plan.pair_kernel == "tile"
    assert max_rel(loc.u, g["u_local"]) <= 1e-12
    assert rel_rms(loc.F, g["F_local"]) <= 1e-12
    ef = esp.evaluate(plan, sysm)
    assert abs(ef.energy - g["energy"]) <= 1e-11 * abs(g["energy"])
    assert rel_rms(ef.F, g["F"]) <= 1e-10
    assert max_rel(ef.u, g["u"]) <= 1e-10


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_tile_matches_full_list(esp, gpu, monkeypatch, name):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), c.eps, c.r_c)


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_tile_evaluate_matches_reference(esp, gpu, monkeypatch, name):
    """Forced cluster pairs through the whole evaluation (graph path) against
    the compiled reference's fixtures (every 16th / 64th atom, norms)."""
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    g = golden(f"{name}_sub.npz")
    plan = _plan(esp, monkeypatch, 1, 1, box, c.eps, c.r_c, gpu)
    ef = esp.evaluate(plan, esp.ParticleSystem(box, q, pos), timings=False)
    assert plan.pair_kernel == "tile"
    idx = g["idx"]
    assert abs(ef.energy - float(g["energy"])) <= 1e-11 * abs(float(g["energy"]))
    assert rel_rms(ef.F[idx], g["F"]) <= 1e-10
    assert max_rel(ef.u[idx], g["u"]) <= 1e-10
    assert abs(np.sum(ef.F ** 2) - float(g["Fnorm2"])) <= 1e-10 * float(g["Fnorm2"])


def test_tile_auto_selection(esp, gpu, monkeypatch):
    """Default: the half-shell warp-per-target kernel from 4096 atoms (cfg4 with
    r_c/2 columns included: since the end of round 2 it is faster there than
    the cluster pairs, which run only with ESP_PAIR_TILE=1), full lists below."""
    from paper_2505_09727_b200 import systems as S
    monkeypatch.delenv("ESP_PAIR_TILE", raising=False)
    monkeypatch.delenv("ESP_PAIR_HALF", raising=False)
    for name, want in (("cfg4", "half"), ("cfg2", "half"), ("cfg1", "full")):
        c = S.config(name)
        pos, q, box = c.system()
        plan = esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu)
        assert plan.pair_kernel == "none"
        esp.local_sum(plan, esp.ParticleSystem(box, q, pos))
        assert plan.pair_kernel == want, name


def test_tile_overflow_path(esp, gpu, monkeypatch):
    """Capacity far below every block's neighbourhood: all blocks take the
    overflow kernel; the results must not change."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    monkeypatch.setenv("ESP_HALF_CAP", "256")
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), c.eps, c.r_c)


def test_tile_clustered_system(esp, gpu, monkeypatch):
    rng = np.random.default_rng(7)
    L = 60.0
    dense = rng.uniform(20.0, 32.0, size=(24000, 3))
    sparse = rng.uniform(0.0, L, size=(6001, 3))
    pos = np.vstack([dense, sparse])
    q = np.where(np.arange(pos.shape[0]) % 2 == 0, 1.0, -1.0)
    q[-1] = 0.0  # odd atom count, neutral
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(np.array([L, L, L]), q, pos),
                     1e-4, 6.0)


@pytest.mark.parametrize("box,r_c", [((30.0, 41.0, 57.0), 5.0), ((24.0, 24.0, 80.0), 3.0)])
def test_tile_non_cubic(esp, gpu, monkeypatch, box, r_c):
    rng = np.random.default_rng(11)
    box = np.array(box)
    n = int(0.08 * np.prod(box)) // 2 * 2 + 1
    pos = rng.uniform(0.0, 1.0, size=(n, 3)) * box
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    q[-1] = 0.0
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), 1e-4, r_c)


def test_tile_coincident_and_close_atoms(esp, gpu, monkeypatch):
    """Pairs at r = 0 are skipped (as the reference's r2 > 0 test), pairs just
    inside r_c count, a cluster's two targets may coincide."""
    rng = np.random.default_rng(3)
    L = 30.0
    n = 6000
    pos = rng.uniform(0.0, L, size=(n, 3))
    pos[1] = pos[0]            # coincident pair
    pos[3] = pos[2] + [0.0, 0.0, 1e-6]
    pos[5] = pos[4] + [4.0 - 1e-9, 0.0, 0.0]
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(np.array([L, L, L]), q, pos),
                     1e-4, 4.0, tol=1e-11)


def test_tile_gaussian_family(esp, gpu, monkeypatch):
    rng = np.random.default_rng(5)
    L = 40.0
    n = 8000
    pos = rng.uniform(0.0, L, size=(n, 3))
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(np.array([L, L, L]), q, pos),
                     1e-4, 5.0, family="gaussian")


def test_tile_repeated_evaluations(esp, gpu, monkeypatch):
    """Accumulators are zero at rest after the cluster kernel too."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg4")
    pos, q, box = c.system()
    n = 200000
    s = esp.ParticleSystem(box, q[:n], pos[:n])
    plan = _plan(esp, monkeypatch, 2, 1, box, c.eps, c.r_c, gpu)
    a = esp.local_sum(plan, s)
    b = esp.local_sum(plan, s)
    assert max_rel(b.u, a.u) <= 1e-13 and rel_rms(b.F, a.F) <= 1e-13
