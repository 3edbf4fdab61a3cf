"""Half-shell K4 (k_pair_half: every unordered pair evaluated once, partner
terms by global REDs into pair-sorted accumulators) against the reference's
golden outputs and against the full-list kernel (k_pair, both orders as in
ewald.hpp:473-509), including the overflow path (blocks whose forward
neighbourhood exceeds the staging capacity, k_pair_half_ovf) and
non-uniform / non-cubic systems.

ESP_PAIR_HALF (read when a plan is built): 0 = full lists, 1 = half-shell from
4096 atoms (default), 2 = half-shell always.  ESP_HALF_CAP (read per launch)
bounds the staging capacity (and forces the half-shell form with the
smallest block, so that the overflow kernel runs).  ESP_PAIR_TILE=0 keeps the
warp-per-target kernel where the cluster-pair one would be chosen."""
import numpy as np
import pytest

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu


def _plan(esp, monkeypatch, mode, box, eps, r_c, gpu):
    monkeypatch.setenv("ESP_PAIR_HALF", str(mode))
    monkeypatch.setenv("ESP_PAIR_TILE", "0")  # warp-per-target kernel (test_gpu_tile.py: clusters)
    return esp.build_plan(box, "pswf", eps, r_c, device=gpu)


def _local(esp, plan, sysm):
    loc = esp.local_sum(plan, sysm)
    return loc, plan.last_pair_count()


def _compare_to_full(esp, monkeypatch, gpu, sysm, eps, r_c, tol=1e-12):
    full = _plan(esp, monkeypatch, 0, sysm.box, eps, r_c, gpu)
    lf, nf = _local(esp, full, sysm)
    half = _plan(esp, monkeypatch, 2, sysm.box, eps, r_c, gpu)
    lh, nh = _local(esp, half, sysm)
    assert full.pair_kernel == "full" and half.pair_kernel == "half"
    assert nh == nf and nf > 0
    assert max_rel(lh.u, lf.u) <= tol
    assert rel_rms(lh.F, lf.F) <= tol
    return half, full


def test_half_cfg1_matches_reference(esp, gpu, monkeypatch):
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg1")
    pos, q, box = c.system()
    sysm = esp.ParticleSystem(box, q, pos)
    g = golden("cfg1.npz")
    plan = _plan(esp, monkeypatch, 2, box, c.eps, c.r_c, gpu)
    loc = esp.local_sum(plan, sysm)
    assert max_rel(loc.u, g["u_local"]) <= 1e-12
    assert rel_rms(loc.F, g["F_local"]) <= 1e-12
    ef = esp.evaluate(plan, sysm)
    assert abs(ef.energy - g["energy"]) <= 1e-11 * abs(g["energy"])
    assert rel_rms(ef.F, g["F"]) <= 1e-10
    assert max_rel(ef.u, g["u"]) <= 1e-10


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_half_matches_full_list(esp, gpu, monkeypatch, name):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), c.eps, c.r_c)


def test_half_overflow_path(esp, gpu, monkeypatch):
    """Capacity far below every block's neighbourhood: all blocks take the
    overflow kernel; the results must not change."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    monkeypatch.setenv("ESP_HALF_CAP", "256")
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), c.eps, c.r_c)


@pytest.mark.parametrize("lcap", ["128", "256"])
def test_half_short_list_pieces(esp, gpu, monkeypatch, lcap):
    """Per-warp list capacity far below a target's candidate count (cfg2:
    ~400 candidates, pieces of 128 / 256 entries): every target takes several
    list pieces, padded column ranges are clipped at piece boundaries and
    survivors that do not fill a round are carried into the next piece."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    monkeypatch.setenv("ESP_PAIR_LCAP", lcap)
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), c.eps, c.r_c)


def test_half_clustered_system(esp, gpu, monkeypatch):
    """Strongly non-uniform density: the dense region's blocks overflow the
    capacity sized for the mean density, the rest take the staged path."""
    rng = np.random.default_rng(7)
    L = 60.0
    n_dense, n_sparse = 24000, 6000
    dense = rng.uniform(20.0, 32.0, size=(n_dense, 3))
    sparse = rng.uniform(0.0, L, size=(n_sparse, 3))
    pos = np.vstack([dense, sparse])
    q = np.where(np.arange(pos.shape[0]) % 2 == 0, 1.0, -1.0)
    sysm = esp.ParticleSystem(np.array([L, L, L]), q, pos)
    _compare_to_full(esp, monkeypatch, gpu, sysm, 1e-4, 6.0)


@pytest.mark.parametrize("box,r_c", [((30.0, 41.0, 57.0), 5.0), ((24.0, 24.0, 80.0), 3.0)])
def test_half_non_cubic(esp, gpu, monkeypatch, box, r_c):
    rng = np.random.default_rng(11)
    box = np.array(box)
    n = int(0.08 * np.prod(box)) // 2 * 2
    pos = rng.uniform(0.0, 1.0, size=(n, 3)) * box
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    _compare_to_full(esp, monkeypatch, gpu, esp.ParticleSystem(box, q, pos), 1e-4, r_c)


def test_half_evaluate_repeated_and_resized(esp, gpu, monkeypatch):
    """The pair-sorted accumulators are zero at rest: repeated evaluations and a
    smaller system on the same plan give identical results."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    plan = _plan(esp, monkeypatch, 2, box, c.eps, c.r_c, gpu)
    s1 = esp.ParticleSystem(box, q, pos)
    a = esp.evaluate(plan, s1)
    b = esp.evaluate(plan, s1)
    assert rel_rms(b.F, a.F) <= 1e-13 and abs(b.energy - a.energy) <= 1e-13 * abs(a.energy)
    n2 = 3 * 6000
    s2 = esp.ParticleSystem(box, q[:n2], pos[:n2])
    l2 = esp.local_sum(plan, s2)
    ref = _plan(esp, monkeypatch, 0, box, c.eps, c.r_c, gpu)
    r2 = esp.local_sum(ref, s2)
    assert max_rel(l2.u, r2.u) <= 1e-12 and rel_rms(l2.F, r2.F) <= 1e-12
    c1 = esp.evaluate(plan, s1)
    assert rel_rms(c1.F, a.F) <= 1e-13


def test_half_gaussian_family(esp, gpu, monkeypatch):
    """Gaussian (Ewald) split: the pair polynomial is the erf kernel's (longer)
    -- half-shell against full lists at N >= 4096."""
    rng = np.random.default_rng(5)
    L = 40.0
    n = 8000
    pos = rng.uniform(0.0, L, size=(n, 3))
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    box = np.array([L, L, L])
    sysm = esp.ParticleSystem(box, q, pos)
    monkeypatch.setenv("ESP_PAIR_HALF", "0")
    monkeypatch.setenv("ESP_PAIR_TILE", "0")
    full = esp.build_plan(box, "gaussian", 1e-4, 5.0, device=gpu)
    lf = esp.local_sum(full, sysm)
    nf = full.last_pair_count()
    monkeypatch.setenv("ESP_PAIR_HALF", "2")
    half = esp.build_plan(box, "gaussian", 1e-4, 5.0, device=gpu)
    lh = esp.local_sum(half, sysm)
    assert half.last_pair_count() == nf > 0
    assert max_rel(lh.u, lf.u) <= 1e-12
    assert rel_rms(lh.F, lf.F) <= 1e-12
    a, b = esp.evaluate(full, sysm), esp.evaluate(half, sysm)
    assert abs(a.energy - b.energy) <= 1e-12 * abs(a.energy)
