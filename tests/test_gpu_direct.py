"""Direct Ewald on the GPU (esp_direct_ewald, the reference's ground-truth
solver reference.hpp:42-238): pinned to the compiled reference's own
direct_ewald output (golden fixtures) and to the numpy target-subset
restatement, then used to certify the ESP path (Delta <= eps,
reference.hpp:241-255) at the benchmark sizes on random target subsets --
beyond the reference's N <= 1e4 cap."""
import numpy as np
import pytest

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu


def _small(name):
    from paper_2505_09727_b200 import systems as S
    g = golden(name + ".npz")
    if name == "cfg1":
        c = S.config("cfg1")
        pos, q, box = c.system()
        return g, pos, q, box, c.eps, c.r_c
    L = float(g["L"])
    box = (L, L, L)
    pos, q = S.generate_system("random", int(g["N"]), box, int(g["seed"]))
    return g, pos, q, box, float(g["eps"]), float(g["r_c"])


@pytest.mark.parametrize("name", ["cfg1", "small_n512", "small_n64_rc34"])
def test_direct_matches_reference_direct(esp, gpu, name):
    g, pos, q, box, eps, r_c = _small(name)
    d = esp.direct_ewald(esp.ParticleSystem(box, q, pos), 1e-9, device=gpu)
    assert abs(d.energy - g["d_energy"]) <= 1e-10 * abs(g["d_energy"])
    assert max_rel(d.u, g["d_u"]) <= 1e-10
    assert rel_rms(d.F, g["d_F"]) <= 1e-10
    assert d.real_shells >= 1 and d.recip_kmax >= 1


def test_direct_target_subset_equals_full(esp, gpu):
    g, pos, q, box, eps, r_c = _small("cfg1")
    s = esp.ParticleSystem(box, q, pos)
    full = esp.direct_ewald(s, 1e-9, device=gpu)
    tg = np.array([0, 5, 17, 999, 500, 3])
    sub = esp.direct_ewald(s, 1e-9, targets=tg, device=gpu)
    assert np.isnan(sub.energy)
    assert max_rel(sub.u, full.u[tg]) <= 1e-12
    assert rel_rms(sub.F, full.F[tg]) <= 1e-12


def test_direct_subset_matches_numpy_restatement(esp, gpu):
    """cfg2 (N = 32001, above the reference's cap): GPU subset vs the numpy
    restatement of direct_ewald_pass (oracle/esp_oracle.py)."""
    from oracle import esp_oracle as O
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    tg = np.random.default_rng(3).choice(q.size, 12, replace=False)
    _, u_o, F_o = O.direct_ewald(pos, q, box, 1e-9, targets=tg)
    d = esp.direct_ewald(esp.ParticleSystem(box, q, pos), 1e-9, targets=tg, device=gpu)
    assert max_rel(d.u, u_o) <= 1e-10
    assert rel_rms(d.F, F_o) <= 1e-10


def test_direct_errors(esp, gpu):
    g, pos, q, box, eps, r_c = _small("small_n512")
    with pytest.raises(esp.InvalidArgument):
        esp.direct_ewald(esp.ParticleSystem(box, q, pos), 1e-13, device=gpu)
    q2 = q.copy()
    q2[0] += 0.5
    with pytest.raises(esp.NumericalError):
        esp.direct_ewald(esp.ParticleSystem(box, q2, pos), 1e-9, device=gpu)
    with pytest.raises(esp.InvalidArgument):
        esp.direct_ewald(esp.ParticleSystem(box, q, pos), 1e-9, targets=[q.size], device=gpu)


@pytest.mark.slow
@pytest.mark.parametrize("name,ntarget", [("cfg2", 1024), ("cfg3", 512), ("cfg4", 512),
                                          ("cfg5", 256)])
def test_esp_within_eps_of_direct_ewald_full_size(esp, gpu, name, ntarget):
    """The paper's accuracy claim at the benchmark sizes: the relative RMS
    force error of the ESP evaluation against direct Ewald stays below the
    requested eps (estimated on a random target subset)."""
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    s = esp.ParticleSystem(box, q, pos)
    ef = esp.evaluate(esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu), s)
    tg = np.random.default_rng(11).choice(q.size, ntarget, replace=False)
    d = esp.direct_ewald(s, 1e-9, targets=tg, device=gpu)
    delta = rel_rms(ef.F[tg], d.F)
    print(f"{name}: Delta(F) on {ntarget} targets = {delta:.3e} (eps {c.eps:g}); "
          f"potential max-rel {max_rel(ef.u[tg], d.u):.3e}")
    assert delta <= c.eps
