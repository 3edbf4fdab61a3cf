"""GPU parity at the BASELINE sizes against the compiled reference's own
`evaluate` (ewald.hpp:619-649, ik, run by tests/golden/make_golden_large.py
on the same seeded systems): cfg3 (300k atoms, P = 8), cfg4 (1M ions, P = 5,
r_c = 8) and cfg5 (8M atoms), plus the Gaussian family (kernels.hpp:105-138
split, kernels.hpp:263-273 B-spline window) on cfg1 and cfg2.

Stated tolerances: energy relative 1e-11; forces relative RMS
(the Delta metric, reference.hpp:241-255) 1e-10; potentials max-abs relative
1e-10 -- on every stored atom (every 16th / 64th / 256th) -- and the
whole-system norms sum F^2, sum u^2 to 1e-10 relative, the net force to
1e-10 of the RMS force per atom."""
import numpy as np
import pytest

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu

E_TOL, F_TOL, U_TOL = 1e-11, 1e-10, 1e-10


def _check(ef, g):
    idx = g["idx"]
    assert abs(ef.energy - float(g["energy"])) <= E_TOL * abs(float(g["energy"]))
    assert rel_rms(ef.F[idx], g["F"]) <= F_TOL
    assert max_rel(ef.u[idx], g["u"]) <= U_TOL
    assert abs(np.sum(ef.F ** 2) - float(g["Fnorm2"])) <= 1e-10 * float(g["Fnorm2"])
    assert abs(np.sum(ef.u ** 2) - float(g["unorm2"])) <= 1e-10 * float(g["unorm2"])
    frms = np.sqrt(float(g["Fnorm2"]) / ef.u.size)
    assert np.max(np.abs(np.sum(ef.F, axis=0) - g["Fsum"])) <= 1e-10 * frms * ef.u.size


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_large_config_matches_reference(esp, gpu, name):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    g = golden(f"{name}_sub.npz")
    plan = esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu)
    # graph-replayed overlapped path (the benchmarked one) and the serialised
    # timed path both match
    ef = esp.evaluate(plan, esp.ParticleSystem(box, q, pos), timings=False)
    _check(ef, g)
    if name != "cfg5":
        _check(esp.evaluate(plan, esp.ParticleSystem(box, q, pos)), g)


def test_gaussian_family_matches_reference(esp, gpu):
    from paper_2505_09727_b200 import systems as S
    for name, fx in (("cfg1", "gauss_cfg1.npz"), ("cfg2", "gauss_cfg2_sub.npz")):
        c = S.config(name)
        pos, q, box = c.system()
        g = golden(fx)
        plan = esp.build_plan(box, "gaussian", c.eps, c.r_c, device=gpu)
        assert plan.nf == tuple(int(v) for v in g["nf"]) and plan.P == int(g["P"])
        _check(esp.evaluate(plan, esp.ParticleSystem(box, q, pos)), g)
