"""Host-side plan construction of the product (C ABI, no GPU needed) against
the reference's parameter selection (golden plans) and the numpy oracle."""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import esp_oracle as O

PLANS = json.load(open(os.path.join(GOLDEN, "plans.json")))


@pytest.mark.parametrize("name", sorted(PLANS))
def test_plan_matches_reference(esp, name):
    g = PLANS[name]
    p = esp.build_plan(g["box"], g.get("family", "pswf"), g["eps"], g["r_c"], device=-1)
    assert list(p.nf) == g["nf"] and list(p.base_nf) == g["base_nf"] and p.P == g["P"]
    assert abs(p.shape - g["shape"]) <= 1e-10 * g["shape"]
    if g.get("family", "pswf") == "pswf":
        assert abs(p.c1 - g["c1"]) <= 1e-9 * g["c1"]
    assert abs(p.stats.E_A - g["E_A"]) <= 1e-8 * g["E_A"]
    assert abs(p.stats.E_T - g["E_T"]) <= 1e-8 * max(g["E_T"], 1e-300)
    np.testing.assert_allclose(p.h, g["h"], rtol=1e-15)


def test_reference_parameter_rows(esp):
    """test_ewald.cpp:26-43 / acceptance criterion 1 (shape table)."""
    base = {1e-3: 32, 5e-4: 36, 1e-4: 40, 5e-5: 48, 1e-5: 48}
    order = {1e-3: 5, 5e-4: 5, 1e-4: 6, 5e-5: 7, 1e-5: 8}
    shape = {1e-3: 9.5392, 5e-4: 10.290, 1e-4: 12.024, 5e-5: 12.762, 1e-5: 14.471}
    for eps in base:
        p = esp.build_plan((10.0, 10.0, 10.0), "pswf", eps, 1.0, device=-1)
        assert p.nf == (base[eps],) * 3 and p.P == order[eps]
        tol = 5e-4 if eps in (1e-3, 1e-4, 1e-5) else 5e-3 * shape[eps]
        assert abs(p.shape - shape[eps]) <= tol
        assert p.shape - 1e-12 <= p.c1 <= 1.5 * p.shape + 1e-12
        assert p.stats.E_A <= eps


def test_kernels_match_oracle(esp):
    p = esp.build_plan((10.0, 10.0, 10.0), "pswf", 1e-4, 1.0, device=-1)
    o = O.build_plan((10.0, 10.0, 10.0), "pswf", 1e-4, 1.0)
    y = np.linspace(0.0, 1.0, 2001)
    np.testing.assert_allclose(p.eval_kernel("Psi", y), o.split.Psi(y), atol=1e-13)
    np.testing.assert_allclose(p.eval_kernel("chi", y), o.split.chi(y), atol=1e-12)
    nu = np.linspace(0.0, 40.0, 401)
    np.testing.assert_allclose(p.eval_kernel("chihat_n", nu), o.split.chihat_n(nu), atol=1e-13)
    x = np.linspace(-1.1 * p.P * p.h[0] / 2, 1.1 * p.P * p.h[0] / 2, 3001)
    phi0 = float(o.win[0].phi(0.0))
    np.testing.assert_allclose(p.eval_kernel("phi", x), o.win[0].phi(x), atol=1e-12 * phi0)
    r = np.linspace(0.01, 0.999, 500)
    pot, fr = O.local_kernel(o.split, r)
    # (1 - Psi) -> 0 at r_c: compare on the kernel's own scale
    np.testing.assert_allclose(p.eval_kernel("local_pot", r), pot, atol=1e-13 * pot.max())
    np.testing.assert_allclose(p.eval_kernel("local_fr", r), fr, atol=1e-13 * fr.max())


def test_influence_matches_oracle(esp):
    p = esp.build_plan((10.0, 10.0, 10.0), "pswf", 1e-4, 1.0, device=-1)
    o = O.build_plan((10.0, 10.0, 10.0), "pswf", 1e-4, 1.0)
    a, b = p.influence, o.influence
    assert a[0, 0, 0] == 0.0
    assert np.abs(a - b).max() <= 1e-10 * np.abs(b).max()
    # p_k = p_{-k} bitwise (test_gridder.cpp:115-135)
    flip = a[(-np.arange(40)) % 40][:, (-np.arange(40)) % 40][:, :, (-np.arange(40)) % 40]
    assert np.array_equal(a, flip)
    # beyond the band chihat_n changes sign (as in the reference); signs agree
    big = np.abs(b) > 1e-9 * np.abs(b).max()
    assert np.array_equal(np.sign(a[big]), np.sign(b[big]))


def test_plan_errors_follow_reference(esp):
    """test_ewald.cpp:151-190."""
    box = (10.0, 10.0, 10.0)
    for bad in [dict(eps=1e-6, r_c=1.0), dict(eps=1e-2, r_c=1.0), dict(eps=1e-4, r_c=5.0),
                dict(eps=1e-4, r_c=-1.0)]:
        with pytest.raises(esp.InvalidArgument):
            esp.build_plan(box, "pswf", device=-1, **bad)
    with pytest.raises(esp.InvalidArgument):
        esp.build_plan((0.0, 10.0, 10.0), "pswf", 1e-4, 1.0, device=-1)
    with pytest.raises(esp.InvalidArgument):
        esp.build_plan(box, "pswf", 1e-4, 1.0, esp.Overrides(nf=15), device=-1)
    with pytest.raises(esp.InvalidArgument):
        esp.build_plan(box, "pswf", 1e-4, 1.0, esp.Overrides(P=2), device=-1)
    with pytest.raises(esp.NumericalError):
        esp.build_plan(box, "pswf", 1e-3, 1.0, esp.Overrides(nf=20), device=-1)
    p = esp.build_plan(box, "pswf", 1e-3, 1.0, esp.Overrides(nf=20, allow_degraded=True),
                       device=-1)
    assert p.nf == (20, 20, 20) and max(p.stats.E_A, p.stats.E_T) > 1e-3
    with pytest.raises(esp.NumericalError):  # footprint bound stays hard
        esp.build_plan(box, "pswf", 1e-4, 1.0, esp.Overrides(nf=16, allow_degraded=True),
                       device=-1)


def test_plan_metadata(esp):
    """test_ewald.cpp:510-516."""
    p = esp.build_plan((10.0, 10.0, 10.0), "pswf", 1e-4, 1.0, device=-1)
    assert p.total_modes() == 40 ** 3
    assert abs(p.avg_neighbors(512) - 4.0 * math.pi / 3.0 * 512.0 / 1000.0) <= 1e-12
    assert abs(p.self_coef - p.chi0 / (4 * math.pi)) <= 1e-15
    q = np.array([2.0, -1.0, 0.5])
    np.testing.assert_allclose(esp.self_correction(p, q), q * p.chi0 / (4 * math.pi), rtol=1e-15)


def test_pair_polynomials_are_exact_change_of_basis(esp):
    for eps in (1e-3, 1e-4, 1e-5):
        p = esp.build_plan((10.0, 10.0, 10.0), "pswf", eps, 1.0, device=-1)
        assert p.pair_fit_err <= 2e-14
        assert p.pair_poly_degree <= len(p.prolate_coef(-1)) - 1


def test_select_parameters_matches_golden_plans():
    """ewald.hpp:338-350: select_parameters alone gives the compiled
    reference's (nf, P, c1) for the benchmark configs."""
    import json
    import os
    import paper_2505_09727_b200 as esp
    from paper_2505_09727_b200 import systems as S
    from conftest import GOLDEN
    plans = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for name in ("cfg1", "cfg2", "cfg4"):
        c = S.config(name)
        ref = plans[name]
        sel = esp.select_parameters("pswf", c.eps, (c.L,) * 3, c.r_c)
        assert list(sel["nf"]) == list(ref["nf"]) and sel["P"] == ref["P"]
        assert abs(sel["c1"] - ref["c1"]) <= 1e-12 * abs(ref["c1"])
