"""K2 fused into the FFT's x pass (k_xpass, engine.cu): the 2-D cuFFT
planes + fused x DFTs / influence multiply / ik derivatives must reproduce
the reference (ewald.hpp:545-548, 567-595; gridder.hpp:162-210) like the
3-D cuFFT + k_scale path.  The fused path is the default for every even
5-smooth n_x; ESP_XPASS=0 forces the 3-D path; both are compared with the
compiled reference's fixtures and with each other."""
import numpy as np
import pytest

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu

E_TOL, F_TOL, U_TOL = 1e-11, 1e-10, 1e-10


def _sys(esp, name):
    from paper_2505_09727_b200 import systems as S
    c = S.config(name)
    pos, q, box = c.system()
    return esp.ParticleSystem(box, q, pos), c


@pytest.mark.parametrize("mode", ["0", "1"])
@pytest.mark.parametrize("fm", ["ik", "ad"])
def test_cfg1_both_paths_match_reference(esp, gpu, monkeypatch, mode, fm):
    monkeypatch.setenv("ESP_XPASS", mode)
    sysm, c = _sys(esp, "cfg1")
    g = golden("cfg1.npz")
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, esp.Overrides(force_method=fm),
                          device=gpu)
    ef = esp.evaluate(plan, sysm)
    pre = "" if fm == "ik" else "ad_"
    e, u, F = g[pre + "energy"], g[pre + "u"], g[pre + "F"]
    assert abs(ef.energy - e) <= E_TOL * abs(e)
    assert rel_rms(ef.F, F) <= F_TOL
    assert max_rel(ef.u, u) <= U_TOL
    sp = esp.spectral_sum(plan, sysm)
    if fm == "ik":
        assert max_rel(sp.u, g["u_spec"]) <= U_TOL
        assert rel_rms(sp.F, g["F_spec"]) <= F_TOL


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_fused_matches_reference_and_3d_path(esp, gpu, monkeypatch, name):
    sysm, c = _sys(esp, name)
    g = golden(f"{name}_sub.npz")
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ESP_XPASS", mode)
        plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, device=gpu)
        ef = esp.evaluate(plan, sysm)
        idx = g["idx"]
        assert abs(ef.energy - float(g["energy"])) <= E_TOL * abs(float(g["energy"]))
        assert rel_rms(ef.F[idx], g["F"]) <= F_TOL
        assert max_rel(ef.u[idx], g["u"]) <= U_TOL
        res[mode] = ef
    # the two transform paths agree to roundoff on every atom
    assert rel_rms(res["1"].F, res["0"].F) <= 1e-12
    assert max_rel(res["1"].u, res["0"].u) <= 1e-12


def _vs_oracle(esp, gpu, box, N, seed, eps, r_c, nf=0, P=0, fm="ik"):
    from oracle import esp_oracle as O
    pos, q = O.random_system(N, box, seed)
    o = O.build_plan(box, "pswf", eps, r_c, nf_ov=nf, P_ov=P, force_method=fm,
                     allow_degraded=True)
    Eo, uo, Fo = O.evaluate(o, pos, q)
    p = esp.build_plan(box, "pswf", eps, r_c,
                       esp.Overrides(nf=nf, P=P, force_method=fm, allow_degraded=True),
                       device=gpu)
    assert p.nf == o.nf and p.P == o.P
    ef = esp.evaluate(p, esp.ParticleSystem(box, q, pos))
    assert abs(ef.energy - Eo) <= E_TOL * abs(Eo)
    assert rel_rms(ef.F, Fo) <= F_TOL
    assert max_rel(ef.u, uo) <= U_TOL


@pytest.mark.parametrize("fm", ["ik", "ad"])
def test_fused_noncubic_vs_oracle(esp, gpu, monkeypatch, fm):
    """n_x, n_y, n_z all different (the x pass indexes [x][ky][kz] with its
    own n_x; xi_y / xi_z by ky / kz), odd P."""
    monkeypatch.setenv("ESP_XPASS", "1")
    _vs_oracle(esp, gpu, (10.0, 12.5, 15.0), 600, 7, 1e-4, 1.0, P=7, fm=fm)


def test_non_smooth_override_keeps_3d_path(esp, gpu, monkeypatch):
    """n_f = 42 = 2 * 3 * 7 (even, an explicit override, not 5-smooth): the
    fused pass has radices 2-5 only, so the 3-D path runs even when forced."""
    monkeypatch.setenv("ESP_XPASS", "1")
    _vs_oracle(esp, gpu, (10.0, 10.0, 10.0), 500, 5, 1e-4, 1.0, nf=42)


def test_mode_reported_by_plan(esp, gpu, monkeypatch):
    """esp_plan_info.fused_xpass: on by default for even 5-smooth n_x (every
    auto-selected grid), never for non-smooth n_x, off with ESP_XPASS=0."""
    from paper_2505_09727_b200 import systems as S
    monkeypatch.delenv("ESP_XPASS", raising=False)
    c5 = S.config("cfg5")
    assert esp.build_plan((c5.L,) * 3, "pswf", c5.eps, c5.r_c, device=gpu).fused_xpass
    assert esp.build_plan((10.0,) * 3, "pswf", 1e-4, 1.0, device=gpu).fused_xpass
    monkeypatch.setenv("ESP_XPASS", "1")
    assert esp.build_plan((10.0,) * 3, "pswf", 1e-4, 1.0, device=gpu).fused_xpass
    assert not esp.build_plan((10.0,) * 3, "pswf", 1e-4, 1.0, esp.Overrides(nf=42),
                              device=gpu).fused_xpass
    monkeypatch.setenv("ESP_XPASS", "0")
    assert not esp.build_plan((c5.L,) * 3, "pswf", c5.eps, c5.r_c, device=gpu).fused_xpass
