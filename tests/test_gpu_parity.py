"""GPU parity against the reference's own outputs (golden fixtures made by
tests/golden/make_golden.py from the compiled reference).

Tolerances (stated in DESIGN.md): energy relative 1e-11,
forces relative RMS (the Delta metric, reference.hpp:241-255) 1e-10,
potentials max-abs relative 1e-10.  Summation order differs (atomics,
cuFFT vs FFTW), so results are not bitwise."""
import numpy as np
import pytest

from conftest import golden, max_rel, rel_rms

pytestmark = pytest.mark.gpu

E_TOL, F_TOL, U_TOL = 1e-11, 1e-10, 1e-10


def _cfg1(esp):
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg1")
    pos, q, box = c.system()
    return esp.ParticleSystem(box, q, pos), c


def test_cfg1_evaluate_matches_reference(esp, gpu):
    sysm, c = _cfg1(esp)
    g = golden("cfg1.npz")
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, device=gpu)
    assert plan.nf == (40, 40, 40) and plan.P == 6
    ef = esp.evaluate(plan, sysm)
    assert abs(ef.energy - g["energy"]) <= E_TOL * abs(g["energy"])
    assert rel_rms(ef.F, g["F"]) <= F_TOL
    assert max_rel(ef.u, g["u"]) <= U_TOL


def test_cfg1_parts_match_reference(esp, gpu):
    sysm, c = _cfg1(esp)
    g = golden("cfg1.npz")
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, device=gpu)
    loc = esp.local_sum(plan, sysm)
    assert max_rel(loc.u, g["u_local"]) <= 1e-12
    assert rel_rms(loc.F, g["F_local"]) <= 1e-12
    sp = esp.spectral_sum(plan, sysm)
    assert max_rel(sp.u, g["u_spec"]) <= U_TOL
    assert rel_rms(sp.F, g["F_spec"]) <= F_TOL
    np.testing.assert_allclose(esp.self_correction(plan, sysm.q), g["self"], rtol=1e-13)


def test_cfg1_direct_ewald_within_eps(esp, gpu):
    """Delta <= eps against direct Ewald (reference.hpp:212-255)."""
    sysm, c = _cfg1(esp)
    g = golden("cfg1.npz")
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, device=gpu)
    ef = esp.evaluate(plan, sysm)
    assert rel_rms(ef.F, g["d_F"]) <= c.eps
    assert abs(ef.energy - g["d_energy"]) <= 10 * c.eps * abs(g["d_energy"])


def test_cfg1_ad_matches_reference(esp, gpu):
    sysm, c = _cfg1(esp)
    g = golden("cfg1.npz")
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, esp.Overrides(force_method="ad"),
                          device=gpu)
    ef = esp.evaluate(plan, sysm)
    assert abs(ef.energy - g["ad_energy"]) <= E_TOL * abs(g["ad_energy"])
    assert rel_rms(ef.F, g["ad_F"]) <= F_TOL


@pytest.mark.parametrize("name", ["small_n16", "small_n128", "small_n512", "small_n64_rc1",
                                  "small_n64_rc34"])
def test_small_systems(esp, gpu, name):
    from paper_2505_09727_b200 import systems as S
    g = golden(name + ".npz")
    L = float(g["L"])
    box = (L, L, L)
    pos, q = S.generate_system("random", int(g["N"]), box, int(g["seed"]))
    sysm = esp.ParticleSystem(box, q, pos)
    plan = esp.build_plan(box, "pswf", float(g["eps"]), float(g["r_c"]), device=gpu)
    loc = esp.local_sum(plan, sysm)
    assert max_rel(loc.u, g["u_local"]) <= 1e-12
    ef = esp.evaluate(plan, sysm)
    assert abs(ef.energy - g["energy"]) <= E_TOL * abs(g["energy"])
    assert rel_rms(ef.F, g["F"]) <= F_TOL
    assert rel_rms(ef.F, g["d_F"]) <= float(g["eps"])


def test_rocksalt_madelung(esp, gpu):
    """test_ewald.cpp:493-508: E = -M/pi within 1e-4, forces vanish."""
    from paper_2505_09727_b200 import systems as S
    pos, q = S.generate_system("rocksalt", 8, (2.0, 2.0, 2.0))
    plan = esp.build_plan((2.0, 2.0, 2.0), "pswf", 1e-5, 0.5, device=gpu)
    ef = esp.evaluate(plan, esp.ParticleSystem((2.0, 2.0, 2.0), q, pos))
    expect = -1.7475645946331822 / np.pi
    assert abs(ef.energy - expect) <= 1e-4 * abs(expect)
    assert np.abs(ef.F).max() <= 1e-6
    g = golden("small_rocksalt.npz")
    assert abs(ef.energy - g["energy"]) <= E_TOL * abs(g["energy"])


def test_spread_and_interpolate_match_reference(esp, gpu):
    sysm, c = _cfg1(esp)
    g = golden("grid_cfg1.npz")
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, device=gpu)
    sub = esp.ParticleSystem(sysm.box, sysm.q[:200], sysm.pos[:200])
    grid = esp.spread(plan, sub)
    assert max_rel(grid, g["spread"]) <= 1e-13
    field = np.random.default_rng(8).uniform(-1.0, 1.0, plan.nf)
    assert max_rel(esp.interpolate(plan, field, sub), g["interp"]) <= 1e-13
    assert max_rel(esp.interpolate_gradient(plan, field, sub), g["interp_grad"]) <= 1e-12


def test_cfg2_subsample_matches_reference(esp, gpu):
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    g = golden("cfg2_sub.npz")
    plan = esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu)
    ef = esp.evaluate(plan, esp.ParticleSystem(box, q, pos))
    idx = g["idx"]
    assert abs(ef.energy - g["energy"]) <= E_TOL * abs(g["energy"])
    assert rel_rms(ef.F[idx], g["F"]) <= F_TOL
    assert max_rel(ef.u[idx], g["u"]) <= U_TOL


def test_device_errors_follow_reference(esp, gpu):
    """ewald.hpp:620-622: box mismatch -> invalid_argument; non-neutral -> NumericalError."""
    from paper_2505_09727_b200 import systems as S
    box = (10.0, 10.0, 10.0)
    plan = esp.build_plan(box, "pswf", 1e-3, 1.0, device=gpu)
    pos, q = S.generate_system("random", 8, (8.0, 8.0, 8.0), 1)
    with pytest.raises(esp.InvalidArgument):
        esp.evaluate(plan, esp.ParticleSystem((8.0, 8.0, 8.0), q, pos))
    with pytest.raises(esp.InvalidArgument):
        esp.spectral_sum(plan, esp.ParticleSystem((8.0, 8.0, 8.0), q, pos))
    pos, q = S.generate_system("random", 8, box, 1)
    q = q.copy()
    q[0] = 2.0
    with pytest.raises(esp.NumericalError):
        esp.evaluate(plan, esp.ParticleSystem(box, q, pos))


@pytest.mark.parametrize("N", [64, 200_000])
def test_non_neutral_leaves_outputs_untouched(esp, gpu, N):
    """ewald.hpp:622: require_neutral runs before any work, so a NumericalError
    leaves the caller's output arrays as they were (both the zero-copy path,
    N <= 2^17, and the bulk-copy path)."""
    from paper_2505_09727_b200 import systems as S
    L = 10.0 if N < 1000 else 60.0
    box = (L, L, L)
    plan = esp.build_plan(box, "pswf", 1e-3, 3.0 if N > 1000 else 1.0, device=gpu)
    pos, q = S.generate_system("random", N, box, 3)
    q = q.copy()
    q[1] += 1e-6
    u = np.full(N, 7.0)
    F = np.full((N, 3), -3.0)
    with pytest.raises(esp.NumericalError):
        esp.evaluate(plan, esp.ParticleSystem(box, q, pos), timings=False, out=(u, F))
    assert np.all(u == 7.0) and np.all(F == -3.0)
    # the plan stays usable after the error
    q[1] -= 1e-6
    ef = esp.evaluate(plan, esp.ParticleSystem(box, q, pos), timings=False, out=(u, F))
    assert np.isfinite(ef.energy) and not np.all(u == 7.0)


def test_stage_timings_follow_reference_keys(esp, gpu):
    """ewald.hpp:628-634 / test_ewald.cpp:378-380: evaluate reports the six
    stage times; spectral_sum adds its five into the caller's map."""
    sysm, c = _cfg1(esp)
    plan = esp.build_plan(sysm.box, "pswf", c.eps, c.r_c, device=gpu)
    ef = esp.evaluate(plan, sysm)
    for k in ("local", "spread", "fft", "ifft", "interpolate"):
        assert ef.timings[k] > 0.0
    assert ef.timings["scale"] >= 0.0  # fused into the FFT callbacks: ~0
    t = {"spread": 1.0}
    esp.spectral_sum(plan, sysm, timings=t)
    assert set(t) == {"spread", "fft", "scale", "ifft", "interpolate"} and t["spread"] > 1.0


def test_zero_and_empty(esp, gpu):
    """test_ewald.cpp:282-291: zero charges give a zero field; N=0 is valid."""
    from paper_2505_09727_b200 import systems as S
    box = (10.0, 10.0, 10.0)
    plan = esp.build_plan(box, "pswf", 1e-3, 1.0, device=gpu)
    pos, q = S.generate_system("random", 10, box, 5)
    sp = esp.spectral_sum(plan, esp.ParticleSystem(box, np.zeros(10), pos))
    assert np.all(sp.u == 0.0) and np.all(sp.F == 0.0)
    ef = esp.evaluate(plan, esp.ParticleSystem(box, np.zeros(0), np.zeros((0, 3))))
    assert ef.energy == 0.0 and ef.u.shape == (0,)


@pytest.mark.parametrize("col_div", ["2", "3"])
@pytest.mark.parametrize("name", ["cfg1", "small_n512", "small_n64_rc1"])
def test_pair_cell_widths(esp, gpu, name, col_div, monkeypatch):
    """Both pair-cell column widths (r_c/2, r_c/3; the engine picks one by
    system size) give the reference's real-space sum."""
    from paper_2505_09727_b200 import systems as S
    monkeypatch.setenv("ESP_COL_DIV", col_div)
    g = golden(name + ".npz")
    if name == "cfg1":
        c = S.config("cfg1")
        pos, q, box = c.system()
        eps, r_c = c.eps, c.r_c
    else:
        L = float(g["L"])
        box = (L, L, L)
        pos, q = S.generate_system("random", int(g["N"]), box, int(g["seed"]))
        eps, r_c = float(g["eps"]), float(g["r_c"])
    sysm = esp.ParticleSystem(box, q, pos)
    plan = esp.build_plan(box, "pswf", eps, r_c, device=gpu)
    loc = esp.local_sum(plan, sysm)
    assert max_rel(loc.u, g["u_local"]) <= 1e-12
    assert rel_rms(loc.F, g["F_local"]) <= 1e-12
    ef = esp.evaluate(plan, sysm)
    assert abs(ef.energy - g["energy"]) <= E_TOL * abs(g["energy"])
    assert rel_rms(ef.F, g["F"]) <= F_TOL


def test_pinned_host_buffers(esp, gpu):
    """Page-locked host arrays take the zero-copy path (positions read and
    u/F written over PCIe by the kernels); results equal the pageable path."""
    import torch
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    plan = esp.build_plan(box, "pswf", c.eps, c.r_c, device=gpu)
    ref = esp.evaluate(plan, esp.ParticleSystem(box, q, pos))
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    sp = esp.ParticleSystem(box, pin(q), pin(pos))
    u, F = pin(np.empty(q.size)), pin(np.empty((q.size, 3)))
    for _ in range(3):  # eager, captured, replayed
        u[:] = np.nan
        F[:] = np.nan
        ef = esp.evaluate(plan, sp, out=(u, F))
        assert abs(ef.energy - ref.energy) <= 1e-13 * abs(ref.energy)
        assert max_rel(u, ref.u) <= 1e-13 and rel_rms(F, ref.F) <= 1e-13
    q2 = pin(q.copy())
    q2[0] += 1.0
    with pytest.raises(esp.NumericalError):
        esp.evaluate(plan, esp.ParticleSystem(box, q2, pin(pos)))


def test_fft_conventions(esp, gpu):
    """gridder.hpp:6-13: forward e^{-i} unnormalised (numpy's fftn), inverse
    e^{+i} unnormalised; inverse(forward(g)) = N g (test_gridder.cpp:44-76)."""
    g = np.random.default_rng(4).normal(size=(6, 10, 15)) + 1j * np.random.default_rng(5).normal(size=(6, 10, 15))
    f = esp.fft_forward(g, device=gpu)
    assert np.abs(f - np.fft.fftn(g)).max() <= 1e-12 * np.abs(f).max()
    back = esp.fft_inverse(f, device=gpu)
    assert np.abs(back / g.size - g).max() <= 1e-13 * np.abs(g).max()
