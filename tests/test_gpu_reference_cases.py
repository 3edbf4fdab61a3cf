"""More of the reference's own test cases, restated against the GPU path:
the truncated mode sum (test_ewald.cpp:293-338), forces as the negative
energy gradient for `ad` (test_ewald.cpp:440-461), the acceptance negative
control (acceptance.cpp:389-414) and the large-lattice family comparison
(acceptance.cpp:417-445)."""
import math

import numpy as np
import pytest

from conftest import rel_rms

pytestmark = pytest.mark.gpu


def _random(esp, N, box, seed):
    from paper_2505_09727_b200 import systems as S
    pos, q = S.generate_system("random", N, box, seed)
    return esp.ParticleSystem(box, q, pos)


def test_long_range_matches_truncated_mode_sum(esp, gpu):
    """Pinned coarse grid (n_f = 16, eps 1e-3, degraded allowed): the spectral
    part sits within 1.5 E_A of the exact truncated mode sum."""
    box = (10.0, 10.0, 10.0)
    plan = esp.build_plan(box, "pswf", 1e-3, 1.0, esp.Overrides(nf=16, allow_degraded=True),
                          device=gpu)
    s = _random(esp, 10, box, 1)
    f = esp.spectral_sum(plan, s)
    V = box[0] * box[1] * box[2]
    m = np.array([i if 2 * i < 16 else i - 16 for i in range(16)], dtype=float)  # signed_mode
    kx, ky, kz = np.meshgrid(*(2 * math.pi * m / L for L in box), indexing="ij")
    xi = np.stack([kx.ravel(), ky.ravel(), kz.ravel()], axis=1)[1:]  # drop (0, 0, 0)
    mag = np.linalg.norm(xi, axis=1)
    shat = plan.eval_kernel("chihat_n", plan.r_c * mag) / mag ** 2   # kernels.hpp:167-171
    ph = s.pos @ xi.T                                                 # (N, modes)
    rho = (s.q[:, None] * np.exp(-1j * ph)).sum(axis=0)
    uref = ((shat / V) * (rho[None, :] * np.exp(1j * ph))).real.sum(axis=1)
    rel = np.sqrt(np.sum((f.u - uref) ** 2) / np.sum(uref ** 2))
    assert rel <= 1.5 * plan.stats.E_A


def test_ad_forces_are_negative_energy_gradient(esp, gpu):
    box = (10.0, 10.0, 10.0)
    plan = esp.build_plan(box, "pswf", 1e-5, 1.0, esp.Overrides(force_method="ad"),
                          device=gpu)
    s = _random(esp, 16, box, 3)
    ef = esp.evaluate(plan, s)
    fscale = np.abs(ef.F).max()
    step = 1e-5 * box[0]
    for d in range(3):
        plus, minus = s.pos.copy(), s.pos.copy()
        plus[0, d] += step
        minus[0, d] -= step
        ep = esp.evaluate(plan, esp.ParticleSystem(box, s.q, plus)).energy
        em = esp.evaluate(plan, esp.ParticleSystem(box, s.q, minus)).energy
        fd = -(ep - em) / (2.0 * step)
        assert abs(fd - ef.F[0, d]) <= 1e-4 * fscale


def test_negative_control_halved_grid_fails(esp, gpu):
    """The selected grid passes Delta <= eps against direct Ewald; half of it
    (an explicit override) fails -- the check has teeth."""
    box = (16.0, 16.0, 16.0)
    s = _random(esp, 512, box, 1)
    d = esp.direct_ewald(s, 1e-9, device=gpu)
    good = esp.build_plan(box, "pswf", 1e-4, 2.0, device=gpu)
    dg = rel_rms(esp.evaluate(good, s).F, d.F)
    bad = esp.build_plan(box, "pswf", 1e-4, 2.0,
                         esp.Overrides(nf=good.nf[0] // 2, allow_degraded=True), device=gpu)
    db = rel_rms(esp.evaluate(bad, s).F, d.F)
    assert dg <= 1e-4 < db


def test_large_lattice_family_comparison(esp, gpu):
    """52,728-site water-like lattice (the reference generator), r_c 6.2, eps
    1e-4: the Gaussian baseline needs >= 3x the PSWF grid modes and its FFT
    stage is slower."""
    from paper_2505_09727_b200 import family as FB
    from paper_2505_09727_b200 import systems as S
    box = (80.6, 80.6, 80.6)
    pos, q = S.generate_system("water-like", 3 * 26 ** 3, box, 1)
    rep = FB.bench(esp.ParticleSystem(box, q, pos), 1e-4, 6.2, reps=3, device=gpu)
    assert rep.baseline.modes / rep.primary.modes >= 3.0
    fft = lambda fb: fb.stages["fft"].mean + fb.stages["scale"].mean + fb.stages["ifft"].mean  # noqa: E731
    assert fft(rep.primary) < fft(rep.baseline)
