"""Family comparison (cmd_bench, reference cli.hpp:203-346) on the GPU:
the PSWF plan against the Gaussian/B-spline baseline at cfg1's settings.
Pinned to the compiled reference: the plans (tests/golden/plans.json, cfg1
and gauss_0.0001), the energies and forces of both families
(cfg1.npz, gauss_cfg1.npz) and, through them, each family's Delta against
the reference's own direct Ewald (cfg1.npz d_F)."""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, max_rel

pytestmark = pytest.mark.gpu


def test_bench_families_cfg1(esp, gpu):
    from paper_2505_09727_b200 import family as FB
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg1")
    pos, q, box = c.system()
    rep = FB.bench(esp.ParticleSystem(box, q, pos), c.eps, c.r_c, reps=2, device=gpu)
    plans = json.load(open(os.path.join(GOLDEN, "plans.json")))
    pp, pg = plans["cfg1"], plans["gauss_0.0001"]
    assert rep.primary.family == "pswf" and rep.baseline.family == "gaussian"
    assert list(rep.primary.nf) == pp["nf"] and list(rep.baseline.nf) == pg["nf"]
    assert rep.primary.P == pp["P"] and rep.baseline.P == pg["P"]
    R_built = math.prod(pg["nf"][d] / pp["nf"][d] for d in range(3))
    R_demand = math.prod(pg["demand"][d] / pp["demand"][d] for d in range(3))
    assert rep.R_built == pytest.approx(R_built, rel=1e-15)
    assert rep.R_demand == pytest.approx(R_demand, rel=1e-10)
    # energies of both families vs the compiled reference
    gp, gg = golden("cfg1.npz"), golden("gauss_cfg1.npz")
    assert abs(rep.primary.energy - float(gp["energy"])) <= 1e-11 * abs(float(gp["energy"]))
    assert abs(rep.baseline.energy - float(gg["energy"])) <= 1e-11 * abs(float(gg["energy"]))
    # Delta vs direct Ewald (N = 1000 <= 1024: computed, as in the reference)
    assert rep.delta_computed
    ref_dp = FB.relative_force_error(gp["F"], gp["d_F"])
    idx = gg["idx"]
    ref_dg = FB.relative_force_error(gg["F"], gp["d_F"][idx])
    assert rep.primary.delta == pytest.approx(ref_dp, rel=1e-4)
    assert rep.baseline.delta == pytest.approx(ref_dg, rel=1e-4)
    assert rep.primary.delta <= c.eps and rep.baseline.delta <= c.eps
    # stage statistics under the reference's keys
    for fb in (rep.primary, rep.baseline):
        for k in ("local", "spread", "fft", "scale", "ifft", "interpolate"):
            assert k in fb.stages and 0.0 < fb.stages[k].min <= fb.stages[k].mean
        assert fb.total.min > 0.0


def test_bench_delta_targets_cfg2(esp, gpu):
    """Delta over a target subset at N > 1024 (the reference skips it there);
    both families stay within eps."""
    from paper_2505_09727_b200 import family as FB
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    tg = np.arange(0, q.size, 97)
    rep = FB.bench(esp.ParticleSystem(box, q, pos), c.eps, c.r_c, reps=1, delta_targets=tg,
                   device=gpu)
    assert rep.delta_computed
    assert 0.0 < rep.primary.delta <= c.eps and 0.0 < rep.baseline.delta <= c.eps
    assert rep.R_built > 1.0
