"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference solver compiled as oracle/_ref/libesp_ref.so
(oracle/Makefile) on seeded inputs and stores its outputs.  Needs
/root/reference (this container) -- the fixtures are committed so the GPU
box, where /root/reference does not exist, can check against them.

    make -C oracle && python tests/golden/make_golden.py

Fixtures (all float64, .npz):
  plans.json            plan parameters (nf, base_nf, P, c, c1, E_A, E_T, h)
                        for the BASELINE configs and the reference's own
                        test rows (test_ewald.cpp:26-68)
  cfg1.npz              cfg1 (N=1000 random ions, L=10, r_c=1, eps=1e-4,
                        seed 1): evaluate / local_sum / spectral_sum / self,
                        direct_ewald(1e-9), per-stage reference timings
  small_*.npz           small systems from the reference tests
  cfg2_sub.npz          cfg2 evaluate: energy + every 16th atom's u, F
  grid_cfg1.npz         spread grid of cfg1 and interpolation of a seeded
                        random grid (adjointness fixture)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402  (pure numpy module)


def plan_dict(p: ref.RefPlan) -> dict:
    return dict(nf=list(p.nf), base_nf=list(p.base_nf), P=p.P, shape=p.shape, c1=p.c1,
                E_A=p.E_A, E_T=p.E_T, E_SI=p.E_SI, h=list(p.h), demand=list(p.demand),
                chi0=p.chi0)


def main():
    ref.set_threads(os.cpu_count() or 1)
    plans = {}
    for name, c in S.CONFIGS.items():
        box = (c.L,) * 3
        p = ref.RefPlan(box, "pswf", c.eps, c.r_c)
        plans[name] = dict(box=list(box), eps=c.eps, r_c=c.r_c, **plan_dict(p))
    rows = {"row_1e-3": 1e-3, "row_5e-4": 5e-4, "row_1e-4": 1e-4, "row_5e-5": 5e-5,
            "row_1e-5": 1e-5}
    for k, eps in rows.items():
        p = ref.RefPlan((10.0, 10.0, 10.0), "pswf", eps, 1.0)
        plans[k] = dict(box=[10.0] * 3, eps=eps, r_c=1.0, **plan_dict(p))
    p = ref.RefPlan((10.0, 10.0, 15.0), "pswf", 1e-4, 1.0)
    plans["box_10_10_15"] = dict(box=[10.0, 10.0, 15.0], eps=1e-4, r_c=1.0, **plan_dict(p))
    for eps in (1e-3, 1e-4):
        p = ref.RefPlan((10.0, 10.0, 10.0), "gaussian", eps, 1.0)
        plans[f"gauss_{eps:g}"] = dict(box=[10.0] * 3, eps=eps, r_c=1.0, family="gaussian",
                                       **plan_dict(p))
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f, indent=1, sort_keys=True)

    # cfg1 full outputs
    c = S.CONFIGS["cfg1"]
    pos, q, box = c.system()
    p = ref.RefPlan(box, "pswf", c.eps, c.r_c)
    r = p.evaluate(pos, q)
    ul, Fl = p.local_sum(pos, q)
    us, Fs = p.spectral_sum(pos, q)
    t = time.time()
    d = ref.direct_ewald(pos, q, box, 1e-9)
    print("direct_ewald cfg1", time.time() - t, "s")
    pad = ref.RefPlan(box, "pswf", c.eps, c.r_c, force_method="ad")
    rad = pad.evaluate(pos, q)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), energy=r.energy, u=r.u, F=r.F,
                        u_local=ul, F_local=Fl, u_spec=us, F_spec=Fs,
                        self=p.self_correction(q), d_energy=d.energy, d_u=d.u, d_F=d.F,
                        ad_energy=rad.energy, ad_u=rad.u, ad_F=rad.F)

    # small systems from the reference tests
    smalls = {
        # test_ewald.cpp:478-491 (both families certify, N=16, L=2 cbrt 16, r_c=L/8)
        "small_n16": dict(N=16, L=2.0 * 16 ** (1 / 3), seed=101, eps=1e-3, rc_frac=1 / 8),
        # acceptance.cpp:107-126 sweep points
        "small_n128": dict(N=128, L=2.0 * 128 ** (1 / 3), seed=128, eps=1e-4, rc_frac=1 / 8),
        "small_n512": dict(N=512, L=2.0 * 512 ** (1 / 3), seed=512, eps=1e-5, rc_frac=1 / 8),
        # test_ewald.cpp:229-274 (cell list vs all pairs): N=64, L=10, seed 17
        "small_n64_rc1": dict(N=64, L=10.0, seed=17, eps=1e-3, rc=1.0),
        "small_n64_rc34": dict(N=64, L=10.0, seed=17, eps=1e-3, rc=3.4),
    }
    for name, sp in smalls.items():
        L = sp["L"]
        box = (L, L, L)
        rc = sp.get("rc", L * sp.get("rc_frac", 0.125))
        pos, q = S.generate_system("random", sp["N"], box, sp["seed"])
        p = ref.RefPlan(box, "pswf", sp["eps"], rc)
        r = p.evaluate(pos, q)
        ul, Fl = p.local_sum(pos, q)
        d = ref.direct_ewald(pos, q, box, 1e-9)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), N=sp["N"], L=L, seed=sp["seed"],
                            eps=sp["eps"], r_c=rc, energy=r.energy, u=r.u, F=r.F,
                            u_local=ul, F_local=Fl, d_energy=d.energy, d_F=d.F, d_u=d.u)

    # rock-salt Madelung (test_ewald.cpp:493-508)
    pos, q = S.generate_system("rocksalt", 8, (2.0, 2.0, 2.0), 1)
    p = ref.RefPlan((2.0, 2.0, 2.0), "pswf", 1e-5, 0.5)
    r = p.evaluate(pos, q)
    np.savez_compressed(os.path.join(HERE, "small_rocksalt.npz"), energy=r.energy, u=r.u, F=r.F)

    # grid fixtures on cfg1's plan
    c = S.CONFIGS["cfg1"]
    pos, q, box = c.system()
    p = ref.RefPlan(box, "pswf", c.eps, c.r_c)
    g = p.spread(pos[:200], q[:200])
    rng = np.random.default_rng(8)
    field = rng.uniform(-1.0, 1.0, p.nf)
    ui = p.interpolate(pos[:200], field)
    gi = p.interpolate_gradient(pos[:200], field)
    # the field is regenerated from its seed (numpy PCG64) by the tests
    np.savez_compressed(os.path.join(HERE, "grid_cfg1.npz"), spread=g, interp=ui,
                        interp_grad=gi)

    # cfg2 subsample
    c = S.CONFIGS["cfg2"]
    pos, q, box = c.system()
    p = ref.RefPlan(box, "pswf", c.eps, c.r_c)
    t = time.time()
    r = p.evaluate(pos, q)
    print("cfg2 reference evaluate", time.time() - t, "s", r.timings)
    idx = np.arange(0, q.size, 16)
    np.savez_compressed(os.path.join(HERE, "cfg2_sub.npz"), energy=r.energy, idx=idx,
                        u=r.u[idx], F=r.F[idx], Fnorm2=float(np.sum(r.F ** 2)),
                        unorm2=float(np.sum(r.u ** 2)))
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
