"""Generate the large-config golden fixtures from the REFERENCE itself.

Runs the unmodified reference `esp::evaluate` (ewald.hpp:619-649, ik forces,
PSWF split) compiled as oracle/_ref/libesp_ref.so (oracle/Makefile) on the
BASELINE cfg3, cfg4 and cfg5 systems (seeded generators, paper_2505_09727_b200
.systems) and stores a strided subsample of its outputs plus whole-system
norms, so the GPU box -- where neither /root/reference nor the compiled
reference exists -- can check the CUDA path at full size.  Also stores two
Gaussian-family evaluations (kernels.hpp:105-138 split, kernels.hpp:263-273
B-spline window) so that family is pinned to the reference too.

    make -C oracle && python tests/golden/make_golden_large.py [cfg3 cfg4 cfg5 gauss]

Fixtures (float64 .npz):
  cfg3_sub.npz  energy, idx = every 16th atom, u[idx], F[idx], sum F^2, sum u^2
  cfg4_sub.npz  same, every 64th atom
  cfg5_sub.npz  same, every 256th atom
  gauss_cfg1.npz  cfg1 system, Gaussian family: energy, u, F (all atoms)
  gauss_cfg2_sub.npz  cfg2 system, Gaussian family: energy, every 16th atom
Each file also holds the reference's per-stage wall times and thread count
(informational only).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2505_09727_b200 import systems as S  # noqa: E402  (pure numpy module)

STRIDE = {"cfg3": 16, "cfg4": 64, "cfg5": 256}


def _store(name, r, stride, t, extra=None):
    idx = np.arange(0, r.u.size, stride)
    stages = np.array([r.timings.get(k, 0.0) for k in
                       ("local", "spread", "fft", "scale", "ifft", "interpolate")])
    np.savez_compressed(os.path.join(HERE, name), energy=r.energy, idx=idx, u=r.u[idx],
                        F=r.F[idx], Fnorm2=float(np.sum(r.F ** 2)),
                        unorm2=float(np.sum(r.u ** 2)), Fsum=np.sum(r.F, axis=0),
                        ref_seconds=t, ref_stage_s=stages, ref_threads=ref.get_threads(),
                        **(extra or {}))


def run_cfg(name):
    c = S.CONFIGS[name]
    pos, q, box = c.system()
    p = ref.RefPlan(box, "pswf", c.eps, c.r_c)
    t = time.time()
    r = p.evaluate(pos, q)
    t = time.time() - t
    print(f"{name}: reference evaluate N={q.size} {t:.1f} s  E={r.energy!r}", r.timings,
          flush=True)
    _store(f"{name}_sub.npz", r, STRIDE[name], t)


def run_gauss():
    for name, stride in (("cfg1", 1), ("cfg2", 16)):
        c = S.CONFIGS[name]
        pos, q, box = c.system()
        p = ref.RefPlan(box, "gaussian", c.eps, c.r_c)
        t = time.time()
        r = p.evaluate(pos, q)
        t = time.time() - t
        print(f"gauss {name}: nf={p.nf} P={p.P} {t:.1f} s E={r.energy!r}", flush=True)
        out = "gauss_cfg1.npz" if name == "cfg1" else "gauss_cfg2_sub.npz"
        _store(out, r, stride, t, dict(nf=np.array(p.nf), P=p.P))


def main(argv):
    ref.set_threads(os.cpu_count() or 1)
    which = argv or ["gauss", "cfg3", "cfg4", "cfg5"]
    for w in which:
        if w == "gauss":
            run_gauss()
        else:
            run_cfg(w)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main(sys.argv[1:])
