"""Family comparison: the PSWF split against the Gaussian/B-spline baseline
at the same tolerance (reference `cli.hpp:203-346`: FamilyBench, BenchReport,
detail::bench_family, cmd_bench -- without its file output).

Both plans run through the same GPU path (`evaluate`); the report carries the
per-family plan parameters, per-stage timing statistics over `reps`
evaluations, the energy, the force error Delta against direct Ewald (when
computed), and the grid ratios R_demand (continuous demand) and R_built
(built n_f after rounding and inflation), baseline over primary
(`cli.hpp:313-318`).

The reference computes Delta only for N <= 1024 (`kBenchOracleMaxN`,
`cli.hpp:47, 306`), its direct Ewald being O(N^2) on the CPU; the GPU
direct Ewald here also takes a target subset, so `delta_targets` extends the
check to any N (Delta over the subset's forces).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (EwaldPlan, Overrides, ParticleSystem, build_plan, direct_ewald, evaluate,
               InvalidArgument)

BENCH_ORACLE_MAX_N = 1024  # cli.hpp:47


@dataclass
class StageStats:
    mean: float = 0.0
    min: float = 0.0


@dataclass
class FamilyBench:
    """cli.hpp:203-216."""
    family: str
    P: int
    shape: float
    c1: float
    demand: tuple
    base_nf: tuple
    nf: tuple
    modes: int
    E_A: float
    E_T: float
    E_SI: float
    delta: float = float("nan")
    stages: dict = field(default_factory=dict)
    total: StageStats = field(default_factory=StageStats)
    energy: float = 0.0


@dataclass
class BenchReport:
    """cli.hpp:218-227."""
    N: int
    box: tuple
    eps: float
    r_c: float
    reps: int
    primary: FamilyBench
    baseline: FamilyBench
    R_demand: float
    R_built: float
    delta_computed: bool


def relative_force_error(F, Fref) -> float:
    """reference.hpp:241-255: sqrt(sum |F - Fref|^2 / sum |Fref|^2)."""
    F = np.asarray(F, dtype=np.float64).ravel()
    R = np.asarray(Fref, dtype=np.float64).ravel()
    den = float(np.sum(R * R))
    num = float(np.sum((F - R) ** 2))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(np.sqrt(num / den))


def bench_family(plan: EwaldPlan, system: ParticleSystem, reps: int, refF=None,
                 targets=None) -> FamilyBench:
    """detail::bench_family (cli.hpp:231-262): `reps` evaluations, per-stage
    mean/min of the reference's timing keys, total = their sum; the energy and
    Delta (against refF, over `targets` if given) from the first one."""
    fb = FamilyBench(plan.family, plan.P, plan.shape, plan.c1, plan.demand, plan.base_nf,
                     plan.nf, plan.total_modes(), plan.stats.E_A, plan.stats.E_T,
                     plan.stats.E_SI)
    for r in range(reps):
        ef = evaluate(plan, system)
        total = 0.0
        for k, v in ef.timings.items():
            if k == "total":  # the call's wall time, not a stage
                continue
            st = fb.stages.setdefault(k, StageStats())
            st.mean += v
            st.min = v if r == 0 else min(st.min, v)
            total += v
        fb.total.mean += total
        fb.total.min = total if r == 0 else min(fb.total.min, total)
        if r == 0:
            fb.energy = ef.energy
            if refF is not None:
                F = ef.F if targets is None else ef.F[np.asarray(targets)]
                fb.delta = relative_force_error(F, refF)
    for st in fb.stages.values():
        st.mean /= reps
    fb.total.mean /= reps
    return fb


def bench(system: ParticleSystem, eps: float, r_c: float, family: str = "pswf",
          baseline_family: str = "gaussian", reps: int = 3,
          overrides: Overrides | None = None, tol: float = 1e-9, delta_targets=None,
          device: int = 0) -> BenchReport:
    """cmd_bench (cli.hpp:288-346) on an in-memory system.  The baseline plan
    runs its family's defaults with the primary's force method
    (cli.hpp:301-303).  Delta is computed against direct Ewald (tolerance
    `tol`) for N <= 1024 as in the reference, or over `delta_targets`."""
    if reps < 1:
        raise InvalidArgument("cmd_bench: reps must be >= 1")
    ov = overrides or Overrides()
    prim = build_plan(system.box, family, eps, r_c, ov, device=device)
    base = build_plan(system.box, baseline_family, eps, r_c,
                      Overrides(force_method=ov.force_method), device=device)
    N = system.size()
    refF = None
    if delta_targets is not None:
        refF = direct_ewald(system, tol, targets=delta_targets, device=device).F
    elif N <= BENCH_ORACLE_MAX_N:
        refF = direct_ewald(system, tol, device=device).F
    rp = bench_family(prim, system, reps, refF, delta_targets)
    rb = bench_family(base, system, reps, refF, delta_targets)
    R_demand = 1.0
    R_built = 1.0
    for d in range(3):
        R_demand *= base.demand[d] / prim.demand[d]
        R_built *= float(base.nf[d]) / prim.nf[d]
    return BenchReport(N, tuple(system.box), eps, r_c, reps, rp, rb, R_demand, R_built,
                       refF is not None)
