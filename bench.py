#!/usr/bin/env python
"""ESP force-evaluation benchmark (BASELINE.json metric: atoms*evals/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5]
    python bench.py --impl reference ...      # the reference CPU arm

Workload: cfg5 by default -- BASELINE configs[4], the 8,000,001-atom water box
the metric is quoted on at 1/2/4/8 B200 (it fits one GPU).  One step = one
full ESP evaluation (real-space pair sum + spread + FFT + influence/ik
multiply + 4 inverse FFTs + interpolation + energy) with positions/charges
already resident in HBM (`value`).  `e2e` is the same metric through the
public API on pinned HOST buffers (H2D of positions+charges and D2H of
potentials, forces and energy inside the timed region).

--gpus N > 1: bench.py launches itself under torch.distributed.run when
WORLD_SIZE is unset (one rank per GPU, NCCL).  The default decomposition for
cfg3/cfg4/cfg5 is ONE system sharded over the ranks (distributed FFT with
local atoms + ghosts, strong scaling, value = N_atoms / max-over-ranks step
time); cfg1/cfg2 (too small to shard) run replicas (weak scaling).

Timing: W >= 3 warm-up steps; then K steps, each preceded by a 256 MiB L2
flush (outside the event pair) and bracketed by CUDA events on the stream
the kernels run on; barrier + synchronize around the timed loop; the max
over ranks is reported.  nvidia-smi clocks are sampled while it runs.

The reference arm (--impl reference) runs the compiled, unmodified reference
(oracle/_ref/libesp_ref.so) on all host cores; it never loads this repo's
CUDA library (systems.py is loaded by file path, not through the package).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ESP force evals: atoms*evals/s"
UNIT = "atoms*evals/s"
FLOPS_PER_UNORDERED_PAIR = 96


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--force-method", default="ik", choices=["ik", "ad"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="budget of the cpu_baseline sample (rank 0, N=1; at least one "
                         "full evaluate)")
    ap.add_argument("--ref-seconds", type=float, default=240.0,
                    help="--impl reference: timed-step budget (at least one step, at most "
                         "--steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--decomp", choices=["auto", "replicas", "slab", "pencil", "pencil-local",
                                         "shard"],
                    default="auto",
                    help="N>1: replicas = one independent system per rank (weak scaling); "
                         "slab = ONE system, x-slabs, NCCL all-reduce of the charge grid and "
                         "outputs; pencil = ONE system with the grid/spectrum/fields split too "
                         "(halo exchanges + all-to-all transposes); pencil-local = the same "
                         "with every rank holding only its own atoms (ghost exchange, energy "
                         "all-reduce); shard = the same decomposition behind the C ABI "
                         "(esp_shard_evaluate: NCCL inside the library, no host "
                         "synchronisation); auto = shard for cfg3/4/5, replicas for cfg1/2")
    ap.add_argument("--strong", action="store_true", help="alias of --decomp slab")
    args = ap.parse_args()
    if args.strong:
        args.decomp = "slab"
    if args.decomp == "auto":
        args.decomp = "shard" if args.workload in ("cfg3", "cfg4", "cfg5") else "replicas"
    args.warmup = max(args.warmup, 3)
    return args


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def load_systems():
    """paper_2505_09727_b200/systems.py loaded by file path: pure numpy, and
    importing it this way does not run the package __init__ (which dlopens
    libesp_b200.so) -- the reference arm must not load the repo's library."""
    import importlib.util
    name = "_esp_bench_systems"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(
        name, os.path.join(ROOT, "paper_2505_09727_b200", "systems.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def parallelism(decomp: str, world: int) -> str:
    if world <= 1:
        return "single GPU"
    return {"slab": f"x-slabs x{world} (NCCL all-reduce of grid + outputs)",
            "pencil": f"distributed FFT x{world} (NCCL halo send/recv + all-to-all transposes)",
            "pencil-local": f"distributed FFT x{world}, local atoms + ghosts (NCCL ghost/halo "
                            "send/recv, all-to-all transposes, energy all-reduce)",
            "shard": f"sharded x{world} behind the C ABI (esp_shard_evaluate: x-slabs by grid "
                     "plane, local atoms + ghosts, NCCL send/recv halos and all-to-all "
                     "transposes inside the library, energy all-reduce)",
            }.get(decomp, f"replicas x{world}")


def bench_config(c, N, box, nf, P, force_method, decomp, world) -> dict:
    """The `config` dict, identical in both arms (same workload, same keys)."""
    return {"workload": c.name, "N": int(N), "box_L": box[0], "r_c": c.r_c, "eps": c.eps,
            "nf": [int(v) for v in nf], "P": int(P), "force_method": force_method,
            "parallelism": parallelism(decomp, world),
            "l2": "GPU arm: 256 MiB flush write before every timed step (outside the events); "
                  "inputs (32 B/atom) also exceed L2 at cfg3-5"}


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: relaunch this script under
    torch.distributed.run (one rank per GPU, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons while the GPU is busy."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join("/tmp", f"esp_bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def nsamples(self) -> int:
        try:
            with open(self.path) as f:
                return sum(1 for ln in f if ln.strip())
        except Exception:
            return 0

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for ln in f:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _ref_lib():
    """oracle/ref.py (ctypes binding of oracle/_ref/libesp_ref.so)."""
    from oracle import ref
    return ref


def cpu_reference_rate(c, pos, q, box, budget_s: float):
    """cpu_baseline: the compiled reference (oracle/_ref) on the host cores,
    a bounded sample -- evaluate() calls of the full workload until about
    budget_s of CPU time has been spent (at least one; no warm-up call when
    one evaluation alone exceeds the budget)."""
    ref = _ref_lib()
    if not ref.available():
        return None
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    plan = ref.RefPlan(box, "pswf", c.eps, c.r_c)
    t0 = time.perf_counter()
    r = plan.evaluate(pos, q)
    first = time.perf_counter() - t0
    times, stages = [], []
    warm = first < 0.5 * budget_s
    if not warm:
        times.append(first)
        stages.append(r.timings)
    t_end = time.perf_counter() + budget_s
    while not times or (time.perf_counter() + statistics.mean(times) < t_end and len(times) < 50):
        t0 = time.perf_counter()
        r = plan.evaluate(pos, q)
        times.append(time.perf_counter() - t0)
        stages.append(r.timings)
    mean = statistics.mean(times)
    st = {k: statistics.mean(s[k] for s in stages) for k in stages[0]}
    return {"value": q.size / mean, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{c.name}: full system, {len(times)} evaluate() call(s)"
                      f"{' after 1 warm-up' if warm else ' (no warm-up)'}, "
                      f"esp::thread_count()={cores}; FFT stage uses the oracle's FFTW3 shim",
            "s_per_eval": mean, "stage_s": st, "energy": r.energy}


def run_reference(args):
    """--impl reference: the compiled, unmodified reference evaluate()
    (ewald.hpp:619-649 via oracle/_ref) on all host cores, same workload and
    config as the GPU arm.  Under torchrun only rank 0 runs.  Each step is one
    full evaluate(); one untimed warm-up (a CPU code has no JIT/caches to
    warm beyond first touch), then timed steps until --steps or the
    --ref-seconds budget is reached (at least one) -- a cfg5 evaluate takes
    ~40 s on 16 host threads."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    S = load_systems()
    ref = _ref_lib()
    c = S.config(args.workload)
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libesp_ref.so not built"}))
        return 0
    pos, q, box = c.system()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    plan = ref.RefPlan(box, "pswf", c.eps, c.r_c)
    cfg = bench_config(c, q.size, box, plan.nf, plan.P, "ik", args.decomp, world)
    t0 = time.perf_counter()
    plan.evaluate(pos, q)
    t_warm = time.perf_counter() - t0
    times = []
    t_end = time.perf_counter() + args.ref_seconds
    while len(times) < args.steps and (not times or time.perf_counter() + t_warm < t_end):
        t0 = time.perf_counter()
        plan.evaluate(pos, q)
        times.append(time.perf_counter() - t0)
    s = statistics.mean(times)
    value = q.size / s
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "steps_requested": args.steps, "warmup": 1,
        "warmup_requested": args.warmup, "ms_per_step": s * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if (world > 1 and args.decomp != "replicas") else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, SURVEY.md 8(d); water-like boxes by "
                "paper_2505_09727_b200/systems.py water_box)",
        "config": cfg,
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{c.name}: one full evaluate() per step on all "
                                   f"{cores} host threads (oracle/_ref, unmodified headers + "
                                   f"FFTW3 shim); {len(times)} timed step(s) after 1 warm-up "
                                   f"(budget {args.ref_seconds:g} s)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    rank, world, local = dist_env()
    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2505_09727_b200 as E
    S = load_systems()

    from paper_2505_09727_b200.dist import max_over_ranks, replica_seed, weak_scaling_value
    base = S.config(args.workload)
    decomp = args.decomp if world > 1 else "replicas"
    strong = decomp != "replicas"
    c = S.Config(base.name, base.kind, base.N, base.L, base.r_c, base.eps,
                 seed=base.seed if strong else replica_seed(base.seed, rank))
    pos, q, box = c.system()
    N = int(q.size)
    plan = E.build_plan(box, "pswf", c.eps, c.r_c, E.Overrides(force_method=args.force_method),
                        device=local)
    dev = torch.device("cuda", local)
    pos_d = torch.from_numpy(pos).to(dev)
    q_d = torch.from_numpy(q).to(dev)
    u_d = torch.empty(N, dtype=torch.float64, device=dev)
    F_d = torch.empty(N * 3, dtype=torch.float64, device=dev)
    e_d = torch.empty(1, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    if decomp == "slab":
        from paper_2505_09727_b200.dist import evaluate_slab
        out_d = torch.empty(4 * N + 1, dtype=torch.float64, device=dev)
        grid_d = torch.empty(E.grid_size(plan), dtype=torch.float64, device=dev)

        def step():
            evaluate_slab(plan, box, N, pos_d, q_d, out_d, grid_d, rank, world,
                          stream.cuda_stream)
    elif decomp == "pencil":
        from paper_2505_09727_b200.dist import PencilBuffers, PencilLayout, evaluate_pencil
        layout = PencilLayout.of(plan, world)
        pbufs = PencilBuffers(layout, rank, N, dev)
        out_d = pbufs.out

        def step():
            evaluate_pencil(plan, box, N, pos_d, q_d, pbufs, layout, rank, stream.cuda_stream)
    elif decomp == "pencil-local":
        from paper_2505_09727_b200.dist import (PencilLayout, atom_owner, evaluate_pencil_local,
                                                fold_positions)
        layout = PencilLayout.of(plan, world)
        own_idx = np.nonzero(atom_owner(layout, fold_positions(pos, box)[:, 0]) == rank)[0]
        pos_d = torch.from_numpy(np.ascontiguousarray(pos[own_idx])).to(dev)
        q_d = torch.from_numpy(q[own_idx]).to(dev)
        res = {}

        def step():
            res["u"], res["F"], res["e"] = evaluate_pencil_local(
                plan, box, pos_d, q_d, layout, rank, c.r_c, stream.cuda_stream, cache=res)
    elif decomp == "shard":
        # each rank passes only its own atoms; the exchanges run inside the
        # library on a NCCL communicator made from a broadcast unique id
        own_idx = np.nonzero(E.shard_owner(plan, world, pos) == rank)[0]
        counts = [None] * world
        dist.all_gather_object(counts, int(own_idx.size))
        uid = [E.shard_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        shard = E.Shard(plan, rank, world, max(counts), nccl_id=uid[0])
        pos_d = torch.from_numpy(np.ascontiguousarray(pos[own_idx])).to(dev)
        q_d = torch.from_numpy(q[own_idx]).to(dev)
        res = {"u": torch.empty(own_idx.size, dtype=torch.float64, device=dev),
               "F": torch.empty((own_idx.size, 3), dtype=torch.float64, device=dev),
               "e": torch.empty(1, dtype=torch.float64, device=dev)}

        def step():
            shard.evaluate(box, own_idx.size, pos_d.data_ptr(), q_d.data_ptr(),
                           res["u"].data_ptr(), res["F"].data_ptr(), res["e"].data_ptr(),
                           stream.cuda_stream)
    else:
        def step():
            E.evaluate_device(plan, box, N, pos_d.data_ptr(), q_d.data_ptr(), u_d.data_ptr(),
                              F_d.data_ptr(), e_d.data_ptr(), stream.cuda_stream)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = plan.last_launch_count()

    # ---- timed region (device-resident inputs)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        ev0[k].record(stream)
        step()
        ev1[k].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    if decomp == "shard":
        shard.check()
    energy = (float(res["e"].item()) if decomp in ("pencil-local", "shard") else
              float(out_d[4 * N].item()) if strong else float(e_d.item()))

    # keep the GPU busy (untimed) until the clock sampler has a few samples
    t_end = time.time() + 3.0
    while clocks.nsamples() < 8 and time.time() < t_end:
        for _ in range(5):
            step()
        torch.cuda.synchronize()
    clk = clocks.stop()

    # ---- per-stage breakdown and the dominant kernel's roofline
    # (whole system on this GPU; a separate plan for the sharded modes, whose
    # shard keeps using its own plan's engine buffers afterwards)
    tplan = plan if not strong else E.build_plan(
        box, "pswf", c.eps, c.r_c, E.Overrides(force_method=args.force_method), device=local)
    tim = []
    for _ in range(5):
        ef = E.evaluate(tplan, E.ParticleSystem(box, q, pos), timings=True)
        tim.append(ef.timings)
    stages_ms = {k: statistics.median(t[k] for t in tim) * 1e3 for k in tim[0] if k != "total"}
    ordered_pairs = tplan.last_pair_count()
    pair_flops = FLOPS_PER_UNORDERED_PAIR * ordered_pairs / 2.0
    t_pair = stages_ms["local"] * 1e-3
    peak64 = E.fp64_peak_tflops(local)
    achieved = pair_flops / t_pair / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "pair_kernel_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tr = json.load(f)
            traffic = tr.get(args.workload)
        except Exception:
            traffic = None
    kname = ("k_pair_half (K4 real-space pair sum, half-shell: each unordered pair once)"
             if N >= 4096 else "k_pair (K4 real-space pair sum, full lists)")
    roofline = {"bound": "fp64", "kernel": kname,
                "achieved": achieved, "peak": peak64, "unit": "TFLOP/s",
                "frac": achieved / peak64 if peak64 > 0 else None, "traffic": traffic,
                "peak_source": "fp64 DFMA microbenchmark measured in this run "
                               "(MEASURED_PEAKS.json has no fp64 entry)",
                "work": f"{FLOPS_PER_UNORDERED_PAIR} flops x {ordered_pairs // 2} unordered "
                        "in-range pairs (counted on device)",
                "kernel_ms": stages_ms["local"],
                "limiter": "instruction issue (profiles/r02j_full_cfg5.md, r02i_k4_lines_cfg5.md; "
                           "cfg5: issue 65-70 % active, fp64 pipe 35 %): ~250 warp instructions per "
                           "32 pairs, 63 of them fp64 pair terms.  On the B200 a warp DFMA holds "
                           "the issue port ~1.4 cycles and any other instruction ~1.2 "
                           "(tools/micro/fp64_issue.cu), so the rounds loop (63 fp64 + ~50 other "
                           "instructions per round) and the neighbour search (~130 per 32 pairs) "
                           "are both issue-bound; DESIGN.md 4 lists what was removed and what is "
                           "left"}

    # ---- every grid-pipeline kernel against the HBM roofline (SURVEY 8(d)
    # algorithmic bytes; serialised stage times).  The grids fit in L2 (cfg5:
    # 47 MB of 126 MB), so these kernels are L1/L2-bound and their HBM
    # fractions are low by construction; the bytes are the algorithmic minimum.
    hbm_peak, hbm_src = None, None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        hbm_peak, hbm_src = 7700.0, "nominal HBM3e (MEASURED_PEAKS.json absent)"
    M = int(np.prod(plan.nf))
    Mh = int(plan.nf[0] * plan.nf[1] * (plan.nf[2] // 2 + 1))
    nfld = 4 if args.force_method == "ik" else 1
    k1name = "K1 k_spread_warp" if plan.spread_kernel == "warp" else "K1 k_spread"
    if plan.fused_xpass:
        # 2-D cuFFT planes + K2 fused into the x pass (read b and p, write the
        # nfld half-transformed fields); the inverse planes write planar fields
        kbytes = {
            k1name: (32 * N + 8 * M, "spread"),
            "K2+x-DFTs k_xpass (fused)": ((24 + 16 * nfld) * Mh, "scale"),
            "K3 k_interp": (8 * nfld * M + 64 * N, "interpolate"),
            "cuFFT D2Z 2-D planes": (8 * M + 16 * Mh, "fft"),
            # (the tiled K3, N >= 2^19, reads the planar fields; smaller
            # systems add an interleaving pass, 16 B per field and node)
            f"cuFFT Z2D 2-D planes, {nfld} field(s) in one batch":
                (nfld * (16 * Mh + 8 * M) + (16 * nfld * M if nfld == 4 and N < (1 << 19) else 0),
                 "ifft"),
        }
    else:
        kbytes = {
            k1name: (32 * N + 8 * M, "spread"),
            "K2 k_scale": ((24 + 16 * nfld) * Mh, "scale"),
            "K3 k_interp": (8 * nfld * M + 64 * N, "interpolate"),
            "cuFFT D2Z": (8 * M + 16 * Mh, "fft"),
            f"cuFFT Z2D x{nfld}": (nfld * (16 * Mh + 8 * M), "ifft"),
        }
    kernels = {}
    for name, (nbytes, stage) in kbytes.items():
        kms = stages_ms.get(stage)
        if not kms:
            continue
        gbs = nbytes / (kms * 1e-3) / 1e9
        kernels[name] = {"bound": "hbm", "bytes": nbytes, "ms": kms, "GB/s": gbs,
                         "frac": gbs / hbm_peak}
    kernels["K4 " + roofline["kernel"].split(" ")[0]] = {
        "bound": "fp64", "flops": pair_flops, "ms": stages_ms["local"],
        "TFLOP/s": achieved, "frac": roofline["frac"]}
    # K1 and K3 move their footprint nodes through shared memory (K1: the
    # tile read-modify-write, 16 B per node; tiled K3: 32 B per node read),
    # so their bound is the SM-wide shared-memory bandwidth: 128 B per clock
    # per SM at the SM clock sampled during the run
    try:
        import torch as _t
        n_sm = _t.cuda.get_device_properties(local).multi_processor_count
    except Exception:
        n_sm = 148
    sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
    smem_peak = n_sm * 128.0 * sm_mhz * 1e6 / 1e9  # GB/s
    P3 = int(plan.P) ** 3
    for name, (nbytes, stage) in {k1name + " (shared-memory tile RMW)": (16 * P3 * N, "spread"),
                                  "K3 (footprint node reads)": (32 * P3 * N, "interpolate")}.items():
        kms = stages_ms.get(stage)
        if kms:
            gbs = nbytes / (kms * 1e-3) / 1e9
            kernels[name] = {"bound": "smem", "bytes": nbytes, "ms": kms, "GB/s": gbs,
                             "frac": gbs / smem_peak}
    kernel_rooflines = {"hbm_peak_GBps": hbm_peak, "hbm_peak_source": hbm_src,
                        "smem_peak_GBps": smem_peak,
                        "smem_peak_source": f"{n_sm} SMs x 128 B/clock x {sm_mhz:g} MHz (sampled)",
                        "kernels": kernels}

    # ---- e2e through the public API on pinned host buffers
    pos_h = torch.from_numpy(pos).pin_memory().numpy()
    q_h = torch.from_numpy(q).pin_memory().numpy()
    u_h = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
    F_h = torch.empty((N, 3), dtype=torch.float64).pin_memory().numpy()
    sysh = E.ParticleSystem(box, q_h, pos_h)
    if decomp in ("pencil-local", "shard"):
        pos_ht = torch.from_numpy(np.ascontiguousarray(pos[own_idx])).pin_memory()
        q_ht = torch.from_numpy(q[own_idx]).pin_memory()
        uo_h = torch.empty(own_idx.size, dtype=torch.float64).pin_memory()
        Fo_h = torch.empty((own_idx.size, 3), dtype=torch.float64).pin_memory()

        def e2e_step():
            pos_d.copy_(pos_ht, non_blocking=True)
            q_d.copy_(q_ht, non_blocking=True)
            step()
            uo_h.copy_(res["u"], non_blocking=True)
            Fo_h.copy_(res["F"], non_blocking=True)
            torch.cuda.synchronize()
    elif strong:
        out_h = torch.empty(4 * N + 1, dtype=torch.float64).pin_memory()
        pos_ht = torch.from_numpy(pos_h)
        q_ht = torch.from_numpy(q_h)

        def e2e_step():
            pos_d.copy_(pos_ht, non_blocking=True)
            q_d.copy_(q_ht, non_blocking=True)
            step()
            out_h.copy_(out_d, non_blocking=True)
            torch.cuda.synchronize()
    else:
        def e2e_step():
            E.evaluate(plan, sysh, timings=False, out=(u_h, F_h))
    for _ in range(2):
        e2e_step()
    if dist:
        dist.barrier()
    t_e2e = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_step()
        t_e2e.append(time.perf_counter() - t0)
    e2e_ms = statistics.mean(t_e2e) * 1e3

    ms, e2e_ms = max_over_ranks([ms, e2e_ms], device=dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(c, pos, q, box, args.cpu_seconds)
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"error": str(exc)}

    if rank == 0:
        value = (N / (ms * 1e-3)) if strong else weak_scaling_value(N, world, ms)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md 8(d); water-like boxes by "
                    "paper_2505_09727_b200/systems.py water_box)",
            "config": bench_config(c, N, box, plan.nf, plan.P, plan.force_method, decomp,
                                   world),
            "impl": "ours",
            "energy": energy,
            "clocks": clk,
            "gpu_launches": launches_per_step * args.steps,
            "launches_per_step": launches_per_step,
            "stages_ms": stages_ms,
            "roofline": roofline,
            "kernel_rooflines": kernel_rooflines,
            "cpu_baseline": cpu,
            "e2e": {"value": (N / (e2e_ms * 1e-3)) if strong else weak_scaling_value(N, world, e2e_ms),
                    "unit": UNIT,
                    "h2d_bytes_per_step": int((own_idx.size if decomp in ("pencil-local", "shard") else N) * 32),
                    "d2h_bytes_per_step": int((own_idx.size if decomp in ("pencil-local", "shard") else N) * 32 + 8),
                    "ms_per_step": e2e_ms},
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
