"""Multi-process plumbing for the benchmark's multi-GPU mode (torch.distributed).

Round 1 runs one independent replica of the workload per rank (weak
scaling, no data-path collective): each rank evaluates its own seeded system
on its own GPU; the only collective is the max-over-ranks reduction of the
measured step times.  Backend "nccl" on the GPU box, "gloo" in the CPU tests.
"""
from __future__ import annotations

import os


def env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def replica_seed(base_seed: int, rank: int) -> int:
    """Seed of rank's replica (rank 0 evaluates the BASELINE seed itself)."""
    return int(base_seed) + int(rank)


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity if not
    initialised).  device: torch device of the tensor used for the
    all-reduce (cuda for NCCL, cpu for gloo)."""
    import torch
    import torch.distributed as dist
    vals = [float(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def weak_scaling_value(atoms_per_rank: int, world: int, ms_per_step: float) -> float:
    """Whole-job atoms*evals/s for `world` replicas timed at the max step time."""
    return atoms_per_rank * world / (ms_per_step * 1e-3)


class _Lib:
    """The real engine: the C-ABI phase entry points (device pointers)."""

    @staticmethod
    def phase_a(plan, box, N, pos, q, rank, nranks, grid, stream):
        from . import eval_phase_a
        eval_phase_a(plan, box, N, pos.data_ptr(), q.data_ptr(), rank, nranks, grid.data_ptr(),
                     stream)

    @staticmethod
    def phase_b(plan, rank, nranks, grid, u, F, e, stream):
        from . import eval_phase_b
        eval_phase_b(plan, rank, nranks, grid.data_ptr(), u.data_ptr(), F.data_ptr(),
                     e.data_ptr(), stream)


def evaluate_slab(plan, box, N, pos, q, out, grid, rank, nranks, stream=0, group=None,
                  engine=_Lib):
    """One rank's share of a slab-decomposed ESP evaluation (strong scaling).

    pos (3N), q (N): the full system on every rank (torch tensors); out: 4N+1
    doubles receiving [u | F | energy] summed over ranks; grid: nx*ny*nz
    doubles of scratch.  Two sums cross the ranks: the partial charge grids
    (after spreading) and the partial outputs -- both NCCL all-reduces over
    NVLink on the GPU box (gloo in the CPU tests).  engine is the per-rank
    compute (the C-ABI phases by default)."""
    import torch.distributed as dist
    use = dist.is_available() and dist.is_initialized() and nranks > 1
    engine.phase_a(plan, box, N, pos, q, rank, nranks, grid, stream)
    if use:
        dist.all_reduce(grid, group=group)
    engine.phase_b(plan, rank, nranks, grid, out[:N], out[N:4 * N], out[4 * N:], stream)
    if use:
        dist.all_reduce(out, group=group)
    return out
