"""Multi-process plumbing (torch.distributed; "nccl" on the GPU box, "gloo" in
the CPU tests).

Three multi-GPU modes:
  * replicas (bench default): one independent seeded system per rank, weak
    scaling, no data-path collective;
  * evaluate_slab: one system, real-space targets and spread/interp atoms
    split into x-slabs, the charge grid all-reduced and the FFT replicated;
  * evaluate_pencil: one system with the grid, spectrum and fields split
    too (halo exchanges + two all-to-all transposes).
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
    def geometry(plan, rank, nranks):
        from . import pencil_geometry
        return pencil_geometry(plan, rank, nranks)

    @staticmethod
    def pencil_phase_a(plan, box, N, pos, q, rank, nranks, slab, stream):
        from . import pencil_phase_a
        pencil_phase_a(plan, box, N, pos.data_ptr(), q.data_ptr(), rank, nranks,
                       slab.data_ptr(), stream)

    @staticmethod
    def pencil_forward(plan, rank, nranks, slab, send, stream):
        from . import pencil_forward
        pencil_forward(plan, rank, nranks, slab.data_ptr(), send.data_ptr(), stream)

    @staticmethod
    def pencil_solve(plan, rank, nranks, recv, A, B, stream):
        from . import pencil_solve
        pencil_solve(plan, rank, nranks, recv.data_ptr(), A.data_ptr(), _ptr(B), stream)

    @staticmethod
    def pencil_backward(plan, rank, nranks, A, B, fslab, stream):
        from . import pencil_backward
        pencil_backward(plan, rank, nranks, A.data_ptr(), _ptr(B), fslab.data_ptr(), stream)

    @staticmethod
    def pencil_phase_b(plan, rank, nranks, fslab, u, F, e, stream):
        from . import pencil_phase_b
        pencil_phase_b(plan, rank, nranks, fslab.data_ptr(), u.data_ptr(), F.data_ptr(),
                       e.data_ptr(), stream)

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


# ----------------------------------------------------------------------------
# Distributed-FFT evaluation (include/esp_b200.h
# esp_pencil_*): the charge grid, the spectrum and the fields are split over
# the ranks -- x-planes in real space, y-rows between the two transposes --
# so no rank holds the whole grid.  Data crossing ranks per evaluation:
# two halo exchanges (P/2+2 planes each side), two all-to-all transposes of
# the half spectrum (the backward one carries A and B for ik), one all-reduce
# of [u | F | E].
# ----------------------------------------------------------------------------


class PencilLayout:
    """Geometry of every rank of a decomposition (esp_pencil_geometry); the
    split sizes and halo offsets below are in doubles (complex = 2)."""

    def __init__(self, geoms):
        self.g = list(geoms)
        self.G = len(self.g)
        g0 = self.g[0]
        self.nx, self.ny, self.nz = g0["nf"]
        self.nzh = self.nz // 2 + 1
        self.halo = g0["halo"]
        self.nfields = g0["nfields"]

    @classmethod
    def of(cls, plan, nranks, engine=None):
        engine = engine or _Lib
        return cls([engine.geometry(plan, r, nranks) for r in range(nranks)])

    def nxl(self, r):
        return self.g[r]["x1"] - self.g[r]["x0"]

    def nyl(self, r):
        return self.g[r]["y1"] - self.g[r]["y0"]

    def plane(self, nfields=1):
        return self.ny * self.nz * nfields

    # forward transpose (rank r's send to s / receive from s)
    def fwd_send_splits(self, r):
        return [2 * self.nxl(r) * self.nyl(s) * self.nzh for s in range(self.G)]

    def fwd_recv_splits(self, r):
        return [2 * self.nxl(s) * self.nyl(r) * self.nzh for s in range(self.G)]

    # backward transpose: the reverse
    def bwd_send_splits(self, r):
        return self.fwd_recv_splits(r)

    def bwd_recv_splits(self, r):
        return self.fwd_send_splits(r)

    def neighbours(self, r):
        return (r - 1) % self.G, (r + 1) % self.G

    def halo_out(self, r, nfields=1):
        """(to left, to right) plane ranges of rank r's spread slab that carry
        the neighbours' charge (its halos), in doubles."""
        pl, h, n = self.plane(nfields), self.halo, self.nxl(r)
        return (0, h * pl), ((n + h) * pl, (n + 2 * h) * pl)

    def halo_in(self, r, nfields=1):
        """(from right, from left) owned-plane ranges of rank r that receive
        the right neighbour's low halo and the left neighbour's high halo."""
        pl, h, n = self.plane(nfields), self.halo, self.nxl(r)
        return (n * pl, (n + h) * pl), (h * pl, 2 * h * pl)

    def fill_out(self, r, nfields):
        """(to left, to right) owned planes of rank r's field slab that fill
        the neighbours' halos."""
        pl, h, n = self.plane(nfields), self.halo, self.nxl(r)
        return (h * pl, 2 * h * pl), (n * pl, (n + h) * pl)

    def fill_in(self, r, nfields):
        """(from right, from left) halo ranges of rank r's field slab."""
        pl, h, n = self.plane(nfields), self.halo, self.nxl(r)
        return ((n + h) * pl, (n + 2 * h) * pl), (0, h * pl)


class PencilBuffers:
    """One rank's device buffers for the distributed-FFT evaluation."""

    def __init__(self, layout, rank, N, device):
        import torch
        g = layout.g[rank]
        f64 = dict(dtype=torch.float64, device=device)
        self.slab = torch.empty(g["slab_reals"], **f64)
        self.send = torch.empty(2 * g["spec_local"], **f64)
        self.recv = torch.empty(max(2 * g["spec_pencil"], 1), **f64)
        self.A = torch.empty(max(2 * g["spec_pencil"], 1), **f64)
        self.B = torch.empty(max(2 * g["spec_pencil"], 1), **f64) if g["nfields"] == 4 else None
        self.A2 = torch.empty(2 * g["spec_local"], **f64)
        self.B2 = torch.empty(2 * g["spec_local"], **f64) if g["nfields"] == 4 else None
        self.fslab = torch.empty(g["nfields"] * g["slab_reals"], **f64)
        self.out = torch.empty(4 * N + 1, **f64)


def _ptr(t):
    return t.data_ptr() if t is not None else 0


def _neighbour_exchange(t, outs, ins, left, right, add, group):
    """Send t[outs[0]] to `left` and t[outs[1]] to `right`; receive the right
    neighbour's piece into t[ins[0]] and the left's into t[ins[1]] (added or
    copied).  One message per peer (with two ranks both pieces go to the same
    peer, concatenated in a fixed order)."""
    import torch
    import torch.distributed as dist
    send = {}
    for peer, (a, b) in ((left, outs[0]), (right, outs[1])):
        send.setdefault(peer, []).append(t[a:b])
    recv_order = {}
    for peer, (a, b) in ((right, ins[0]), (left, ins[1])):
        recv_order.setdefault(peer, []).append((a, b))
    ops, bufs = [], {}
    for peer, parts in send.items():
        ops.append(dist.P2POp(dist.isend, torch.cat(parts) if len(parts) > 1 else parts[0].contiguous(),
                              peer, group))
    for peer, rngs in recv_order.items():
        bufs[peer] = torch.empty(sum(b - a for a, b in rngs), dtype=t.dtype, device=t.device)
        ops.append(dist.P2POp(dist.irecv, bufs[peer], peer, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for peer, rngs in recv_order.items():
        off = 0
        for a, b in rngs:
            piece = bufs[peer][off:off + (b - a)]
            if add:
                t[a:b] += piece
            else:
                t[a:b] = piece
            off += b - a


def evaluate_pencil(plan, box, N, pos, q, bufs, layout, rank, stream=0, group=None, engine=None,
                    reduce_outputs=True):
    """One rank's share of a distributed-FFT ESP evaluation (strong scaling;
    every rank calls this collectively).  pos (3N), q (N): the full system on
    every rank, or this rank's own atoms plus its ghosts (see
    evaluate_pencil_local); returns bufs.out = [u | F | E], summed over the
    ranks when reduce_outputs (replicated inputs), else this rank's share
    (its own atoms' u and F, zero elsewhere, and its energy part)."""
    import torch.distributed as dist
    engine = engine or _Lib
    G = layout.G
    left, right = layout.neighbours(rank)
    engine.pencil_phase_a(plan, box, N, pos, q, rank, G, bufs.slab, stream)
    _neighbour_exchange(bufs.slab, layout.halo_out(rank), layout.halo_in(rank), left, right,
                        True, group)
    engine.pencil_forward(plan, rank, G, bufs.slab, bufs.send, stream)
    dist.all_to_all_single(bufs.recv, bufs.send, layout.fwd_recv_splits(rank),
                           layout.fwd_send_splits(rank), group=group)
    engine.pencil_solve(plan, rank, G, bufs.recv, bufs.A, bufs.B, stream)
    dist.all_to_all_single(bufs.A2, bufs.A, layout.bwd_recv_splits(rank),
                           layout.bwd_send_splits(rank), group=group)
    if bufs.B is not None:
        dist.all_to_all_single(bufs.B2, bufs.B, layout.bwd_recv_splits(rank),
                               layout.bwd_send_splits(rank), group=group)
    engine.pencil_backward(plan, rank, G, bufs.A2, bufs.B2, bufs.fslab, stream)
    nf = layout.nfields
    _neighbour_exchange(bufs.fslab, layout.fill_out(rank, nf), layout.fill_in(rank, nf), left,
                        right, False, group)
    N_ = N
    engine.pencil_phase_b(plan, rank, G, bufs.fslab, bufs.out[:N_], bufs.out[N_:4 * N_],
                          bufs.out[4 * N_:], stream)
    if reduce_outputs:
        dist.all_reduce(bufs.out, group=group)
    return bufs.out


def evaluate_pencil_emulated(plans, box, N, pos, q, bufs, layout, stream=0, engine=None):
    """The same algorithm with all ranks in one process (lockstep; the
    exchanges become device copies): one plan and one PencilBuffers per
    emulated rank.  N, pos, q: the whole system (replicated inputs), or lists
    with one (local) system per rank.  Used by the single-GPU tests; the
    rank sum must equal evaluate() on the whole system."""
    engine = engine or _Lib
    G = layout.G
    per_rank = isinstance(N, (list, tuple))
    Ns = list(N) if per_rank else [N] * G
    poss = list(pos) if per_rank else [pos] * G
    qs = list(q) if per_rank else [q] * G
    for r in range(G):
        engine.pencil_phase_a(plans[r], box, Ns[r], poss[r], qs[r], r, G, bufs[r].slab, stream)
    _emulated_exchange([b.slab for b in bufs], layout, 1, add=True)
    for r in range(G):
        engine.pencil_forward(plans[r], r, G, bufs[r].slab, bufs[r].send, stream)
    _emulated_alltoall([b.send for b in bufs], [b.recv for b in bufs],
                       [layout.fwd_send_splits(r) for r in range(G)])
    for r in range(G):
        engine.pencil_solve(plans[r], r, G, bufs[r].recv, bufs[r].A, bufs[r].B, stream)
    _emulated_alltoall([b.A for b in bufs], [b.A2 for b in bufs],
                       [layout.bwd_send_splits(r) for r in range(G)])
    if layout.nfields == 4:
        _emulated_alltoall([b.B for b in bufs], [b.B2 for b in bufs],
                           [layout.bwd_send_splits(r) for r in range(G)])
    for r in range(G):
        engine.pencil_backward(plans[r], r, G, bufs[r].A2, bufs[r].B2, bufs[r].fslab, stream)
    _emulated_exchange([b.fslab for b in bufs], layout, layout.nfields, add=False)
    for r in range(G):
        o, n = bufs[r].out, Ns[r]
        engine.pencil_phase_b(plans[r], r, G, bufs[r].fslab, o[:n], o[n:4 * n], o[4 * n:],
                              stream)
    return [b.out for b in bufs] if per_rank else sum(b.out for b in bufs)


def _emulated_exchange(ts, layout, nfields, add):
    G = layout.G
    if add:
        outs = [layout.halo_out(r, nfields) for r in range(G)]
        ins = [layout.halo_in(r, nfields) for r in range(G)]
    else:
        outs = [layout.fill_out(r, nfields) for r in range(G)]
        ins = [layout.fill_in(r, nfields) for r in range(G)]
    # snapshot the outgoing pieces first (a copy may overwrite a halo another
    # rank still has to send from -- never for adds, but keep it uniform)
    pieces = [(ts[r][slice(*outs[r][0])].clone(), ts[r][slice(*outs[r][1])].clone())
              for r in range(G)]
    for r in range(G):
        left, right = layout.neighbours(r)
        to_left, to_right = pieces[r]
        # left neighbour receives it "from right"; right neighbour "from left"
        for peer, piece, which in ((left, to_left, 0), (right, to_right, 1)):
            a, b = ins[peer][which]
            if add:
                ts[peer][a:b] += piece
            else:
                ts[peer][a:b] = piece


def _emulated_alltoall(sends, recvs, send_splits):
    G = len(sends)
    offs = []
    for r in range(G):
        o, acc = [], 0
        for n in send_splits[r]:
            o.append(acc)
            acc += n
        offs.append(o)
    for r in range(G):
        pos = 0
        for s in range(G):
            n = send_splits[s][r]
            recvs[r][pos:pos + n] = sends[s][offs[s][r]:offs[s][r] + n]
            pos += n


# ---- local inputs: own atoms + ghosts instead of the replicated system -----


def fold_positions(pos, box):
    """system.hpp:29-36 on an (N, 3) numpy array or torch tensor (the
    engine's own fold; idempotent)."""
    import numpy as np
    if isinstance(pos, np.ndarray):
        L = np.asarray(box, dtype=np.float64)
        p = pos - L * np.floor(pos / L)
        return np.where(p >= L, 0.0, p)
    import torch
    L = torch.tensor(box, dtype=pos.dtype, device=pos.device)
    p = pos - L * torch.floor(pos / L)
    return torch.where(p >= L, torch.zeros_like(p), p)


def atom_owner(layout, x):
    """Rank owning each atom, from its folded x: the rank whose planes
    [x0, x1) hold clamp(floor(x/hx), 0, nx-1) (the engine's formula)."""
    import numpy as np
    hx, nx = layout.g[0]["hx"], layout.nx
    ends = [g["x1"] for g in layout.g]
    if isinstance(x, np.ndarray):
        pl = np.clip(np.floor(x / hx).astype(np.int64), 0, nx - 1)
        return np.searchsorted(np.asarray(ends), pl, side="right")
    import torch
    pl = torch.clamp(torch.floor(x / hx).to(torch.int64), 0, nx - 1)
    return torch.searchsorted(torch.tensor(ends, device=x.device), pl, right=True)


def slab_bounds(layout, r, box_x):
    """[X0, X1) of rank r's atoms in x."""
    g, hx = layout.g[r], layout.g[0]["hx"]
    X0 = g["x0"] * hx
    X1 = box_x if g["x1"] >= layout.nx else g["x1"] * hx
    return X0, X1


def check_ghost_reach(layout, box_x, r_c):
    """Ghosts come from the two x-neighbours only: every slab must be at
    least r_c wide."""
    for r in range(layout.G):
        X0, X1 = slab_bounds(layout, r, box_x)
        if X1 - X0 < r_c * (1.0 + 1e-9):
            from . import InvalidArgument
            raise InvalidArgument(f"distributed FFT: rank {r} slab ({X1 - X0:.3g}) is narrower "
                                  f"than r_c ({r_c:g}); use fewer ranks")


def ghost_masks(layout, r, x, box_x, r_c):
    """Masks of rank r's own atoms (folded x) to send to its left and right
    neighbours: those within r_c (plus a margin) of the shared slab faces."""
    X0, X1 = slab_bounds(layout, r, box_x)
    reach = r_c * (1.0 + 1e-9) + 1e-12 * box_x
    return (x - X0) <= reach, (X1 - x) <= reach


def exchange_ghosts(layout, rank, pos_own, q_own, box, r_c, group=None, return_plan=False):
    """Send this rank's atoms near its x-faces to the neighbours and receive
    theirs (NCCL send/recv on the GPU box, gloo in the CPU tests): returns the
    ghost positions (k, 3) and charges (k,).  pos_own must be folded.  With
    return_plan, also the bookkeeping return_ghost_terms needs (peers in
    receive order, own indices sent to each peer, rows received from each)."""
    import torch
    import torch.distributed as dist
    left, right = layout.neighbours(rank)
    to_l, to_r = ghost_masks(layout, rank, pos_own[:, 0], box[0], r_c)
    packed = torch.cat([pos_own, q_own[:, None]], dim=1)
    sends, sent_idx = {}, {}
    if left == right:
        sent_idx[left] = torch.nonzero(to_l | to_r).flatten()
    else:
        sent_idx[left] = torch.nonzero(to_l).flatten()
        sent_idx[right] = torch.nonzero(to_r).flatten()
    for p_, idx in sent_idx.items():
        sends[p_] = packed[idx]
    peers = sorted(sends)
    cnt_out = {p: torch.tensor([sends[p].shape[0]], dtype=torch.int64, device=pos_own.device)
               for p in peers}
    cnt_in = {p: torch.zeros(1, dtype=torch.int64, device=pos_own.device) for p in peers}
    ops = [dist.P2POp(dist.isend, cnt_out[p], p, group) for p in peers]
    ops += [dist.P2POp(dist.irecv, cnt_in[p], p, group) for p in peers]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    recv = {p: torch.empty((int(cnt_in[p].item()), 4), dtype=pos_own.dtype, device=pos_own.device)
            for p in peers}
    ops = [dist.P2POp(dist.isend, sends[p].contiguous(), p, group)
           for p in peers if sends[p].shape[0] > 0]
    ops += [dist.P2POp(dist.irecv, recv[p], p, group) for p in peers if recv[p].shape[0] > 0]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    g = torch.cat([recv[p] for p in peers], dim=0)
    if return_plan:
        plan = {"peers": peers, "sent_idx": sent_idx,
                "recv_cnt": {p: recv[p].shape[0] for p in peers}}
        return g[:, :3].contiguous(), g[:, 3].contiguous(), plan
    return g[:, :3].contiguous(), g[:, 3].contiguous()


def return_ghost_terms(plan, ghost_rows, own_rows, group=None):
    """Reverse of exchange_ghosts for the half-shell pair sum
    (ESP_PENCIL_HALF=1): a rank's evaluation leaves partner terms
    (u, Fx, Fy, Fz) on its ghost atoms; each ghost row goes back to the rank
    that owns the atom and is added to that atom's row there.  ghost_rows:
    (k, 4) in receive order; own_rows: (n, 4), updated in place."""
    import torch
    import torch.distributed as dist
    peers = plan["peers"]
    segs, o = {}, 0
    for p in peers:
        segs[p] = ghost_rows[o:o + plan["recv_cnt"][p]].contiguous()
        o += plan["recv_cnt"][p]
    back = {p: torch.empty((plan["sent_idx"][p].numel(), 4), dtype=own_rows.dtype,
                           device=own_rows.device) for p in peers}
    ops = [dist.P2POp(dist.isend, segs[p], p, group) for p in peers if segs[p].shape[0] > 0]
    ops += [dist.P2POp(dist.irecv, back[p], p, group) for p in peers if back[p].shape[0] > 0]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for p in peers:
        if back[p].shape[0] > 0:
            own_rows.index_add_(0, plan["sent_idx"][p].to(own_rows.device), back[p])


def pencil_half_enabled(plan=None) -> bool:
    """Whether the distributed FFT's K4 runs half-shell (then local inputs
    return ghost partner terms).  The mode is fixed when the plan is built
    (esp_plan_info.pencil_half); it is read from the plan, never from the
    environment at call time.  plan=None (engine-less callers) gives the
    build-time default, ESP_PENCIL_HALF != 0."""
    if plan is not None and hasattr(plan, "pencil_half"):
        return bool(plan.pencil_half)
    import os
    return os.environ.get("ESP_PENCIL_HALF", "1") != "0"


def evaluate_pencil_local(plan, box, pos_own, q_own, layout, rank, r_c, stream=0, group=None,
                          engine=None, cache=None):
    """Distributed-FFT evaluation from LOCAL inputs: each rank holds only the
    atoms it owns (atom_owner), receives its ghosts from the x-neighbours,
    and returns (u, F) of its own atoms plus the total energy (one all-reduce
    of a double) -- no rank ever holds the whole system.  pos_own: (n, 3)
    torch tensor (folded or not), q_own: (n,).  cache: optional dict keeping
    the rank's buffers between calls."""
    import torch
    import torch.distributed as dist
    check_ghost_reach(layout, box[0], r_c)
    pos_own = fold_positions(pos_own, box)
    gpos, gq, gplan = exchange_ghosts(layout, rank, pos_own, q_own, box, r_c, group,
                                      return_plan=True)
    pos_l = torch.cat([pos_own, gpos], dim=0).contiguous()
    q_l = torch.cat([q_own, gq]).contiguous()
    n_own, n = q_own.numel(), q_l.numel()
    bufs = cache.get("bufs") if cache is not None else None
    if bufs is None or bufs.out.numel() != 4 * n + 1:
        bufs = PencilBuffers(layout, rank, n, pos_l.device)
        if cache is not None:
            cache["bufs"] = bufs
    out = evaluate_pencil(plan, box, n, pos_l.reshape(-1), q_l, bufs, layout, rank, stream,
                          group, engine, reduce_outputs=False)
    if pencil_half_enabled(plan):
        # half-shell K4: the ghost rows hold partner terms owed to their owners;
        # return them, then E = 1/2 sum q u over the owned atoms (ewald.hpp:641-647)
        rows = torch.cat([out[:n, None], out[n:4 * n].reshape(n, 3)], dim=1)
        own_rows = rows[:n_own].clone()
        return_ghost_terms(gplan, rows[n_own:], own_rows, group)
        e = (0.5 * torch.dot(q_own.to(own_rows.dtype), own_rows[:, 0])).reshape(1)
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(e, group=group)
        return own_rows[:, 0].contiguous(), own_rows[:, 1:].contiguous(), e
    e = out[4 * n:].clone()
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(e, group=group)
    return out[:n_own], out[n:4 * n].reshape(n, 3)[:n_own], e
