"""Multi-process path of bench.py (replicas + max-over-ranks timing) on CPU
with the gloo backend, world_size 2."""
import os

import numpy as np
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_09727_b200 import systems as S
    from paper_2505_09727_b200.dist import env, max_over_ranks, replica_seed, weak_scaling_value
    r, w, lr = env()
    base = S.config("cfg1")
    c = S.Config(base.name, base.kind, base.N, base.L, base.r_c, base.eps,
                 seed=replica_seed(base.seed, r))
    pos, q, box = c.system()
    ms = [1.0 + r, 10.0 - r]  # per-rank "step times"
    mx = max_over_ranks(ms)
    out[r] = (r, w, lr, float(pos[0, 0]), mx, weak_scaling_value(q.size, w, mx[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_and_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert (r0[0], r0[1], r0[2]) == (0, 2, 0) and (r1[0], r1[1], r1[2]) == (1, 2, 1)
    assert r0[3] != r1[3]                       # replicas are distinct systems
    assert r0[4] == r1[4] == [2.0, 10.0]        # element-wise max over ranks
    assert r0[5] == pytest.approx(1000 * 2 / 2e-3)


def test_single_process_identity():
    from paper_2505_09727_b200.dist import max_over_ranks, replica_seed
    assert max_over_ranks([1.5, 2.5]) == [1.5, 2.5]
    assert replica_seed(1, 0) == 1 and replica_seed(1, 3) == 4


class _OracleEngine:
    """CPU stand-in for the per-rank C-ABI phases (test infrastructure): slabs
    are index ranges, the physics is the numpy oracle."""

    def __init__(self, oplan, pos, q):
        from oracle import esp_oracle as O
        self.O, self.p, self.pos, self.q = O, oplan, pos, q

    def _own(self, rank, nranks):
        N = self.q.size
        return slice(N * rank // nranks, N * (rank + 1) // nranks)

    def phase_a(self, plan, box, N, pos, q, rank, nranks, grid, stream):
        own = self._own(rank, nranks)
        g = self.O.spread(self.p, self.O.fold(self.pos[own], box), self.q[own])
        grid.copy_(torch.from_numpy(g.ravel()))
        ul, Fl = self.O.local_sum(self.p, self.pos, self.q)
        self.ul = np.zeros_like(ul)
        self.Fl = np.zeros_like(Fl)
        self.ul[own], self.Fl[own] = ul[own], Fl[own]

    def phase_b(self, plan, rank, nranks, grid, u, F, e, stream):
        own = self._own(rank, nranks)
        us, Fs = self.O.spectral_from_grid(self.p, grid.numpy(), self.pos, self.q)
        uu = self.ul.copy()
        FF = self.Fl.copy()
        uu[own] += us[own] - self.O.self_correction(self.p, self.q)[own]
        FF[own] += Fs[own]
        u.copy_(torch.from_numpy(uu))
        F.copy_(torch.from_numpy(FF.ravel()))
        e.fill_(0.5 * float(np.dot(self.q, uu)))


def _slab_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import esp_oracle as O
    from paper_2505_09727_b200.dist import evaluate_slab
    box = (10.0, 10.0, 10.0)
    pos, q = O.random_system(300, box, 3)
    p = O.build_plan(box, "pswf", 1e-3, 1.0)
    N = q.size
    res = torch.empty(4 * N + 1, dtype=torch.float64)
    grid = torch.empty(int(np.prod(p.nf)), dtype=torch.float64)
    evaluate_slab(p, box, N, None, None, res, grid, rank, world,
                  engine=_OracleEngine(p, pos, q))
    out[rank] = res.numpy().copy()
    dist.destroy_process_group()


def test_slab_decomposition_plumbing_gloo():
    """Two ranks: partial grids and partial outputs summed by all-reduce
    reproduce the single-process evaluation."""
    import numpy as np  # noqa: F811
    from oracle import esp_oracle as O
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    box = (10.0, 10.0, 10.0)
    pos, q = O.random_system(300, box, 3)
    E, u, F = O.evaluate(O.build_plan(box, "pswf", 1e-3, 1.0), pos, q)
    N = q.size
    for r in range(world):
        res = out[r]
        assert np.allclose(res[:N], u, rtol=0, atol=1e-12 * np.abs(u).max())
        assert np.allclose(res[N:4 * N].reshape(N, 3), F, rtol=0, atol=1e-12 * np.abs(F).max())
        assert abs(res[4 * N] - E) <= 1e-12 * abs(E)


# ---- distributed FFT (dist.evaluate_pencil) ---------------------------------


class _OraclePencilEngine:
    """CPU stand-in for the esp_pencil_* phases (test infrastructure): same
    buffer layouts, sizes and atom ownership as the C ABI
    (include/esp_b200.h), physics from the numpy oracle.  The inputs of
    pencil_phase_a (whole system or own atoms + ghosts) are what the rank
    computes with; it owns the atoms in its grid planes."""

    def __init__(self, oplan, host_plan):
        from oracle import esp_oracle as O
        self.O, self.p = O, oplan
        self.host_plan = host_plan
        self.state = {}

    def geometry(self, plan, rank, nranks):
        import paper_2505_09727_b200 as esp
        return esp.pencil_geometry(self.host_plan, rank, nranks)

    def _owned(self, g, pos):
        pl = np.clip(np.floor(pos[:, 0] / g["hx"]).astype(np.int64), 0, g["nf"][0] - 1)
        return (pl >= g["x0"]) & (pl < g["x1"])

    def _planes(self, g):
        return np.arange(g["x0"] - g["halo"], g["x1"] + g["halo"]) % self.p.nf[0]

    def pencil_phase_a(self, plan, box, N, pos, q, rank, nranks, slab, stream):
        g = self.geometry(plan, rank, nranks)
        pos = self.O.fold(np.asarray(pos).reshape(-1, 3), self.p.box)
        q = np.asarray(q)
        own = self._owned(g, pos)
        full = self.O.spread(self.p, pos[own], q[own])
        # own atoms touch only [x0-halo, x1+halo): the slab is exact
        slab.copy_(torch.from_numpy(np.ascontiguousarray(full[self._planes(g)]).ravel()))
        ul, Fl = self.O.local_sum(self.p, pos, q)
        u0, F0 = np.zeros_like(ul), np.zeros_like(Fl)
        u0[own], F0[own] = ul[own], Fl[own]
        self.state[rank] = (u0, F0, pos, q, own)

    def pencil_forward(self, plan, rank, nranks, slab, send, stream):
        g = self.geometry(plan, rank, nranks)
        nx, ny, nz = g["nf"]
        h, nxl = g["halo"], g["x1"] - g["x0"]
        own = slab.numpy().reshape(nxl + 2 * h, ny, nz)[h:h + nxl]
        spec = np.fft.rfft2(own, axes=(1, 2))                       # [nxl][ny][nzh]
        parts = []
        for s in range(nranks):
            gs = self.geometry(plan, s, nranks)
            parts.append(spec[:, gs["y0"]:gs["y1"], :].ravel())
        send.copy_(torch.from_numpy(np.concatenate(parts).view(np.float64)))

    def pencil_solve(self, plan, rank, nranks, recv, A, B, stream):
        g = self.geometry(plan, rank, nranks)
        nx, ny, nz = g["nf"]
        nyl, nzh = g["y1"] - g["y0"], nz // 2 + 1
        T = recv.numpy()[:2 * nx * nyl * nzh].view(np.complex128).reshape(nx, nyl, nzh)
        T = np.fft.fft(T, axis=0)
        c = T * self.p.influence[:, g["y0"]:g["y1"], :nzh]
        xi = np.where(2 * np.arange(nx) == nx, 0.0,
                      2 * np.pi * self.O.signed_mode(nx) / self.p.box[0])
        a = np.fft.ifft(c, axis=0) * nx
        A[:a.size * 2].copy_(torch.from_numpy(a.ravel().view(np.float64)))
        if B is not None:
            b = np.fft.ifft(c * (1j * xi)[:, None, None], axis=0) * nx
            B[:b.size * 2].copy_(torch.from_numpy(b.ravel().view(np.float64)))

    def pencil_backward(self, plan, rank, nranks, A, B, fslab, stream):
        g = self.geometry(plan, rank, nranks)
        nx, ny, nz = g["nf"]
        h, nxl, nzh, nf = g["halo"], g["x1"] - g["x0"], nz // 2 + 1, g["nfields"]
        def unpack(t):
            out = np.empty((nxl, ny, nzh), complex)
            flat = t.numpy().view(np.complex128)
            off = 0
            for s in range(nranks):
                gs = self.geometry(plan, s, nranks)
                n = nxl * (gs["y1"] - gs["y0"]) * nzh
                out[:, gs["y0"]:gs["y1"], :] = flat[off:off + n].reshape(nxl, -1, nzh)
                off += n
            return out
        a = unpack(A)
        specs = [a]
        if nf == 4:
            xiy = np.where(2 * np.arange(ny) == ny, 0.0,
                           2 * np.pi * self.O.signed_mode(ny) / self.p.box[1])
            xiz = np.where(2 * np.arange(nzh) == nz, 0.0,
                           2 * np.pi * np.arange(nzh) / self.p.box[2])
            specs += [unpack(B), a * (1j * xiy)[None, :, None], a * (1j * xiz)[None, None, :]]
        fs = fslab.numpy().reshape(nxl + 2 * h, ny, nz, nf)
        fs[:] = 0.0
        for f, sp in enumerate(specs):
            fs[h:h + nxl, :, :, f] = np.fft.irfft2(sp, s=(ny, nz), axes=(1, 2)) * (ny * nz)

    def pencil_phase_b(self, plan, rank, nranks, fslab, u, F, e, stream):
        g = self.geometry(plan, rank, nranks)
        nx, ny, nz = g["nf"]
        h, nxl, nf = g["halo"], g["x1"] - g["x0"], g["nfields"]
        fs = fslab.numpy().reshape(nxl + 2 * h, ny, nz, nf)
        uu, FF, pos, q, own = self.state[rank]
        P = pos[own]
        uu, FF = uu.copy(), FF.copy()
        full = np.zeros((nx, ny, nz))
        def interp(f, deriv=-1):
            full[:] = 0.0
            full[self._planes(g)] = fs[:, :, :, f]   # halo copies agree with their owners
            return self.O.interpolate(self.p, full, P, deriv)
        qo = q[own]
        uu[own] += interp(0) - self.O.self_correction(self.p, qo)
        if nf == 4:
            for d in range(3):
                FF[own, d] += -qo * interp(1 + d)
        else:
            for d in range(3):
                FF[own, d] += -qo * interp(0, d)
        u.copy_(torch.from_numpy(uu))
        F.copy_(torch.from_numpy(FF.ravel()))
        e.fill_(0.5 * float(np.dot(q, uu)))


def _pencil_case(fm="ik"):
    from oracle import esp_oracle as O
    import paper_2505_09727_b200 as esp
    box = (12.0, 10.0, 11.0)
    pos, q = O.random_system(240, box, 5)
    p = O.build_plan(box, "pswf", 1e-3, 1.0, force_method=fm)
    hp = esp.build_plan(box, "pswf", 1e-3, 1.0, esp.Overrides(force_method=fm), device=-1)
    return box, pos, q, p, hp


def _pencil_worker(rank, world, port, fm, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_09727_b200.dist import PencilBuffers, PencilLayout, evaluate_pencil
    box, pos, q, p, hp = _pencil_case(fm)
    eng = _OraclePencilEngine(p, hp)
    layout = PencilLayout.of(hp, world, engine=eng)
    bufs = PencilBuffers(layout, rank, q.size, "cpu")
    res = evaluate_pencil(hp, box, q.size, torch.from_numpy(pos.ravel().copy()),
                          torch.from_numpy(q), bufs, layout, rank, engine=eng)
    out[rank] = res.numpy().copy()
    dist.destroy_process_group()


def _check_against_oracle(res, p, pos, q):
    from oracle import esp_oracle as O
    E, u, F = O.evaluate(p, pos, q)
    N = q.size
    assert np.allclose(res[:N], u, rtol=0, atol=1e-11 * np.abs(u).max())
    assert np.allclose(res[N:4 * N].reshape(N, 3), F, rtol=0, atol=1e-11 * np.abs(F).max())
    assert abs(res[4 * N] - E) <= 1e-11 * abs(E)


@pytest.mark.parametrize("world,fm", [(2, "ik"), (3, "ik"), (2, "ad")])
def test_pencil_decomposition_gloo(world, fm):
    """Halo exchanges + both all-to-all transposes over gloo reproduce the
    single-process oracle evaluation."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pencil_worker, args=(world, _free_port(), fm, out), nprocs=world, join=True)
    box, pos, q, p, hp = _pencil_case(fm)
    for r in range(world):
        _check_against_oracle(out[r], p, pos, q)


@pytest.mark.parametrize("world", [2, 3])
def test_pencil_emulated_matches_oracle(world):
    """The lockstep emulation (the single-GPU test driver) on the same engine."""
    from paper_2505_09727_b200.dist import PencilBuffers, PencilLayout, evaluate_pencil_emulated
    box, pos, q, p, hp = _pencil_case()
    eng = _OraclePencilEngine(p, hp)
    layout = PencilLayout.of(hp, world, engine=eng)
    bufs = [PencilBuffers(layout, r, q.size, "cpu") for r in range(world)]
    res = evaluate_pencil_emulated([hp] * world, box, q.size, pos.ravel(), q, bufs, layout,
                                   engine=eng)
    _check_against_oracle(res.numpy(), p, pos, q)


def test_pencil_geometry_host():
    """Geometry from a host-only plan: planes and rows tile the grid; a rank
    with fewer planes than the halo is refused."""
    import paper_2505_09727_b200 as esp
    hp = esp.build_plan((12.0, 10.0, 11.0), "pswf", 1e-3, 1.0, device=-1)
    for G in (2, 3):
        gs = [esp.pencil_geometry(hp, r, G) for r in range(G)]
        assert gs[0]["x0"] == 0 and gs[-1]["x1"] == gs[0]["nf"][0]
        assert gs[0]["y0"] == 0 and gs[-1]["y1"] == gs[0]["nf"][1]
        for a, b in zip(gs, gs[1:]):
            assert a["x1"] == b["x0"] and a["y1"] == b["y0"]
        for g in gs:
            assert g["x1"] - g["x0"] >= g["halo"]
    with pytest.raises(esp.InvalidArgument):
        esp.pencil_geometry(hp, 0, 64)
    with pytest.raises(esp.InvalidArgument):
        esp.pencil_geometry(hp, 0, 1)


def _pencil_local_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_09727_b200.dist import (PencilLayout, atom_owner, evaluate_pencil_local,
                                            fold_positions)
    box, pos, q, p, hp = _pencil_case()
    eng = _OraclePencilEngine(p, hp)
    layout = PencilLayout.of(hp, world, engine=eng)
    posf = fold_positions(pos, box)
    idx = np.nonzero(atom_owner(layout, posf[:, 0]) == rank)[0]
    # this rank only ever sees its own atoms (unfolded, to exercise the fold)
    mine = pos[idx] + np.array(box) * (rank + 1)
    u, F, E = evaluate_pencil_local(hp, box, torch.from_numpy(mine), torch.from_numpy(q[idx]),
                                    layout, rank, 1.0, engine=eng)
    out[rank] = (idx, u.numpy().copy(), F.numpy().copy(), float(E))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pencil_local_inputs_gloo(world):
    """Each rank holds only its own atoms; ghosts travel between x-neighbours
    (send/recv), only the energy is all-reduced; the union of the ranks'
    outputs is the single-process oracle evaluation."""
    from oracle import esp_oracle as O
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pencil_local_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    box, pos, q, p, hp = _pencil_case()
    E, u, F = O.evaluate(p, pos, q)
    seen = np.zeros(q.size, dtype=int)
    for r in range(world):
        idx, ur, Fr, Er = out[r]
        seen[idx] += 1
        assert np.allclose(ur, u[idx], rtol=0, atol=1e-11 * np.abs(u).max())
        assert np.allclose(Fr, F[idx], rtol=0, atol=1e-11 * np.abs(F).max())
        assert abs(Er - E) <= 1e-11 * abs(E)
    assert (seen == 1).all()


def test_ghost_selection_host():
    """Ghost masks: an atom within r_c of a slab face goes to that neighbour;
    every atom within r_c (periodic, in x) of a rank's slab is either owned
    by it or one of its ghosts."""
    import paper_2505_09727_b200 as esp
    from paper_2505_09727_b200.dist import (PencilLayout, atom_owner, fold_positions,
                                            ghost_masks, slab_bounds)
    box = (12.0, 10.0, 11.0)
    hp = esp.build_plan(box, "pswf", 1e-3, 1.0, device=-1)
    pos = np.random.default_rng(2).uniform(-3.0, 15.0, (4000, 3))
    posf = fold_positions(pos, box)
    for G in (2, 3, 4):
        lay = PencilLayout.of(hp, G)
        own = atom_owner(lay, posf[:, 0])
        for r in range(G):
            X0, X1 = slab_bounds(lay, r, box[0])
            left, right = lay.neighbours(r)
            have = own == r
            for nb, side in ((left, 1), (right, 0)):
                m = own == nb
                tl, tr = ghost_masks(lay, nb, posf[:, 0], box[0], 1.0)
                have |= m & (tr if side == 1 else tl)
            d = np.minimum.reduce([np.abs(posf[:, 0] - X0), np.abs(posf[:, 0] - X1),
                                   np.abs(posf[:, 0] - X0 + box[0]),
                                   np.abs(posf[:, 0] - X1 - box[0])])
            inside = (posf[:, 0] >= X0) & (posf[:, 0] < X1)
            need = inside | (d < 1.0)
            assert (have | ~need).all()


def _ghost_return_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_09727_b200.dist import return_ghost_terms
    # ring: each rank sent atoms sent_idx[p] to peer p and received ghosts from p
    left, right = (rank - 1) % world, (rank + 1) % world
    peers = sorted({left, right})
    n_own = 10
    sent_idx = {p: torch.tensor([(3 * p + k) % n_own for k in range(2 + p)]) for p in peers}
    # the ghosts this rank holds from peer p are the atoms p sent to this rank:
    # p's sent_idx[rank] has 2 + rank entries
    recv_cnt = {p: 2 + rank for p in peers}
    rows = []
    for p in peers:
        for k in range(recv_cnt[p]):
            # term owed to atom k of p's send list to `rank`, tagged by (sender, k)
            rows.append([1000.0 * rank + k, p, k, 1.0])
    ghost_rows = torch.tensor(rows, dtype=torch.float64)
    own_rows = torch.zeros((n_own, 4), dtype=torch.float64)
    return_ghost_terms({"peers": peers, "sent_idx": sent_idx, "recv_cnt": recv_cnt},
                       ghost_rows, own_rows)
    out[rank] = (own_rows.numpy().copy(), {p: sent_idx[p].numpy().copy() for p in peers})
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_return_ghost_terms_gloo(world):
    """dist.return_ghost_terms (the half-shell distributed FFT's reverse ghost
    exchange): every ghost row reaches the rank that owns the atom and is added
    at the index that rank sent it from."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ghost_return_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        own, sent = out[r]
        expect = np.zeros((10, 4))
        for p, idx in sent.items():
            for k, i in enumerate(idx):
                expect[i] += [1000.0 * p + k, r, k, 1.0]
        assert np.array_equal(own, expect)


@pytest.mark.parametrize("world", [2])
def test_pencil_local_inputs_full_list_mode_gloo(world, monkeypatch):
    """ESP_PENCIL_HALF=0 path of evaluate_pencil_local (no reverse exchange,
    the engine's energy); the default path (half-shell: reverse ghost exchange,
    energy from the owned rows) is test_pencil_local_inputs_gloo."""
    monkeypatch.setenv("ESP_PENCIL_HALF", "0")
    test_pencil_local_inputs_gloo(world)
