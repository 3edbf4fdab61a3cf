"""B200-native ESP (Ewald summation with prolates) -- Python mirror of the
reference solver interface (/root/reference/proj/include/esp, namespace esp).

The names, argument meanings and error behaviour follow the reference:

    plan = build_plan(box, "pswf", eps=1e-4, r_c=1.0)          # ewald.hpp:355
    ef   = evaluate(plan, ParticleSystem(box, q, pos))           # ewald.hpp:619
    ef.energy, ef.u, ef.F, ef.timings

All compute runs in libesp_b200.so (hand-written sm_100a kernels + cuFFT)
through the C ABI declared in include/esp_b200.h.  There is no CPU
fallback: importing this package fails loudly if the library is missing,
and evaluating on a machine without a GPU raises CudaError.

Exceptions: InvalidArgument (a ValueError) where the reference throws
std::invalid_argument; NumericalError where it throws esp::NumericalError.
"""
from __future__ import annotations

import ctypes as C
import os
import time as _time
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "InvalidArgument", "NumericalError", "CudaError", "Overrides", "EwaldPlan",
    "ParticleSystem", "EnergyForces", "PartialField", "build_plan", "evaluate",
    "evaluate_device", "local_sum", "spectral_sum", "self_correction", "spread",
    "interpolate", "interpolate_gradient", "require_neutral", "fold", "device_count",
    "direct_ewald", "ReferenceResult", "fft_forward", "fft_inverse", "select_parameters",
    "LIB_PATH", "Shard", "shard_owner", "shard_unique_id", "evaluate_sharded_emulated",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
# ESP_B200_CHECKED=1 loads the checked build (device-side bounds checks,
# build.py --checked): a diagnostics variant of the same library
LIB_PATH = os.path.join(_PKG, "libesp_b200_checked.so" if os.environ.get("ESP_B200_CHECKED") == "1"
                        else "libesp_b200.so")
# experiments: an A/B build made by `build.py --variant NAME -D...`
if os.environ.get("ESP_B200_LIB"):
    LIB_PATH = os.path.join(_PKG, os.environ["ESP_B200_LIB"])

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2505_09727_b200/build.py` "
        "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class NumericalError(RuntimeError):
    """esp::NumericalError (prolate.hpp:17-20)."""


class CudaError(RuntimeError):
    """CUDA / cuFFT failure, or a device entry point on a host-only plan."""


class _Overrides(C.Structure):
    _fields_ = [("nf", C.c_int), ("P", C.c_int), ("c1", C.c_double),
                ("force_method", C.c_int), ("allow_degraded", C.c_int)]


class _Info(C.Structure):
    _fields_ = [
        ("family", C.c_int), ("force_method", C.c_int), ("P", C.c_int),
        ("nf", C.c_int * 3), ("base_nf", C.c_int * 3),
        ("eps", C.c_double), ("r_c", C.c_double), ("shape", C.c_double), ("c1", C.c_double),
        ("chi0", C.c_double),
        ("box", C.c_double * 3), ("h", C.c_double * 3), ("demand", C.c_double * 3),
        ("E_A", C.c_double), ("E_T", C.c_double), ("E_SI", C.c_double),
        ("self_coef", C.c_double),
        ("n_split_coef", C.c_int), ("n_window_coef", C.c_int), ("pair_poly_degree", C.c_int),
        ("pair_fit_err", C.c_double), ("device", C.c_int), ("pair_cells", C.c_int * 3),
        ("pencil_half", C.c_int), ("fused_xpass", C.c_int), ("deterministic", C.c_int),
        ("pair_kernel", C.c_int), ("spread_kernel", C.c_int),
    ]


class _PencilInfo(C.Structure):
    _fields_ = [
        ("nranks", C.c_int), ("rank", C.c_int), ("halo", C.c_int), ("x0", C.c_int),
        ("x1", C.c_int), ("y0", C.c_int), ("y1", C.c_int), ("nfields", C.c_int),
        ("nf", C.c_int * 3), ("hx", C.c_double), ("S", C.c_int), ("nbx", C.c_int),
        ("bx0", C.c_int), ("bx1", C.c_int),
        ("slab_reals", C.c_long), ("spec_local", C.c_long), ("spec_pencil", C.c_long),
    ]


class _ShardInfo(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("x0", C.c_int), ("x1", C.c_int),
                ("X0", C.c_double), ("X1", C.c_double), ("max_own_atoms", C.c_long),
                ("ghost_capacity", C.c_long), ("local_atoms", C.c_long),
                ("pencil_half", C.c_int), ("fused_xpass", C.c_int), ("deterministic", C.c_int), ("nccl", C.c_int)]


class _DirectInfo(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("real_shells", C.c_int), ("recip_kmax", C.c_int),
                ("tail_bound", C.c_double)]


class _Timings(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("local", "spread", "fft", "scale", "ifft", "interpolate", "bin")]


def _sig(name, args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_vp = C.c_void_p
_sig("esp_last_error", [], C.c_char_p)
_sig("esp_version", [], C.c_char_p)
_sig("esp_device_count", [])
_sig("esp_plan_create", [_dp, C.c_int, C.c_double, C.c_double, C.POINTER(_Overrides), C.c_int,
                         C.POINTER(_vp)])
_sig("esp_plan_destroy", [_vp], None)
_sig("esp_plan_get_info", [_vp, C.POINTER(_Info)])
_sig("esp_plan_set_deterministic", [_vp, C.c_int])
_sig("esp_plan_get_influence", [_vp, _dp])
_sig("esp_plan_get_table", [_vp, C.c_int, C.c_int, _vp, C.POINTER(C.c_int)])
_sig("esp_plan_get_prolate", [_vp, C.c_int, _vp, C.POINTER(C.c_int)])
_sig("esp_plan_eval_kernel", [_vp, C.c_int, C.c_long, _dp, _dp])
_sig("esp_evaluate", [_vp, _dp, C.c_long, _dp, _dp, _dp, _dp, C.POINTER(C.c_double),
                      C.POINTER(_Timings)])
_sig("esp_evaluate_device", [_vp, _dp, C.c_long, _vp, _vp, _vp, _vp, _vp, _vp])
_sig("esp_check_neutral", [C.c_long, _dp])
_sig("esp_shard_unique_id", [_vp])
_sig("esp_shard_create", [_vp, _vp, C.c_int, C.c_int, C.c_long, C.c_long, C.POINTER(_vp)])
_sig("esp_shard_destroy", [_vp], None)
_sig("esp_shard_info", [_vp, C.POINTER(_ShardInfo)])
_sig("esp_shard_owner", [_vp, C.c_int, C.c_long, _dp, _vp])
_sig("esp_shard_evaluate", [_vp, _dp, C.c_long, _vp, _vp, _vp, _vp, _vp, _vp])
_sig("esp_shard_evaluate_emulated", [_vp, C.c_int, _dp, _vp, _vp, _vp, _vp, _vp, _vp, _vp])
_sig("esp_shard_check", [_vp])
_sig("esp_local_sum", [_vp, _dp, C.c_long, _dp, _dp, _dp, _dp])
_sig("esp_spectral_sum", [_vp, _dp, C.c_long, _dp, _dp, _dp, _dp, C.POINTER(_Timings)])
_sig("esp_self_correction", [_vp, C.c_long, _dp, _dp])
_sig("esp_spread", [_vp, C.c_long, _dp, _dp, _dp])
_sig("esp_interpolate", [_vp, C.c_long, _dp, _dp, _dp])
_sig("esp_interpolate_gradient", [_vp, C.c_long, _dp, _dp, _dp])
_sig("esp_last_launch_count", [_vp])
_sig("esp_eval_phase_a", [_vp, _dp, C.c_long, _vp, _vp, C.c_int, C.c_int, _vp, _vp])
_sig("esp_eval_phase_b", [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp])
_sig("esp_grid_size", [_vp], C.c_long)
_sig("esp_fft3", [C.POINTER(C.c_int), _vp, C.c_int, C.c_int])
_sig("esp_direct_ewald", [_dp, C.c_long, _dp, _dp, C.c_long, _vp, C.c_double, C.c_double, _dp,
                          _dp, C.POINTER(C.c_double), C.POINTER(_DirectInfo), C.c_int])
_sig("esp_pencil_geometry", [_vp, C.c_int, C.c_int, C.POINTER(_PencilInfo)])
_sig("esp_pencil_phase_a", [_vp, _dp, C.c_long, _vp, _vp, C.c_int, C.c_int, _vp, _vp])
_sig("esp_pencil_forward", [_vp, C.c_int, C.c_int, _vp, _vp, _vp])
_sig("esp_pencil_solve", [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp])
_sig("esp_pencil_backward", [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp])
_sig("esp_pencil_phase_b", [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp])
_sig("esp_last_pair_count", [_vp, C.POINTER(C.c_ulonglong)])
_sig("esp_fp64_peak", [C.c_int, C.POINTER(C.c_double)])
_sig("esp_pair_eval_rate", [_vp, C.POINTER(C.c_double)])


def _check(rc: int):
    if rc == 0:
        return
    msg = (_lib.esp_last_error() or b"").decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 2:
        raise NumericalError(msg)
    if rc in (3, 4):
        raise CudaError(msg)
    raise RuntimeError(msg)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def device_count() -> int:
    return int(_lib.esp_device_count())


def version() -> str:
    return _lib.esp_version().decode()


@dataclass
class Overrides:
    """ewald.hpp:38-47."""
    nf: int = 0
    P: int = 0
    c1: float = 0.0
    force_method: str = "ik"
    allow_degraded: bool = False

    def _c(self) -> _Overrides:
        if self.force_method not in ("ik", "ad"):
            raise InvalidArgument("unknown force method: " + str(self.force_method))
        return _Overrides(int(self.nf), int(self.P), float(self.c1),
                          1 if self.force_method == "ad" else 0, int(bool(self.allow_degraded)))


@dataclass
class PlanStats:
    E_A: float
    E_T: float
    E_SI: float


class EwaldPlan:
    """Immutable plan (ewald.hpp:67-94) owning its device state."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        info = _Info()
        _check(_lib.esp_plan_get_info(self._h, C.byref(info)))
        self._info = info
        self.family = "gaussian" if info.family == 1 else "pswf"
        self.window_family = "bspline" if info.family == 1 else "pswf"
        self.force_method = "ad" if info.force_method == 1 else "ik"
        self.eps = info.eps
        self.r_c = info.r_c
        self.box = tuple(info.box)
        self.nf = tuple(info.nf)
        self.base_nf = tuple(info.base_nf)
        self.demand = tuple(info.demand)
        self.h = tuple(info.h)
        self.P = info.P
        self.shape = info.shape
        self.c1 = info.c1
        self.chi0 = info.chi0
        self.self_coef = info.self_coef
        self.stats = PlanStats(info.E_A, info.E_T, info.E_SI)
        self.device = info.device
        self.pair_poly_degree = info.pair_poly_degree
        self.pair_fit_err = info.pair_fit_err
        self.pair_cells = tuple(info.pair_cells)
        # distributed-FFT K4 mode, fixed at plan build (include/esp_b200.h)
        self.pencil_half = bool(info.pencil_half)
        # K2 inside the FFT's x pass (include/esp_b200.h)
        self.fused_xpass = bool(info.fused_xpass)

    @property
    def pair_kernel(self) -> str:
        """Real-space kernel of the plan's last evaluation (esp_plan_info.pair_kernel):
        "none", "full", "half", "tile" (cluster pairs) or "allpairs"."""
        info = _Info()
        _check(_lib.esp_plan_get_info(self._h, C.byref(info)))
        return {-1: "none", 0: "full", 1: "half", 2: "tile", 3: "allpairs"}[info.pair_kernel]

    @property
    def spread_kernel(self) -> str:
        """Spreading kernel of the plan's last evaluation (esp_plan_info.spread_kernel):
        "none", "cta" (k_spread) or "warp" (k_spread_warp)."""
        info = _Info()
        _check(_lib.esp_plan_get_info(self._h, C.byref(info)))
        return {-1: "none", 0: "cta", 1: "warp"}[info.spread_kernel]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.esp_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def total_modes(self) -> int:
        return int(self.nf[0]) * int(self.nf[1]) * int(self.nf[2])

    def avg_neighbors(self, N: int) -> float:
        return (4.0 / 3.0) * np.pi * self.r_c ** 3 * N / float(np.prod(self.box))

    @property
    def influence(self) -> np.ndarray:
        out = np.empty(self.total_modes())
        _check(_lib.esp_plan_get_influence(self._h, out))
        return out.reshape(self.nf)

    def table(self, which: str, dim: int = 0) -> np.ndarray:
        sel = {"Psi": 0, "chi": 1, "phi": 2, "dphi": 3}[which]
        n = C.c_int()
        _check(_lib.esp_plan_get_table(self._h, sel, dim, None, C.byref(n)))
        out = np.empty(n.value * 13)
        _check(_lib.esp_plan_get_table(self._h, sel, dim, out.ctypes.data, C.byref(n)))
        return out.reshape(n.value, 13)

    def prolate_coef(self, which: int = -1) -> np.ndarray:
        n = C.c_int()
        _check(_lib.esp_plan_get_prolate(self._h, which, None, C.byref(n)))
        out = np.empty(n.value)
        _check(_lib.esp_plan_get_prolate(self._h, which, out.ctypes.data, C.byref(n)))
        return out

    def eval_kernel(self, what: str, x) -> np.ndarray:
        sel = {"Psi": 0, "chi": 1, "chihat_n": 2, "phi": 3, "dphi": 4, "phi_hat": 5,
               "local_pot": 6, "local_fr": 7}[what]
        x = _f64(np.atleast_1d(x))
        y = np.empty_like(x)
        _check(_lib.esp_plan_eval_kernel(self._h, sel, x.size, x, y))
        return y

    def set_deterministic(self, on: bool = True) -> None:
        """esp_plan_set_deterministic: bitwise-reproducible evaluations (slower)."""
        _check(_lib.esp_plan_set_deterministic(self._h, 1 if on else 0))

    @property
    def deterministic(self) -> bool:
        info = _Info()
        _check(_lib.esp_plan_get_info(self._h, C.byref(info)))
        return bool(info.deterministic)

    def last_launch_count(self) -> int:
        return int(_lib.esp_last_launch_count(self._h))

    def last_pair_count(self) -> int:
        """Ordered in-range pairs evaluated by the last pair-sum launch."""
        v = C.c_ulonglong()
        _check(_lib.esp_last_pair_count(self._h, C.byref(v)))
        return int(v.value)


def pair_eval_rate(plan) -> float:
    """Ordered pairs/s of the K4 evaluation alone (no neighbour search)."""
    v = C.c_double()
    _check(_lib.esp_pair_eval_rate(plan._h, C.byref(v)))
    return float(v.value)


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured DFMA throughput of `device` (TFLOP/s)."""
    v = C.c_double()
    _check(_lib.esp_fp64_peak(int(device), C.byref(v)))
    return float(v.value)


@dataclass
class ParticleSystem:
    """system.hpp:19-26: box edges, charges, positions (N x 3)."""
    box: tuple
    q: np.ndarray
    pos: np.ndarray

    def __post_init__(self):
        self.box = tuple(float(b) for b in self.box)
        self.q = _f64(self.q)
        self.pos = _f64(self.pos).reshape(-1, 3)
        if self.pos.shape[0] != self.q.shape[0]:
            raise InvalidArgument("positions and charges differ in length")

    def size(self) -> int:
        return int(self.q.shape[0])

    def volume(self) -> float:
        return float(np.prod(self.box))


@dataclass
class EnergyForces:
    """system.hpp:49-55."""
    energy: float
    u: np.ndarray
    F: np.ndarray
    timings: dict = field(default_factory=dict)


@dataclass
class PartialField:
    """ewald.hpp:411-414."""
    u: np.ndarray
    F: np.ndarray


def build_plan(box, family: str = "pswf", eps: float = 1e-4, r_c: float = 1.0,
               ov: Overrides | None = None, device: int | None = None) -> EwaldPlan:
    """ewald.hpp:355-405.  device=None picks GPU 0 when one is visible and
    builds a host-only plan (parameters and tables, no evaluation) otherwise."""
    if family not in ("pswf", "gaussian"):
        raise InvalidArgument("unknown screen family: " + str(family))
    if device is None:
        device = 0 if device_count() > 0 else -1
    ov = ov or Overrides()
    h = C.c_void_p()
    _check(_lib.esp_plan_create(_f64(box, (3,)), 1 if family == "gaussian" else 0, float(eps),
                                float(r_c), C.byref(ov._c()), int(device), C.byref(h)))
    return EwaldPlan(h)


def fold(system: ParticleSystem) -> ParticleSystem:
    """system.hpp:29-36 (host helper; the device path folds inside K0)."""
    L = np.asarray(system.box)
    p = system.pos - L * np.floor(system.pos / L)
    p = np.where(p >= L, 0.0, p)
    return ParticleSystem(system.box, system.q.copy(), p)


def require_neutral(system: ParticleSystem) -> None:
    """system.hpp:39-47."""
    _check(_lib.esp_check_neutral(system.size(), system.q))


def evaluate(plan: EwaldPlan, system: ParticleSystem, timings: bool = True,
             out: tuple | None = None) -> EnergyForces:
    """ewald.hpp:619-649 on host arrays (H2D, GPU evaluation, D2H).

    Like the reference, the result's timings hold the per-stage times
    (seconds) under its keys {local, spread, fft, scale, ifft, interpolate}
    -- the stages then run serialised, each timed alone with CUDA events --
    plus the GPU-only 'bin' (fold, cell keys, sorts).  timings=False selects
    the overlapped CUDA-graph path (real-space sum concurrent with the grid
    pipeline) and reports only 'total', the host wall time of the call.
    out=(u, F) supplies preallocated (e.g. pinned) float64 output arrays."""
    N = system.size()
    if out is not None:
        u, F = out
        if u.shape != (N,) or F.shape != (N, 3) or u.dtype != np.float64 or F.dtype != np.float64:
            raise InvalidArgument("out arrays must be float64 (N,) and (N, 3)")
    else:
        u = np.empty(N)
        F = np.empty((N, 3))
    e = C.c_double()
    t = _Timings() if timings else None
    t0 = _time.perf_counter()
    _check(_lib.esp_evaluate(plan._h, _f64(system.box, (3,)), N, system.pos, system.q, u, F,
                             C.byref(e), C.byref(t) if t is not None else None))
    wall = _time.perf_counter() - t0
    tim = {k: getattr(t, k) for k, _ in _Timings._fields_} if t is not None else {}
    tim["total"] = wall
    return EnergyForces(e.value, u, F, tim)


def evaluate_device(plan: EwaldPlan, box, N: int, pos_ptr: int, q_ptr: int, u_ptr: int,
                    F_ptr: int, energy_ptr: int, stream: int = 0) -> None:
    """Device-resident evaluate (asynchronous on `stream`); pointers are raw
    device addresses (e.g. torch.Tensor.data_ptr())."""
    _check(_lib.esp_evaluate_device(plan._h, _f64(box, (3,)), int(N), C.c_void_p(pos_ptr),
                                    C.c_void_p(q_ptr), C.c_void_p(u_ptr), C.c_void_p(F_ptr),
                                    C.c_void_p(energy_ptr), C.c_void_p(stream)))


def eval_phase_a(plan: EwaldPlan, box, N: int, pos_ptr: int, q_ptr: int, rank: int, nranks: int,
                 grid_ptr: int, stream: int = 0) -> None:
    """Slab decomposition, phase A (see include/esp_b200.h): real-space sum for
    this rank's targets, spread of its atoms into the grid at grid_ptr."""
    _check(_lib.esp_eval_phase_a(plan._h, _f64(box, (3,)), int(N), C.c_void_p(pos_ptr),
                                 C.c_void_p(q_ptr), int(rank), int(nranks), C.c_void_p(grid_ptr),
                                 C.c_void_p(stream)))


def eval_phase_b(plan: EwaldPlan, rank: int, nranks: int, grid_ptr: int, u_ptr: int, F_ptr: int,
                 energy_ptr: int, stream: int = 0) -> None:
    """Phase B on the rank-summed grid: this rank's partial u, F, energy."""
    _check(_lib.esp_eval_phase_b(plan._h, int(rank), int(nranks), C.c_void_p(grid_ptr),
                                 C.c_void_p(u_ptr), C.c_void_p(F_ptr), C.c_void_p(energy_ptr),
                                 C.c_void_p(stream)))


def pencil_geometry(plan: EwaldPlan, rank: int, nranks: int) -> dict:
    """Distributed-FFT geometry of one rank (include/esp_b200.h esp_pencil_info):
    owned x-planes [x0, x1) with `halo` planes each side, spectral rows
    [y0, y1), buffer sizes.  Host-only plans work too."""
    g = _PencilInfo()
    _check(_lib.esp_pencil_geometry(plan._h, int(rank), int(nranks), C.byref(g)))
    d = {k: getattr(g, k) for k, _ in _PencilInfo._fields_}
    d["nf"] = tuple(g.nf)
    return d


def pencil_phase_a(plan: EwaldPlan, box, N: int, pos_ptr: int, q_ptr: int, rank: int,
                   nranks: int, slab_ptr: int, stream: int = 0) -> None:
    _check(_lib.esp_pencil_phase_a(plan._h, _f64(box, (3,)), int(N), C.c_void_p(pos_ptr),
                                   C.c_void_p(q_ptr), int(rank), int(nranks),
                                   C.c_void_p(slab_ptr), C.c_void_p(stream)))


def pencil_forward(plan: EwaldPlan, rank: int, nranks: int, slab_ptr: int, send_ptr: int,
                   stream: int = 0) -> None:
    _check(_lib.esp_pencil_forward(plan._h, int(rank), int(nranks), C.c_void_p(slab_ptr),
                                   C.c_void_p(send_ptr), C.c_void_p(stream)))


def pencil_solve(plan: EwaldPlan, rank: int, nranks: int, recv_ptr: int, A_ptr: int,
                 B_ptr: int, stream: int = 0) -> None:
    _check(_lib.esp_pencil_solve(plan._h, int(rank), int(nranks), C.c_void_p(recv_ptr),
                                 C.c_void_p(A_ptr), C.c_void_p(B_ptr or None),
                                 C.c_void_p(stream)))


def pencil_backward(plan: EwaldPlan, rank: int, nranks: int, A_ptr: int, B_ptr: int,
                    fslab_ptr: int, stream: int = 0) -> None:
    _check(_lib.esp_pencil_backward(plan._h, int(rank), int(nranks), C.c_void_p(A_ptr),
                                    C.c_void_p(B_ptr or None), C.c_void_p(fslab_ptr),
                                    C.c_void_p(stream)))


def pencil_phase_b(plan: EwaldPlan, rank: int, nranks: int, fslab_ptr: int, u_ptr: int,
                   F_ptr: int, energy_ptr: int, stream: int = 0) -> None:
    _check(_lib.esp_pencil_phase_b(plan._h, int(rank), int(nranks), C.c_void_p(fslab_ptr),
                                   C.c_void_p(u_ptr), C.c_void_p(F_ptr), C.c_void_p(energy_ptr),
                                   C.c_void_p(stream)))


@dataclass
class ReferenceResult:
    """reference.hpp:21-29 (u, F for the targets; energy NaN for subsets)."""
    u: np.ndarray
    F: np.ndarray
    energy: float
    lambda_: float
    real_shells: int
    recip_kmax: int
    residual: float


def _direct_pass(system: ParticleSystem, tol, lam, targets, device):
    N = system.size()
    tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    n = N if tg is None else tg.size
    u = np.empty(n)
    F = np.empty((n, 3))
    e = C.c_double()
    info = _DirectInfo()
    _check(_lib.esp_direct_ewald(_f64(system.box, (3,)), N, system.pos, system.q,
                                 0 if tg is None else tg.size,
                                 None if tg is None else tg.ctypes.data_as(C.c_void_p),
                                 float(tol), float(lam), u, F, C.byref(e), C.byref(info),
                                 int(device)))
    return u, F, e.value, info


def direct_ewald(system: ParticleSystem, tol: float = 1e-9, targets=None,
                 device: int = 0) -> ReferenceResult:
    """esp::direct_ewald (reference.hpp:212-238) on the GPU: a pass at
    lambda = min(L)/6 and a check pass at 1.3 lambda, whose gap (energy, or the
    target potentials for a subset) must stay within tol.  targets: optional
    atom indices (the subset form has no N cap; the reference's is 1e4)."""
    lam = min(system.box) / 6.0
    u1, F1, E1, i1 = _direct_pass(system, tol, lam, targets, device)
    u2, F2, E2, _ = _direct_pass(system, tol, 1.3 * lam, targets, device)
    if targets is None:
        gap = abs(E1 - E2)
        scale = max(1.0, abs(E1))
    else:
        gap = float(np.max(np.abs(u1 - u2))) if u1.size else 0.0
        scale = max(1.0, float(np.max(np.abs(u1))) if u1.size else 1.0)
    if gap > tol * scale:
        raise NumericalError("direct_ewald: splitting-width invariance check failed")
    return ReferenceResult(u1, F1, E1, i1.lambda_, i1.real_shells, i1.recip_kmax,
                           max(gap, i1.tail_bound))


def fft_forward(grid: np.ndarray, device: int = 0) -> np.ndarray:
    """gridder.hpp:153: unnormalised forward 3-D DFT (e^{-i}) on the GPU;
    returns a new complex128 array of the same shape."""
    return _fft3(grid, -1, device)


def fft_inverse(grid: np.ndarray, device: int = 0) -> np.ndarray:
    """gridder.hpp:154: unnormalised inverse 3-D DFT (e^{+i}) on the GPU."""
    return _fft3(grid, 1, device)


def _fft3(grid, direction, device):
    g = np.ascontiguousarray(grid, dtype=np.complex128).copy()
    if g.ndim != 3:
        raise InvalidArgument("fft: need a 3-D grid")
    nf = (C.c_int * 3)(*g.shape)
    _check(_lib.esp_fft3(nf, g.ctypes.data_as(C.c_void_p), int(direction), int(device)))
    return g


def select_parameters(family: str, eps: float, box, r_c: float,
                      overrides: Overrides | None = None) -> dict:
    """ewald.hpp:338-350 (SelectResult): the parameter choice alone."""
    p = build_plan(box, family, eps, r_c, overrides, device=-1)
    return {"family": p.family, "shape": p.shape, "P": p.P, "c1": p.c1, "demand": p.demand,
            "base_nf": p.base_nf, "nf": p.nf, "E_A": p.stats.E_A, "E_SI": p.stats.E_SI}


def grid_size(plan: EwaldPlan) -> int:
    return int(_lib.esp_grid_size(plan._h))


def local_sum(plan: EwaldPlan, system: ParticleSystem) -> PartialField:
    """ewald.hpp:419-515."""
    N = system.size()
    u = np.empty(N)
    F = np.empty((N, 3))
    _check(_lib.esp_local_sum(plan._h, _f64(system.box, (3,)), N, system.pos, system.q, u, F))
    return PartialField(u, F)


def spectral_sum(plan: EwaldPlan, system: ParticleSystem,
                 timings: dict | None = None) -> PartialField:
    """ewald.hpp:524-604.  Like the reference, a `timings` dict receives the
    stage times (seconds, added to existing values) under spread, fft, scale,
    ifft, interpolate."""
    N = system.size()
    u = np.empty(N)
    F = np.empty((N, 3))
    t = _Timings() if timings is not None else None
    _check(_lib.esp_spectral_sum(plan._h, _f64(system.box, (3,)), N, system.pos, system.q, u,
                                 F, C.byref(t) if t is not None else None))
    if t is not None:
        for k in ("spread", "fft", "scale", "ifft", "interpolate"):
            timings[k] = timings.get(k, 0.0) + getattr(t, k)
    return PartialField(u, F)


def self_correction(plan: EwaldPlan, q) -> np.ndarray:
    """ewald.hpp:609-615."""
    q = _f64(q)
    out = np.empty_like(q)
    _check(_lib.esp_self_correction(plan._h, q.size, q, out))
    return out


def spread(plan: EwaldPlan, system: ParticleSystem) -> np.ndarray:
    """gridder.hpp:215-241: the real charge grid (nx, ny, nz)."""
    g = np.empty(plan.total_modes())
    _check(_lib.esp_spread(plan._h, system.size(), system.pos, system.q, g))
    return g.reshape(plan.nf)


def interpolate(plan: EwaldPlan, grid, system: ParticleSystem) -> np.ndarray:
    """gridder.hpp:244-277 of a real grid."""
    out = np.empty(system.size())
    _check(_lib.esp_interpolate(plan._h, system.size(), system.pos, _f64(grid).ravel(), out))
    return out


def interpolate_gradient(plan: EwaldPlan, grid, system: ParticleSystem) -> np.ndarray:
    """gridder.hpp:280-314."""
    out = np.empty((system.size(), 3))
    _check(_lib.esp_interpolate_gradient(plan._h, system.size(), system.pos,
                                         _f64(grid).ravel(), out))
    return out


# ---- sharded evaluation over the GPUs of one box (include/esp_b200.h esp_shard_*)


def shard_unique_id() -> bytes:
    """A new NCCL unique id (128 bytes), to be shared with every rank."""
    buf = C.create_string_buffer(128)
    _check(_lib.esp_shard_unique_id(buf))
    return buf.raw


def shard_owner(plan: EwaldPlan, nranks: int, pos) -> np.ndarray:
    """Owner rank of every atom (host (N, 3) positions, any image)."""
    pos = _f64(pos).reshape(-1, 3)
    out = np.empty(pos.shape[0], dtype=np.int32)
    _check(_lib.esp_shard_owner(plan._h, int(nranks), pos.shape[0], pos, out.ctypes.data))
    return out


class Shard:
    """One rank of a sharded evaluation (esp_shard_create).  nccl_id=None
    makes an emulation member for evaluate_sharded_emulated."""

    def __init__(self, plan: EwaldPlan, rank: int, nranks: int, max_own_atoms: int,
                 nccl_id: bytes | None = None, ghost_capacity: int = 0):
        self.plan = plan  # keeps the plan alive
        h = C.c_void_p()
        idb = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(_lib.esp_shard_create(plan._h, idb, int(rank), int(nranks), int(max_own_atoms),
                                     int(ghost_capacity), C.byref(h)))
        self._h = h
        info = _ShardInfo()
        _check(_lib.esp_shard_info(self._h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in _ShardInfo._fields_}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.esp_shard_destroy(h)
            except Exception:
                pass
            self._h = None

    def evaluate(self, box, n_own: int, pos_ptr: int, q_ptr: int, u_ptr: int, F_ptr: int,
                 energy_ptr: int, stream: int = 0) -> None:
        """esp_shard_evaluate (collective; device pointers, asynchronous)."""
        _check(_lib.esp_shard_evaluate(self._h, _f64(box, (3,)), int(n_own), C.c_void_p(pos_ptr),
                                       C.c_void_p(q_ptr), C.c_void_p(u_ptr), C.c_void_p(F_ptr),
                                       C.c_void_p(energy_ptr), C.c_void_p(stream)))

    def check(self) -> None:
        _check(_lib.esp_shard_check(self._h))


def evaluate_sharded_emulated(shards, box, n_own, pos_ptrs, q_ptrs, u_ptrs, F_ptrs, e_ptrs,
                              stream: int = 0) -> None:
    """All ranks of one decomposition in this process, in lockstep on one GPU
    (esp_shard_evaluate_emulated); per-rank lists of counts and device
    pointers."""
    G = len(shards)
    arr = lambda vals: (C.c_void_p * G)(*[C.c_void_p(v) for v in vals])  # noqa: E731
    hs = (C.c_void_p * G)(*[s._h for s in shards])
    ns = (C.c_long * G)(*[int(v) for v in n_own])
    _check(_lib.esp_shard_evaluate_emulated(hs, G, _f64(box, (3,)), ns, arr(pos_ptrs),
                                            arr(q_ptrs), arr(u_ptrs), arr(F_ptrs), arr(e_ptrs),
                                            C.c_void_p(stream)))
