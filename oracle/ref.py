"""ctypes binding of oracle/_ref/libesp_ref.so -- the unmodified reference
solver (/root/reference/proj/include/esp) compiled by oracle/Makefile.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker and the timed
CPU reference.  The product package never imports this module.

Each function mirrors the reference entry point named in its docstring
(file:line into /root/reference/proj/include/esp) and raises the Python
counterpart of the reference's exception (ValueError for
std::invalid_argument, RefNumericalError for esp::NumericalError).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libesp_ref.so")

_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class RefNumericalError(RuntimeError):
    """esp::NumericalError raised inside the reference (prolate.hpp:17-20)."""


class RefIoError(RuntimeError):
    """esp::IoError (io.hpp:27-30)."""


class _Info(C.Structure):
    _fields_ = [
        ("family", C.c_int), ("window_family", C.c_int), ("force_method", C.c_int),
        ("P", C.c_int), ("nf", C.c_int * 3), ("base_nf", C.c_int * 3),
        ("eps", C.c_double), ("r_c", C.c_double), ("shape", C.c_double), ("c1", C.c_double),
        ("chi0", C.c_double), ("C0_split", C.c_double),
        ("box", C.c_double * 3), ("h", C.c_double * 3), ("demand", C.c_double * 3),
        ("E_A", C.c_double), ("E_T", C.c_double), ("E_SI", C.c_double),
        ("split_ncoef", C.c_int), ("split_nterms", C.c_int), ("win_nterms", C.c_int),
        ("pad", C.c_int),
    ]


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: build it with `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_plan.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_plan_free.argtypes = [C.c_void_p]
        L.ref_plan_info_get.argtypes = [C.c_void_p, C.POINTER(_Info)]
        L.ref_plan_influence.argtypes = [C.c_void_p, _dp]
        L.ref_plan_split_tables.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_plan_prolate_coef.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_plan_window_tables.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.ref_plan_eval_kernels.argtypes = [C.c_void_p, C.c_int, C.c_long, _dp, _dp]
        L.ref_evaluate.argtypes = [C.c_void_p, _dp, C.c_long, _dp, _dp, _dp, _dp,
                                   C.POINTER(C.c_double), _dp]
        L.ref_local_sum.argtypes = [C.c_void_p, _dp, C.c_long, _dp, _dp, _dp, _dp]
        L.ref_spectral_sum.argtypes = [C.c_void_p, _dp, C.c_long, _dp, _dp, _dp, _dp]
        L.ref_self_correction.argtypes = [C.c_void_p, C.c_long, _dp, _dp]
        L.ref_spread.argtypes = [C.c_void_p, C.c_long, _dp, _dp, _dp]
        L.ref_interpolate.argtypes = [C.c_void_p, C.c_long, _dp, _dp, _dp]
        L.ref_interpolate_gradient.argtypes = [C.c_void_p, C.c_long, _dp, _dp, _dp]
        L.ref_fft3.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int]
        L.ref_direct_ewald.argtypes = [_dp, C.c_long, _dp, _dp, C.c_double, _dp, _dp,
                                       C.POINTER(C.c_double), _dp]
        L.ref_relative_force_error.argtypes = [C.c_long, _dp, _dp, C.POINTER(C.c_double)]
        L.ref_generate.argtypes = [C.c_int, C.c_long, _dp, C.c_ulonglong, _dp, _dp]
        L.ref_solve_c.argtypes = [C.c_double, C.POINTER(C.c_double)]
        L.ref_next_even_5smooth.argtypes = [C.c_double, C.POINTER(C.c_int)]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_get_threads.restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RefNumericalError(msg)
    if rc == 3:
        raise RefIoError(msg)
    raise RuntimeError(msg)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int):
    """esp::thread_count() (threads.hpp:14-17)."""
    lib().ref_set_threads(int(n))


def get_threads() -> int:
    return lib().ref_get_threads()


@dataclass
class RefResult:
    energy: float
    u: np.ndarray
    F: np.ndarray
    timings: dict | None = None


class RefPlan:
    """esp::build_plan (ewald.hpp:355-405) held by the reference itself."""

    def __init__(self, box, family="pswf", eps=1e-4, r_c=1.0, nf=0, P=0, c1=0.0,
                 force_method="ik", allow_degraded=False):
        h = C.c_void_p()
        _check(lib().ref_build_plan(_f64(box), 1 if family == "gaussian" else 0, float(eps),
                                    float(r_c), int(nf), int(P), float(c1),
                                    1 if force_method == "ad" else 0, int(bool(allow_degraded)),
                                    C.byref(h)))
        self._h = h
        info = _Info()
        _check(lib().ref_plan_info_get(self._h, C.byref(info)))
        self.info = info
        self.nf = tuple(info.nf)
        self.base_nf = tuple(info.base_nf)
        self.P = info.P
        self.shape = info.shape
        self.c1 = info.c1
        self.box = tuple(info.box)
        self.h = tuple(info.h)
        self.demand = tuple(info.demand)
        self.eps = info.eps
        self.r_c = info.r_c
        self.chi0 = info.chi0
        self.E_A, self.E_T, self.E_SI = info.E_A, info.E_T, info.E_SI

    def __del__(self):
        try:
            if self._h:
                lib().ref_plan_free(self._h)
        except Exception:
            pass

    # ---- plan tables -------------------------------------------------------
    def influence(self) -> np.ndarray:
        out = np.empty(int(np.prod(self.nf)), dtype=np.float64)
        _check(lib().ref_plan_influence(self._h, out))
        return out.reshape(self.nf)

    def split_tables(self):
        psi = np.empty(16 * 13)
        chi = np.empty(16 * 13)
        geom = np.empty(5)
        _check(lib().ref_plan_split_tables(self._h, psi, chi, geom))
        return psi.reshape(16, 13), chi.reshape(16, 13), geom

    def window_tables(self, d: int):
        n = 4 * self.P
        phi = np.empty(n * 13)
        dphi = np.empty(n * 13)
        geom = np.empty(5)
        _check(lib().ref_plan_window_tables(self._h, int(d), phi, dphi, geom))
        return phi.reshape(n, 13), dphi.reshape(n, 13), geom

    def prolate_coef(self, which: int = -1) -> np.ndarray:
        n = self.info.split_nterms if which < 0 else self.info.win_nterms
        out = np.empty(n)
        _check(lib().ref_plan_prolate_coef(self._h, int(which), out))
        return out

    def eval_kernel(self, what: str, x) -> np.ndarray:
        sel = {"Psi": 0, "chi": 1, "chihat_n": 2, "phi": 3, "dphi": 4, "phi_hat": 5,
               "local_pot": 6, "local_fr": 7}[what]
        x = _f64(np.atleast_1d(x))
        y = np.empty_like(x)
        _check(lib().ref_plan_eval_kernels(self._h, sel, x.size, x, y))
        return y

    # ---- hot path ----------------------------------------------------------
    def evaluate(self, pos, q, box=None) -> RefResult:
        """esp::evaluate (ewald.hpp:619-649)."""
        pos = _f64(pos).reshape(-1, 3)
        q = _f64(q)
        N = q.size
        u = np.empty(N)
        F = np.empty((N, 3))
        e = C.c_double()
        t = np.empty(6)
        _check(lib().ref_evaluate(self._h, _f64(box if box is not None else self.box), N, pos,
                                  q, u, F, C.byref(e), t))
        keys = ["local", "spread", "fft", "scale", "ifft", "interpolate"]
        return RefResult(e.value, u, F, dict(zip(keys, t.tolist())))

    def local_sum(self, pos, q, box=None):
        """esp::local_sum (ewald.hpp:419-515)."""
        pos = _f64(pos).reshape(-1, 3)
        q = _f64(q)
        u = np.empty(q.size)
        F = np.empty((q.size, 3))
        _check(lib().ref_local_sum(self._h, _f64(box if box is not None else self.box), q.size,
                                   pos, q, u, F))
        return u, F

    def spectral_sum(self, pos, q, box=None):
        """esp::spectral_sum (ewald.hpp:524-604)."""
        pos = _f64(pos).reshape(-1, 3)
        q = _f64(q)
        u = np.empty(q.size)
        F = np.empty((q.size, 3))
        _check(lib().ref_spectral_sum(self._h, _f64(box if box is not None else self.box),
                                      q.size, pos, q, u, F))
        return u, F

    def self_correction(self, q):
        q = _f64(q)
        out = np.empty_like(q)
        _check(lib().ref_self_correction(self._h, q.size, q, out))
        return out

    def spread(self, pos, q) -> np.ndarray:
        """esp::spread (gridder.hpp:215-241), real part."""
        pos = _f64(pos).reshape(-1, 3)
        q = _f64(q)
        g = np.empty(int(np.prod(self.nf)))
        _check(lib().ref_spread(self._h, q.size, pos, q, g))
        return g.reshape(self.nf)

    def interpolate(self, pos, grid) -> np.ndarray:
        """esp::interpolate (gridder.hpp:244-277) of a real grid."""
        pos = _f64(pos).reshape(-1, 3)
        out = np.empty(pos.shape[0])
        _check(lib().ref_interpolate(self._h, pos.shape[0], pos, _f64(grid).ravel(), out))
        return out

    def interpolate_gradient(self, pos, grid) -> np.ndarray:
        """esp::interpolate_gradient (gridder.hpp:280-314)."""
        pos = _f64(pos).reshape(-1, 3)
        out = np.empty((pos.shape[0], 3))
        _check(lib().ref_interpolate_gradient(self._h, pos.shape[0], pos, _f64(grid).ravel(),
                                              out))
        return out


def direct_ewald(pos, q, box, tol=1e-9) -> RefResult:
    """esp::direct_ewald (reference.hpp:212-238); N <= 1e4."""
    pos = _f64(pos).reshape(-1, 3)
    q = _f64(q)
    u = np.empty(q.size)
    F = np.empty((q.size, 3))
    e = C.c_double()
    info = np.empty(4)
    _check(lib().ref_direct_ewald(_f64(box), q.size, pos, q, float(tol), u, F, C.byref(e),
                                  info))
    r = RefResult(e.value, u, F)
    r.info = dict(zip(["lambda", "real_shells", "recip_kmax", "residual"], info.tolist()))
    return r


def relative_force_error(test, ref) -> float:
    """esp::relative_force_error (reference.hpp:241-255)."""
    t = _f64(test).reshape(-1, 3)
    r = _f64(ref).reshape(-1, 3)
    out = C.c_double()
    _check(lib().ref_relative_force_error(t.shape[0], t, r, C.byref(out)))
    return out.value


def generate(kind: str, N: int, box, seed: int = 1):
    """esp::generate_system (io.hpp:82-148)."""
    k = {"random": 0, "rocksalt": 1, "water-like": 2}[kind]
    pos = np.empty((N, 3))
    q = np.empty(N)
    _check(lib().ref_generate(k, int(N), _f64(box), C.c_ulonglong(seed), pos, q))
    return pos, q


def fft3(data: np.ndarray, sign: int) -> np.ndarray:
    """gridder.hpp fft_forward (sign<0) / fft_inverse (sign>0) via the FFTW shim."""
    a = np.ascontiguousarray(data, dtype=np.complex128)
    buf = a.view(np.float64).ravel().copy()
    _check(lib().ref_fft3(a.shape[0], a.shape[1], a.shape[2], buf, int(sign)))
    return buf.view(np.complex128).reshape(a.shape)


def solve_c(eps: float) -> float:
    """esp::solve_c (prolate.hpp:254-263)."""
    out = C.c_double()
    _check(lib().ref_solve_c(float(eps), C.byref(out)))
    return out.value


def next_even_5smooth(x: float) -> int:
    out = C.c_int()
    _check(lib().ref_next_even_5smooth(float(x), C.byref(out)))
    return out.value
