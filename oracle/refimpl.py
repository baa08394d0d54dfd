"""ctypes binding of oracle/_ref/libfse_ref.so -- TEST INFRASTRUCTURE.

The library is the UNMODIFIED reference (/root/reference/proj/src/*.cpp)
compiled by oracle/Makefile against the FFTW shim, plus the marshalling shims
of oracle/ref_capi.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
package never does.

Kinds: 0 stokeslet, 1 stresslet, 2 rotlet (fse::KernelKind order,
/root/reference/proj/include/fse/kernels.hpp:16).  Green kinds: 0 harmonic,
1 biharmonic (greens.hpp:19).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libfse_ref.so")

STOKESLET, STRESSLET, ROTLET = 0, 1, 2
HARMONIC, BIHARMONIC = 0, 1

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

_lib = None


class RefError(Exception):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


class RefDomainError(RefError, ArithmeticError):
    pass


class RefRuntimeError(RefError, RuntimeError):
    pass


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"{LIB_PATH} not built (make -C oracle ref)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    raise {1: RefInvalidArgument, 2: RefDomainError, 3: RefRuntimeError}.get(rc, RefError)(msg)


def arity(kind: int) -> int:
    return 9 if kind == STRESSLET else 3


def green_kind_for(kind: int) -> int:
    return HARMONIC if kind == ROTLET else BIHARMONIC


@dataclass
class Cfg:
    """fse::EwaldConfig fields (ewald.hpp:16-35)."""

    L: float
    xi: float
    rc: float
    M: int
    P: int
    h: float
    d: float
    m: float
    eta: float
    deltaL: float
    Ltilde: float
    Mtilde: int
    kinf: float
    R: float
    sf: float
    deterministic: bool = False

    @property
    def D(self) -> int:
        return 2 * self.Mtilde

    def args(self):
        return (self.L, self.xi, self.rc, self.M, self.P, self.sf)


def _cfg_from(v) -> Cfg:
    return Cfg(v[0], v[1], v[2], int(v[3]), int(v[4]), v[5], v[6], v[7], v[8], v[9], v[10],
               int(v[11]), v[12], v[13], v[14], bool(v[15]))


def set_threads(n: int):
    lib().ref_set_threads(C.c_int(n))


def max_threads() -> int:
    return lib().ref_max_threads()


def make_config(L, xi, rc, M, P, sf=0.0) -> Cfg:
    out = np.zeros(16)
    f = lib().ref_make_config
    f.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, _dp]
    _check(f(L, xi, rc, M, P, sf, out))
    return _cfg_from(out)


def _a(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def build_cell_list(pos, L, rc, pad=0.0):
    pos = _a(pos)
    n = pos.shape[0]
    dims = np.zeros(3, np.int32)
    cs = C.c_double()
    org = C.c_double()
    f = lib().ref_build_cell_list
    f.argtypes = [_dp, C.c_int64, C.c_double, C.c_double, C.c_double, _i32p,
                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
    _check(f(pos, n, L, rc, pad, dims, C.byref(cs), C.byref(org), None, None))
    ncell = int(dims[0]) * int(dims[1]) * int(dims[2])
    bstart = np.zeros(ncell + 1, np.int64)
    perm = np.zeros(max(n, 1), np.int64)
    _check(f(pos, n, L, rc, pad, dims, C.byref(cs), C.byref(org),
             bstart.ctypes.data_as(C.c_void_p), perm.ctypes.data_as(C.c_void_p)))
    return dict(dims=dims.copy(), cell_side=cs.value, origin=org.value, bstart=bstart,
                perm=perm[:n])


def real_space_sum(kind, pos, strengths, L, xi, rc, targets):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    f = lib().ref_real_space_sum
    f.argtypes = [C.c_int, _dp, _dp, C.c_int64, C.c_double, C.c_double, C.c_double, _dp,
                  C.c_int64, _dp]
    _check(f(kind, pos, strengths, pos.shape[0], L, xi, rc, targets, targets.shape[0], u))
    return u


def eval_real_kernel(kind, r, xi, f_):
    out = np.zeros(3)
    f = lib().ref_eval_real_kernel
    f.argtypes = [C.c_int, _dp, C.c_double, _dp, _dp]
    _check(f(kind, _a(r), xi, _a(f_), out))
    return out


def eval_kernel(kind, r, f_):
    out = np.zeros(3)
    f = lib().ref_eval_kernel
    f.argtypes = [C.c_int, _dp, _dp, _dp]
    _check(f(kind, _a(r), _a(f_), out))
    return out


def spread(cfg: Cfg, kind, pos, strengths, use_fgg=True, deterministic=False):
    pos, strengths = _a(pos), _a(strengths)
    Mt = cfg.Mtilde
    grid = np.zeros((arity(kind), Mt, Mt, Mt))
    f = lib().ref_spread
    f.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                  C.c_int, _dp, _dp, C.c_int64, C.c_int, _dp]
    _check(f(*cfg.args(), int(deterministic), kind, pos, strengths, pos.shape[0],
             int(use_fgg), grid))
    return grid


def kspace_scale(cfg: Cfg, kind, green_fourier, ghat):
    """ghat: (arity, D, D, D) complex128.  Returns (3, D, D, D) complex128."""
    D = cfg.D
    ghat = np.ascontiguousarray(ghat, dtype=np.complex128)
    out = np.zeros((3, D, D, D), np.complex128)
    f = lib().ref_kspace_scale
    f.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                  _dp, C.c_void_p, C.c_void_p]
    _check(f(*cfg.args(), kind, _a(green_fourier).reshape(-1), ghat.ctypes.data_as(C.c_void_p),
             out.ctypes.data_as(C.c_void_p)))
    return out


def _sum(fn, cfg: Cfg, kind, pos, strengths, targets, green_fourier, timings=None):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    t = np.zeros(7)
    fn.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                   _dp, _dp, C.c_int64, _dp, C.c_int64, _dp, _dp, _dp]
    _check(fn(*cfg.args(), kind, pos, strengths, pos.shape[0], targets, targets.shape[0],
              _a(green_fourier).reshape(-1), u, t))
    if timings is not None:
        timings.update(dict(zip(["precompute", "spread", "fft", "scale", "quadrature",
                                 "realspace", "total"], t.tolist())))
    return u


def fourier_sum(cfg, kind, pos, strengths, targets, green_fourier, timings=None):
    return _sum(lib().ref_fourier_sum, cfg, kind, pos, strengths, targets, green_fourier,
                timings)


def total_sum(cfg, kind, pos, strengths, targets, green_fourier, timings=None):
    return _sum(lib().ref_total_sum, cfg, kind, pos, strengths, targets, green_fourier, timings)


def precompute_green(gkind, Ltilde, Mtilde, sf):
    D = 2 * Mtilde
    out = np.zeros((D, D, D))
    f = lib().ref_precompute_green
    f.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, _dp]
    _check(f(gkind, Ltilde, Mtilde, sf, out))
    return out


def hhat(k, R):
    out = C.c_double()
    f = lib().ref_hhat
    f.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
    _check(f(k, R, C.byref(out)))
    return out.value


def bhat(k, R):
    out = C.c_double()
    f = lib().ref_bhat
    f.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
    _check(f(k, R, C.byref(out)))
    return out.value


def save_green(gkind, Ltilde, Mtilde, sf, path):
    f = lib().ref_save_green
    f.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_char_p]
    _check(f(gkind, Ltilde, Mtilde, sf, path.encode()))


def load_green(path):
    """load_mollified_green (greens.cpp:173-203): (kind, Ltilde, h, R, Mtilde, table)."""
    f = lib().ref_load_green
    gk, Mt = C.c_int(), C.c_int()
    Lt, h, R = C.c_double(), C.c_double(), C.c_double()
    f.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double),
                  C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p]
    _check(f(path.encode(), C.byref(gk), C.byref(Lt), C.byref(h), C.byref(R), C.byref(Mt), None))
    D = 2 * Mt.value
    out = np.zeros((D, D, D))
    _check(f(path.encode(), C.byref(gk), C.byref(Lt), C.byref(h), C.byref(R), C.byref(Mt),
             out.ctypes.data_as(C.c_void_p)))
    return gk.value, Lt.value, h.value, R.value, Mt.value, out


def direct_sum(kind, pos, strengths, L, targets, exclude_self):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    f = lib().ref_direct_sum
    f.argtypes = [C.c_int, _dp, _dp, C.c_int64, C.c_double, _dp, C.c_int64, C.c_int, _dp]
    _check(f(kind, pos, strengths, pos.shape[0], L, targets, targets.shape[0],
             int(exclude_self), u))
    return u


def error_budget(kind, L, xi, rc, M, P, Q):
    a, b = C.c_double(), C.c_double()
    f = lib().ref_error_budget
    f.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
    _check(f(kind, L, xi, rc, M, P, Q, C.byref(a), C.byref(b)))
    return a.value, b.value


def select_parameters(kind, n, L, Q, xi, tol):
    out = np.zeros(16)
    feas = C.c_int()
    f = lib().ref_select_parameters
    f.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, _dp,
                  C.POINTER(C.c_int)]
    _check(f(kind, n, L, Q, xi, tol, out, C.byref(feas)))
    return _cfg_from(out), bool(feas.value)


def generate_system(kind, n, L, seed):
    pos = np.zeros((n, 3))
    st = np.zeros((n, arity(kind)))
    f = lib().ref_generate_system
    f.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_uint64, _dp, _dp]
    _check(f(kind, n, L, seed, pos, st))
    return pos, st


def generate_workload(which, n, seed):
    """SURVEY 8(d) workload streams (ref_capi.cpp ref_generate_workload):
    returns (positions, strengths, targets or None)."""
    a = 9 if which == 3 else 3
    pos = np.zeros((n, 3))
    st = np.zeros((n, a))
    tgt = np.zeros((n, 3)) if which == 5 else np.zeros((1, 3))
    f = lib().ref_generate_workload
    f.argtypes = [C.c_int, C.c_int64, C.c_uint64, _dp, _dp, _dp]
    _check(f(which, n, seed, pos, st, tgt))
    return pos, st, (tgt if which == 5 else None)


def fft3d(data, inverse=False):
    d = np.ascontiguousarray(data, dtype=np.complex128).copy()
    f = lib().ref_fft3d
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
    n0, n1, n2 = d.shape
    _check(f(d.ctypes.data_as(C.c_void_p), n0, n1, n2, int(inverse)))
    return d
