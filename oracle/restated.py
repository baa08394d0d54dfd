"""ctypes binding of oracle/build/libfse_oracle.so -- TEST INFRASTRUCTURE.

The plain-C restatement of the reference hot path (oracle/fse_oracle.c).  It
is the parity CHECKER for the CUDA product; only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.
Same call surface as oracle/refimpl.py so tests can run either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .refimpl import (BIHARMONIC, HARMONIC, ROTLET, STOKESLET, STRESSLET, Cfg, arity,
                      green_kind_for)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libfse_oracle.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

__all__ = ["STOKESLET", "STRESSLET", "ROTLET", "HARMONIC", "BIHARMONIC", "arity",
           "green_kind_for", "make_config"]


class _OrCfg(C.Structure):
    _fields_ = [("L", C.c_double), ("xi", C.c_double), ("rc", C.c_double), ("M", C.c_int),
                ("P", C.c_int), ("h", C.c_double), ("d", C.c_double), ("m", C.c_double),
                ("eta", C.c_double), ("deltaL", C.c_double), ("Ltilde", C.c_double),
                ("Mtilde", C.c_int), ("kinf", C.c_double), ("R", C.c_double),
                ("sf", C.c_double), ("deterministic", C.c_int)]


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class OracleDomainError(OracleError, ArithmeticError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", HERE, "restated"], check=True)
        _lib = C.CDLL(LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        _lib.or_hhat.restype = C.c_double
        _lib.or_hhat.argtypes = [C.c_double, C.c_double]
        _lib.or_bhat.restype = C.c_double
        _lib.or_bhat.argtypes = [C.c_double, C.c_double]
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    raise {1: OracleInvalidArgument, 2: OracleDomainError}.get(rc, OracleError)(msg)


def _a(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _c(cfg: Cfg) -> _OrCfg:
    return _OrCfg(cfg.L, cfg.xi, cfg.rc, cfg.M, cfg.P, cfg.h, cfg.d, cfg.m, cfg.eta,
                  cfg.deltaL, cfg.Ltilde, cfg.Mtilde, cfg.kinf, cfg.R, cfg.sf,
                  int(cfg.deterministic))


def make_config(L, xi, rc, M, P, sf=0.0) -> Cfg:
    o = _OrCfg()
    f = lib().or_make_config
    f.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                  C.POINTER(_OrCfg)]
    _check(f(L, xi, rc, M, P, sf, C.byref(o)))
    return Cfg(o.L, o.xi, o.rc, o.M, o.P, o.h, o.d, o.m, o.eta, o.deltaL, o.Ltilde, o.Mtilde,
               o.kinf, o.R, o.sf, bool(o.deterministic))


def build_cell_list(pos, L, rc, pad=0.0):
    pos = _a(pos)
    n = pos.shape[0]
    dims = np.zeros(3, np.int32)
    cs, org = C.c_double(), C.c_double()
    f = lib().or_build_cell_list
    f.argtypes = [_dp, C.c_int64, C.c_double, C.c_double, C.c_double, _i32p,
                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
    _check(f(pos, n, L, rc, pad, dims, C.byref(cs), C.byref(org), None, None))
    ncell = int(np.prod(dims.astype(np.int64)))
    bstart = np.zeros(ncell + 1, np.int64)
    perm = np.zeros(max(n, 1), np.int64)
    _check(f(pos, n, L, rc, pad, dims, C.byref(cs), C.byref(org),
             bstart.ctypes.data_as(C.c_void_p), perm.ctypes.data_as(C.c_void_p)))
    return dict(dims=dims.copy(), cell_side=cs.value, origin=org.value, bstart=bstart,
                perm=perm[:n])


def eval_real_kernel(kind, r, xi, f_):
    out = np.zeros(3)
    f = lib().or_eval_real_kernel
    f.argtypes = [C.c_int, _dp, C.c_double, _dp, _dp]
    _check(f(kind, _a(r), xi, _a(f_), out))
    return out


def eval_kernel(kind, r, f_):
    out = np.zeros(3)
    f = lib().or_eval_kernel
    f.argtypes = [C.c_int, _dp, _dp, _dp]
    _check(f(kind, _a(r), _a(f_), out))
    return out


def real_space_sum(kind, pos, strengths, L, xi, rc, targets):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    f = lib().or_real_space_sum
    f.argtypes = [C.c_int, _dp, _dp, C.c_int64, C.c_double, C.c_double, C.c_double, _dp,
                  C.c_int64, _dp]
    _check(f(kind, pos, strengths, pos.shape[0], L, xi, rc, targets, targets.shape[0], u))
    return u


def support(cfg: Cfg, x, use_fgg=True):
    i0 = np.zeros(3, np.int32)
    w = np.zeros(3 * cfg.P)
    f = lib().or_support
    f.argtypes = [C.POINTER(_OrCfg), _dp, C.c_int, _i32p, _dp]
    c = _c(cfg)
    rc = f(C.byref(c), _a(x), int(use_fgg), i0, w)
    return i0, w.reshape(3, cfg.P), rc == 0


def support_index(cfg: Cfg, pts):
    """i0 of every point (n, 3) int32 (or_support_index)."""
    pts = _a(pts).reshape(-1, 3)
    i0 = np.zeros((pts.shape[0], 3), np.int32)
    f = lib().or_support_index
    f.restype = C.c_int64
    f.argtypes = [C.POINTER(_OrCfg), _dp, C.c_int64, _i32p]
    c = _c(cfg)
    f(C.byref(c), pts, pts.shape[0], i0)
    return i0


def spread(cfg: Cfg, kind, pos, strengths, use_fgg=True, box_side=None):
    pos, strengths = _a(pos), _a(strengths)
    Mt = cfg.Mtilde
    grid = np.zeros((arity(kind), Mt, Mt, Mt))
    f = lib().or_spread
    f.argtypes = [C.POINTER(_OrCfg), C.c_int, _dp, _dp, C.c_int64, C.c_double, C.c_int, _dp]
    c = _c(cfg)
    _check(f(C.byref(c), kind, pos, strengths, pos.shape[0],
             cfg.L if box_side is None else box_side, int(use_fgg), grid))
    return grid


def kspace_scale(cfg: Cfg, kind, green_fourier, ghat):
    D = cfg.D
    ghat = np.ascontiguousarray(ghat, dtype=np.complex128)
    out = np.zeros((3, D, D, D), np.complex128)
    f = lib().or_kspace_scale
    f.argtypes = [C.POINTER(_OrCfg), C.c_int, _dp, C.c_void_p, C.c_void_p]
    c = _c(cfg)
    _check(f(C.byref(c), kind, _a(green_fourier).reshape(-1), ghat.ctypes.data_as(C.c_void_p),
             out.ctypes.data_as(C.c_void_p)))
    return out


def fourier_sum(cfg, kind, pos, strengths, targets, green_fourier, return_w=False,
                box_side=None):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    Mt = cfg.Mtilde
    w = np.zeros((3, Mt, Mt, Mt)) if return_w else None
    f = lib().or_fourier_sum
    f.argtypes = [C.POINTER(_OrCfg), C.c_int, _dp, _dp, C.c_int64, C.c_double, _dp, C.c_int64,
                  _dp, _dp, C.c_void_p]
    c = _c(cfg)
    _check(f(C.byref(c), kind, pos, strengths, pos.shape[0],
             cfg.L if box_side is None else box_side, targets, targets.shape[0],
             _a(green_fourier).reshape(-1), u,
             w.ctypes.data_as(C.c_void_p) if return_w else None))
    return (u, w) if return_w else u


def total_sum(cfg, kind, pos, strengths, targets, green_fourier, box_side=None):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    f = lib().or_total_sum
    f.argtypes = [C.POINTER(_OrCfg), C.c_int, _dp, _dp, C.c_int64, C.c_double, _dp, C.c_int64,
                  _dp, _dp]
    c = _c(cfg)
    _check(f(C.byref(c), kind, pos, strengths, pos.shape[0],
             cfg.L if box_side is None else box_side, targets, targets.shape[0],
             _a(green_fourier).reshape(-1), u))
    return u


def hhat(k, R):
    return lib().or_hhat(k, R)


def bhat(k, R):
    return lib().or_bhat(k, R)


def precompute_green(gkind, Ltilde, Mtilde, sf):
    D = 2 * Mtilde
    out = np.zeros((D, D, D))
    f = lib().or_precompute_green
    f.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, _dp]
    _check(f(gkind, Ltilde, Mtilde, sf, out))
    return out


def direct_sum(kind, pos, strengths, targets, exclude_self):
    pos, strengths, targets = _a(pos), _a(strengths), _a(targets)
    u = np.zeros((targets.shape[0], 3))
    f = lib().or_direct_sum
    f.argtypes = [C.c_int, _dp, _dp, C.c_int64, _dp, C.c_int64, C.c_int, _dp]
    _check(f(kind, pos, strengths, pos.shape[0], targets, targets.shape[0], int(exclude_self),
             u))
    return u


def fft3d(data, inverse=False):
    d = np.ascontiguousarray(data, dtype=np.complex128).copy()
    f = lib().or_fft3d
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
    n0, n1, n2 = d.shape
    f(d.ctypes.data_as(C.c_void_p), n0, n1, n2, int(inverse))
    return d
