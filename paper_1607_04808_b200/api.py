"""Python mirror of the reference's fse:: hot-path API over the C-ABI.

Names, argument order, argument meaning and error behaviour follow the
reference C++ library (/root/reference/proj/include/fse/*.hpp):

    make_config(L, xi, rc, M, P, sf=0)                      ewald.hpp:37
    precompute_mollified_green(kind, Ltilde, Mtilde, sf)     greens.hpp:71-72
    spread(system, cfg, kind)                                ewald.hpp:45-46
    kspace_scale(ghat, cfg, kind, green)                     ewald.hpp:51-53
    fourier_sum(system, cfg, kind, targets, green, timings)  ewald.hpp:69-71
    total_sum(system, kind, cfg, targets, green, timings)    ewald.hpp:75-77
    real_space_sum(system, kind, xi, rc, targets)            realspace.hpp:35-36
    build_cell_list(system, rc, domain_pad=0)                realspace.hpp:31
    direct_sum(system, kind, targets, exclude_self)          kernels.hpp:78-79
    fft3d_forward / fft3d_inverse                            fft.hpp:11,14
    save_mollified_green / load_mollified_green              greens.hpp:79-80

std::invalid_argument -> InvalidArgument (a ValueError), std::domain_error ->
DomainError (an ArithmeticError), everything else -> FseRuntimeError.

All computation runs in libfse_b200.so on the GPU (sm_100a); there is no CPU
fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSE_LIB_PATH: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("FSE_LIB_PATH") or os.path.join(_HERE, "libfse_b200.so")


class FseError(Exception):
    pass


class InvalidArgument(FseError, ValueError):
    """std::invalid_argument"""


class DomainError(FseError, ArithmeticError):
    """std::domain_error"""


class FseRuntimeError(FseError, RuntimeError):
    """std::runtime_error (I/O) and CUDA / cuFFT / allocation failures"""


class KernelKind(enum.IntEnum):  # kernels.hpp:16
    Stokeslet = 0
    Stresslet = 1
    Rotlet = 2


class GreenKind(enum.IntEnum):  # greens.hpp:19
    Harmonic = 0
    Biharmonic = 1


def strength_arity(kind) -> int:  # kernels.hpp:19-21
    return 9 if int(kind) == KernelKind.Stresslet else 3


def green_kind_for(kind) -> GreenKind:  # ewald.hpp:80-82
    return GreenKind.Harmonic if int(kind) == KernelKind.Rotlet else GreenKind.Biharmonic


class EwaldConfig(C.Structure):
    """Bitwise mirror of fse::EwaldConfig (ewald.hpp:16-35) / fse_config."""

    _fields_ = [("L", C.c_double), ("xi", C.c_double), ("rc", C.c_double), ("M", C.c_int32),
                ("P", C.c_int32), ("h", C.c_double), ("d", C.c_double), ("m", C.c_double),
                ("eta", C.c_double), ("deltaL", C.c_double), ("Ltilde", C.c_double),
                ("Mtilde", C.c_int32), ("_pad0", C.c_int32), ("kinf", C.c_double),
                ("R", C.c_double), ("sf", C.c_double), ("deterministic", C.c_uint8),
                ("_pad1", C.c_uint8 * 7)]

    @property
    def D(self) -> int:
        return 2 * self.Mtilde

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}

    def __repr__(self):
        return "EwaldConfig(" + ", ".join(f"{k}={v!r}" for k, v in self.as_dict().items()) + ")"


assert C.sizeof(EwaldConfig) == 120


class StageTimings(C.Structure):
    """Mirror of fse::StageTimings (ewald.hpp:56-64), seconds; calls accumulate."""

    _fields_ = [(k, C.c_double) for k in
                ("precompute", "spread", "fft", "scale", "quadrature", "realspace", "total")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ErrorBudget(C.Structure):
    """fse::ErrorBudget (estimates.hpp:11-17): predicted RMS truncation errors."""
    _fields_ = [("kind", C.c_int), ("xi", C.c_double), ("rc", C.c_double),
                ("k_inf", C.c_double), ("L", C.c_double), ("R", C.c_double), ("Q", C.c_double),
                ("predicted_real_rms", C.c_double), ("predicted_fourier_rms", C.c_double)]


def _est(fn, *args):
    v = C.c_double()
    st = fn(*args, C.byref(v))
    if st != 0:
        _raise(st, f"{fn.__name__}: bad arguments")
    return v.value


def fourier_error_estimate(kind, Q, xi, k_inf, L, R) -> float:  # estimates.cpp:14-29
    return _est(_load().fse_fourier_error_estimate, int(kind), float(Q), float(xi),
                float(k_inf), float(L), float(R))


def real_error_estimate(kind, Q, xi, rc, L) -> float:  # estimates.cpp:31-47
    return _est(_load().fse_real_error_estimate, int(kind), float(Q), float(xi), float(rc),
                float(L))


def reference_velocity_rms(kind, Q, L, N) -> float:  # estimates.cpp:64-79
    return _est(_load().fse_reference_velocity_rms, int(kind), float(Q), float(L), int(N))


def error_budget(kind, cfg, Q) -> ErrorBudget:  # estimates.cpp:49-62
    b = ErrorBudget()
    st = _load().fse_error_budget(int(kind), C.byref(cfg), float(Q), C.byref(b))
    if st != 0:
        _raise(st, "error_budget: bad arguments")
    return b


def select_parameters(kind, N, L, Q, xi, tol):  # estimates.cpp:81-126
    """-> (EwaldConfig, feasible)"""
    cfg = EwaldConfig()
    feas = C.c_int()
    st = _load().fse_select_parameters(int(kind), int(N), float(L), float(Q), float(xi),
                                       float(tol), C.byref(cfg), C.byref(feas))
    if st != 0:
        _raise(st, "select_parameters: bad arguments or no feasible grid size")
    return cfg, bool(feas.value)


class SlabInfo(C.Structure):
    """fse_slab_info (include/fse_cuda.h): this rank's part of the z-slab decomposition."""
    _fields_ = [("x_lo", C.c_int), ("nx", C.c_int), ("nxs", C.c_int), ("ky_lo", C.c_int),
                ("nky", C.c_int), ("nkys", C.c_int), ("block_complex", C.c_int64)]


def slab_info(cfg, kind, rank, nslabs) -> SlabInfo:
    out = SlabInfo()
    st = _load().fse_cuda_slab_info(C.byref(cfg), int(kind), int(rank), int(nslabs),
                                    C.byref(out))
    if st != 0:
        _raise(st, "fse_cuda_slab_info: invalid slab request (P <= 25 needed for nslabs > 1)")
    return out


@dataclass
class SourceSystem:
    """fse::SourceSystem (kernels.hpp:59-66): positions (N,3), strengths (N,a)."""

    positions: np.ndarray
    strengths: np.ndarray
    box_side: float = 1.0

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1, 3)
        s = np.ascontiguousarray(self.strengths, dtype=np.float64)
        self.strengths = s.reshape(self.positions.shape[0], -1) if s.size else s.reshape(0, 3)

    def size(self) -> int:
        return self.positions.shape[0]


@dataclass
class CellList:
    """fse::CellList (realspace.hpp:14-24) in bucket-contiguous form:
    bucket b holds perm[bstart[b]:bstart[b+1]] (ascending source indices)."""

    cell_side: float
    origin: float
    dims: tuple
    bstart: np.ndarray
    perm: np.ndarray

    @property
    def buckets(self):
        return [self.perm[self.bstart[b]:self.bstart[b + 1]].tolist()
                for b in range(len(self.bstart) - 1)]

    def cell_of(self, coord: float, axis: int) -> int:  # realspace.cpp:60-63
        c = int(np.floor((coord - self.origin) / self.cell_side))
        return min(max(c, 0), self.dims[axis] - 1)


# --------------------------------------------------------------------- library
_dp = C.POINTER(C.c_double)
_lib = None
_lib_lock = threading.Lock()


def library_path() -> str:
    return LIB_PATH


def _load():
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        i64 = C.c_int64
        lib.fse_cuda_last_error.restype = C.c_char_p
        lib.fse_cuda_last_error.argtypes = [vp]
        lib.fse_cuda_create.argtypes = [C.c_int, C.POINTER(vp)]
        lib.fse_cuda_destroy.argtypes = [vp]
        lib.fse_cuda_launch_count.restype = C.c_uint64
        lib.fse_cuda_launch_count.argtypes = [vp]
        lib.fse_make_config.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_double, C.POINTER(EwaldConfig), C.c_char_p, C.c_size_t]
        lib.fse_cuda_green_precompute.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_double,
                                                  C.POINTER(vp)]
        lib.fse_cuda_green_upload.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_double,
                                              C.c_double, _dp, C.POINTER(vp)]
        lib.fse_cuda_green_download.argtypes = [vp, vp, _dp]
        lib.fse_cuda_green_info.argtypes = [vp, C.POINTER(C.c_int), _dp, _dp, _dp,
                                            C.POINTER(C.c_int)]
        lib.fse_cuda_green_free.argtypes = [vp]
        lib.fse_cuda_green_save.argtypes = [vp, vp, C.c_char_p]
        lib.fse_cuda_green_load.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
        lib.fse_cuda_total_sum.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, _dp, _dp, i64,
                                           C.c_double, _dp, i64, C.c_int, vp, _dp,
                                           C.POINTER(StageTimings)]
        lib.fse_cuda_total_sum_dev.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, vp, i64,
                                               C.c_double, vp, i64, C.c_int, vp, vp,
                                               C.POINTER(StageTimings)]
        lib.fse_cuda_fourier_sum.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, _dp, _dp, i64,
                                             C.c_double, _dp, i64, vp, _dp,
                                             C.POINTER(StageTimings)]
        lib.fse_cuda_real_space_sum.argtypes = [vp, C.c_int, _dp, _dp, i64, C.c_double,
                                                C.c_double, C.c_double, _dp, i64, _dp]
        lib.fse_cuda_spread.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, _dp, _dp, i64,
                                        C.c_double, _dp]
        lib.fse_cuda_spread_ex.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, _dp, _dp, i64,
                                           C.c_double, C.c_int, _dp]
        lib.fse_cuda_kspace_scale.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, _dp, _dp]
        lib.fse_cuda_build_cell_list.argtypes = [vp, _dp, i64, C.c_double, C.c_double,
                                                 C.c_double, C.POINTER(C.c_int), _dp, _dp,
                                                 C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.fse_cuda_support_index.argtypes = [vp, C.POINTER(EwaldConfig), _dp, i64,
                                               C.POINTER(C.c_int32)]
        lib.fse_cuda_direct_sum.argtypes = [vp, C.c_int, _dp, _dp, i64, _dp, i64, C.c_int, _dp]
        lib.fse_cuda_fft3d.argtypes = [vp, _dp, C.c_int, C.c_int, C.c_int, C.c_int]
        lib.fse_cuda_fft_columns.argtypes = [vp, C.c_int, C.c_int, _dp, C.c_int]
        lib.fse_cuda_nccl_unique_id.argtypes = [vp]
        lib.fse_cuda_dist_create.argtypes = [vp, C.c_int, C.c_int, vp, C.POINTER(vp)]
        lib.fse_cuda_dist_destroy.argtypes = [vp]
        lib.fse_cuda_dist_total_sum.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, vp, i64,
                                                i64, vp, i64, C.c_int, vp, vp]
        lib.fse_cuda_dist_virtual_total_sum.argtypes = [vp, C.c_int, C.POINTER(EwaldConfig),
                                                        C.c_int, vp, vp, i64, vp, i64, C.c_int,
                                                        vp, vp, vp]
        lib.fse_cuda_multi_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
        lib.fse_cuda_multi_destroy.argtypes = [vp]
        lib.fse_cuda_multi_last_error.restype = C.c_char_p
        lib.fse_cuda_multi_last_error.argtypes = [vp]
        lib.fse_cuda_multi_total_sum.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, _dp, _dp, i64,
                                                 C.c_double, _dp, i64, C.c_int, vp, _dp,
                                                 C.POINTER(StageTimings)]
        lib.fse_dist_owner.argtypes = [C.POINTER(EwaldConfig), C.c_int, _dp, i64,
                                       C.POINTER(C.c_int32)]
        lib.fse_dist_masks.argtypes = [C.POINTER(EwaldConfig), C.c_int, _dp, i64, C.c_int,
                                       C.POINTER(C.c_uint32)]
        lib.fse_cuda_xscale_probe.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp,
                                              C.c_uint64, C.c_int, C.POINTER(C.c_int),
                                              C.POINTER(C.c_int), _dp, _dp]
        lib.fse_cuda_host_alloc.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
        lib.fse_cuda_host_free.argtypes = [vp]
        lib.fse_cuda_dev_alloc.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
        lib.fse_cuda_dev_free.argtypes = [vp, vp]
        lib.fse_cuda_memcpy.argtypes = [vp, vp, vp, C.c_size_t]
        lib.fse_cuda_mark.argtypes = [vp]
        lib.fse_cuda_elapsed_ms.argtypes = [vp, _dp]
        lib.fse_cuda_trim.argtypes = [vp]
        lib.fse_cuda_kernel_ms.argtypes = [vp, _dp, C.c_int]
        lib.fse_cuda_fp64_peak.argtypes = [vp, _dp]
        lib.fse_cuda_set_overlap.argtypes = [vp, C.c_int]
        lib.fse_cuda_freespace_solve.argtypes = [vp, vp, _dp, _dp]
        lib.fse_cuda_slab_info.argtypes = [C.POINTER(EwaldConfig), C.c_int, C.c_int, C.c_int,
                                           C.POINTER(SlabInfo)]
        lib.fse_cuda_slab_forward.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, vp, i64,
                                              C.c_int, C.c_int, vp]
        lib.fse_cuda_slab_scale.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, C.c_int,
                                            C.c_int, vp]
        lib.fse_cuda_slab_inverse.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, vp, i64,
                                              vp, C.c_int, C.c_int, vp, i64, C.c_int, vp]
        lib.fse_cuda_slab_forward_peers.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp, vp,
                                                    i64, C.c_int, C.c_int, C.POINTER(vp)]
        lib.fse_cuda_slab_scale_peers.argtypes = [vp, C.POINTER(EwaldConfig), C.c_int, vp,
                                                  C.c_int, C.c_int, vp, C.POINTER(vp)]
        lib.fse_cuda_realspace_counts.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.fse_fourier_error_estimate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                                   C.c_double, C.c_double, _dp]
        lib.fse_real_error_estimate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                                C.c_double, _dp]
        lib.fse_error_budget.argtypes = [C.c_int, C.POINTER(EwaldConfig), C.c_double,
                                         C.POINTER(ErrorBudget)]
        lib.fse_reference_velocity_rms.argtypes = [C.c_int, C.c_double, C.c_double, C.c_uint64,
                                                   _dp]
        lib.fse_select_parameters.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double,
                                              C.c_double, C.c_double, C.POINTER(EwaldConfig),
                                              C.POINTER(C.c_int)]
        lib.fse_generate_system.argtypes = [C.c_int, i64, C.c_double, C.c_uint64, _dp, _dp]
        lib.fse_generate_workload.argtypes = [C.c_int, i64, C.c_uint64, _dp, _dp, _dp]
        _lib = lib
        return lib


def lib():
    return _load()


_ERRORS = {1: InvalidArgument, 2: DomainError}


def _raise(status: int, msg: str):
    raise _ERRORS.get(status, FseRuntimeError)(f"[fse status {status}] {msg}")


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


# ------------------------------------------------------------------ config
def make_config(L, xi, rc, M, P, sf=0.0) -> EwaldConfig:
    cfg = EwaldConfig()
    err = C.create_string_buffer(256)
    st = _load().fse_make_config(float(L), float(xi), float(rc), int(M), int(P), float(sf),
                                 C.byref(cfg), err, 256)
    if st:
        _raise(st, err.value.decode())
    return cfg


# ------------------------------------------------------------------ context
class MollifiedGreen:
    """Device-resident fse::MollifiedGreen (greens.hpp:57-66).  `fourier`
    downloads the (2 Mtilde)^3 table in the reference layout."""

    def __init__(self, ctx: "Context", handle):
        self._ctx = ctx
        self._h = handle
        k, lt, h, R, mt = C.c_int(), C.c_double(), C.c_double(), C.c_double(), C.c_int()
        _load().fse_cuda_green_info(handle, C.byref(k), C.byref(lt), C.byref(h), C.byref(R),
                                    C.byref(mt))
        self.kind = GreenKind(k.value)
        self.Ltilde, self.h, self.R, self.Mtilde = lt.value, h.value, R.value, mt.value

    def doubled(self) -> int:
        return 2 * self.Mtilde

    @property
    def handle(self):
        return self._h

    @property
    def fourier(self) -> np.ndarray:
        D = self.doubled()
        out = np.empty((D, D, D))
        self._ctx._call(_load().fse_cuda_green_download, self._h, _p(out))
        return out

    def free(self):
        if self._h:
            _load().fse_cuda_green_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One GPU context (streams, cached buffers, cuFFT plans).  Thread-safe."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = _load().fse_cuda_create(int(device), C.byref(h))
        if st:
            _raise(st, f"fse_cuda_create(device={device}) failed")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            _load().fse_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def _call(self, fn, *args):
        st = fn(self._h, *args)
        if st:
            _raise(st, _load().fse_cuda_last_error(self._h).decode())

    @property
    def launch_count(self) -> int:
        return int(_load().fse_cuda_launch_count(self._h))

    def trim(self):
        self._call(_load().fse_cuda_trim)

    def kernel_ms(self):
        """Per-stage device ms of the last sum (see fse_cuda_kernel_ms)."""
        out = np.zeros(11)
        self._call(_load().fse_cuda_kernel_ms, _p(out), 11)
        return out.tolist()

    def set_overlap(self, on: bool):
        """Overlap the real-space sum with the Fourier part (default True)."""
        self._call(_load().fse_cuda_set_overlap, 1 if on else 0)

    def realspace_counts(self):
        """(candidates, pairs) of the last real-space pair kernel."""
        a, b = C.c_uint64(), C.c_uint64()
        self._call(_load().fse_cuda_realspace_counts, C.byref(a), C.byref(b))
        return a.value, b.value

    def measure_fp64_peak(self) -> float:
        v = C.c_double()
        self._call(_load().fse_cuda_fp64_peak, C.byref(v))
        return v.value

    # -- Green's functions
    def precompute_mollified_green(self, kind, Ltilde, Mtilde, sf) -> MollifiedGreen:
        h = C.c_void_p()
        self._call(_load().fse_cuda_green_precompute, int(kind), float(Ltilde), int(Mtilde),
                   float(sf), C.byref(h))
        return MollifiedGreen(self, h)

    def upload_mollified_green(self, kind, Ltilde, Mtilde, h, R, fourier) -> MollifiedGreen:
        f = _f64(fourier).reshape(-1)
        D = 2 * int(Mtilde)
        if f.size != D ** 3:
            raise InvalidArgument("green table must hold (2 Mtilde)^3 values")
        hd = C.c_void_p()
        self._call(_load().fse_cuda_green_upload, int(kind), float(Ltilde), int(Mtilde),
                   float(h), float(R), _p(f), C.byref(hd))
        return MollifiedGreen(self, hd)

    def save_mollified_green(self, green: MollifiedGreen, path: str):
        self._call(_load().fse_cuda_green_save, green.handle, path.encode())

    def load_mollified_green(self, path: str) -> MollifiedGreen:
        hd = C.c_void_p()
        self._call(_load().fse_cuda_green_load, path.encode(), C.byref(hd))
        return MollifiedGreen(self, hd)

    # -- hot path
    def total_sum(self, system: SourceSystem, kind, cfg: EwaldConfig, targets, green,
                  timings: StageTimings | None = None, targets_are_sources: int = -1,
                  out: np.ndarray | None = None):
        """fse::total_sum (ewald.cpp:394-415).  ``out``: optional (NT, 3) float64
        C-contiguous array to receive the velocities (e.g. pinned host memory
        from ``host_alloc``, which the device->host copy reads at full speed)."""
        t = _f64(targets, (-1, 3))
        if out is None:
            u = np.empty((t.shape[0], 3))
        else:
            if (out.shape != (t.shape[0], 3) or out.dtype != np.float64
                    or not out.flags["C_CONTIGUOUS"]):
                raise InvalidArgument("total_sum: out must be a C-contiguous (NT, 3) float64 array")
            u = out
        self._call(_load().fse_cuda_total_sum, C.byref(cfg), int(kind),
                   _p(system.positions), _p(system.strengths), system.size(),
                   float(system.box_side), _p(t), t.shape[0], int(targets_are_sources),
                   green.handle, _p(u), C.byref(timings) if timings is not None else None)
        return u

    def total_sum_dev(self, cfg, kind, d_pos, d_str, n, box_side, d_tgt, nt, green, d_u,
                      targets_are_sources=-1, timings=None):
        """Device-pointer variant (ints holding device addresses)."""
        self._call(_load().fse_cuda_total_sum_dev, C.byref(cfg), int(kind), C.c_void_p(d_pos),
                   C.c_void_p(d_str), int(n), float(box_side), C.c_void_p(d_tgt), int(nt),
                   int(targets_are_sources), green.handle, C.c_void_p(d_u),
                   C.byref(timings) if timings is not None else None)

    def freespace_solve(self, green: MollifiedGreen, rhs) -> np.ndarray:
        """fse::freespace_solve (greens.cpp:115-139): rhs (M~, M~, M~) on the green's grid."""
        M = green.Mtilde
        r = _f64(rhs)
        if r.shape != (M, M, M):
            raise InvalidArgument("freespace_solve: rhs extents must match green")
        out = np.empty((M, M, M))
        self._call(_load().fse_cuda_freespace_solve, green.handle, _p(r), _p(out))
        return out

    # -- z-slab decomposition (device pointers; see fse_cuda_slab_* and slabs.py)
    def slab_forward(self, cfg, kind, d_pos, d_str, n, rank, nslabs, d_spec):
        self._call(_load().fse_cuda_slab_forward, C.byref(cfg), int(kind), C.c_void_p(d_pos),
                   C.c_void_p(d_str), int(n), int(rank), int(nslabs), C.c_void_p(d_spec))

    def slab_scale(self, cfg, kind, green, rank, nslabs, d_spec):
        self._call(_load().fse_cuda_slab_scale, C.byref(cfg), int(kind), green.handle,
                   int(rank), int(nslabs), C.c_void_p(d_spec))

    # peer-direct exchange: dst_bufs[s] = rank s's exchange buffer mapped here
    def slab_forward_peers(self, cfg, kind, d_pos, d_str, n, rank, nslabs, dst_bufs):
        ptrs = (C.c_void_p * len(dst_bufs))(*[int(q) for q in dst_bufs])
        self._call(_load().fse_cuda_slab_forward_peers, C.byref(cfg), int(kind),
                   C.c_void_p(d_pos), C.c_void_p(d_str), int(n), int(rank), int(nslabs), ptrs)

    def slab_scale_peers(self, cfg, kind, green, rank, nslabs, d_spec, dst_bufs):
        ptrs = (C.c_void_p * len(dst_bufs))(*[int(q) for q in dst_bufs])
        self._call(_load().fse_cuda_slab_scale_peers, C.byref(cfg), int(kind), green.handle,
                   int(rank), int(nslabs), C.c_void_p(d_spec), ptrs)

    def slab_inverse(self, cfg, kind, d_pos, d_str, n, d_spec, rank, nslabs, d_tgt, nt, tas,
                     d_u):
        self._call(_load().fse_cuda_slab_inverse, C.byref(cfg), int(kind), C.c_void_p(d_pos),
                   C.c_void_p(d_str), int(n), C.c_void_p(d_spec), int(rank), int(nslabs),
                   C.c_void_p(d_tgt), int(nt), int(tas), C.c_void_p(d_u))

    def fourier_sum(self, system: SourceSystem, cfg: EwaldConfig, kind, targets, green,
                    timings: StageTimings | None = None):
        t = _f64(targets, (-1, 3))
        u = np.empty((t.shape[0], 3))
        self._call(_load().fse_cuda_fourier_sum, C.byref(cfg), int(kind), _p(system.positions),
                   _p(system.strengths), system.size(), float(system.box_side), _p(t),
                   t.shape[0], green.handle, _p(u),
                   C.byref(timings) if timings is not None else None)
        return u

    def real_space_sum(self, system: SourceSystem, kind, xi, rc, targets):
        t = _f64(targets, (-1, 3))
        u = np.empty((t.shape[0], 3))
        self._call(_load().fse_cuda_real_space_sum, int(kind), _p(system.positions),
                   _p(system.strengths), system.size(), float(system.box_side), float(xi),
                   float(rc), _p(t), t.shape[0], _p(u))
        return u

    def spread(self, system: SourceSystem, cfg: EwaldConfig, kind, use_fgg: bool = True):
        """fse::spread (ewald.cpp:136-214); use_fgg=False: one exp per node
        (axis_weights_naive, ewald.cpp:53-66)."""
        a = strength_arity(kind)
        Mt = cfg.Mtilde
        grid = np.empty((a, Mt, Mt, Mt))
        self._call(_load().fse_cuda_spread_ex, C.byref(cfg), int(kind), _p(system.positions),
                   _p(system.strengths), system.size(), float(system.box_side),
                   int(bool(use_fgg)), _p(grid))
        return grid

    def kspace_scale(self, ghat, cfg: EwaldConfig, kind, green):
        a = strength_arity(kind)
        D = cfg.D
        gh = np.ascontiguousarray(ghat, dtype=np.complex128)
        if gh.shape != (a, D, D, D):
            raise InvalidArgument("kspace_scale: component count / plane size does not match")
        out = np.empty((3, D, D, D), np.complex128)
        self._call(_load().fse_cuda_kspace_scale, C.byref(cfg), int(kind), green.handle,
                   gh.ctypes.data_as(_dp), out.ctypes.data_as(_dp))
        return out

    def build_cell_list(self, system: SourceSystem, rc, domain_pad=0.0) -> CellList:
        dims = (C.c_int * 3)()
        side, origin = C.c_double(), C.c_double()
        n = system.size()
        fn = _load().fse_cuda_build_cell_list
        self._call(fn, _p(system.positions), n, float(system.box_side), float(rc),
                   float(domain_pad), dims, C.byref(side), C.byref(origin), None, None)
        ncell = dims[0] * dims[1] * dims[2]
        bstart = np.empty(ncell + 1, np.int64)
        perm = np.empty(max(n, 1), np.int64)
        self._call(fn, _p(system.positions), n, float(system.box_side), float(rc),
                   float(domain_pad), dims, C.byref(side), C.byref(origin),
                   bstart.ctypes.data_as(C.POINTER(C.c_int64)),
                   perm.ctypes.data_as(C.POINTER(C.c_int64)))
        return CellList(side.value, origin.value, tuple(dims), bstart, perm[:n])

    def support_index(self, cfg: EwaldConfig, points):
        p = _f64(points, (-1, 3))
        i0 = np.empty((p.shape[0], 3), np.int32)
        self._call(_load().fse_cuda_support_index, C.byref(cfg), _p(p), p.shape[0],
                   i0.ctypes.data_as(C.POINTER(C.c_int32)))
        return i0

    def direct_sum(self, system: SourceSystem, kind, targets, exclude_self: bool):
        t = _f64(targets, (-1, 3))
        u = np.empty((t.shape[0], 3))
        self._call(_load().fse_cuda_direct_sum, int(kind), _p(system.positions),
                   _p(system.strengths), system.size(), _p(t), t.shape[0], int(exclude_self),
                   _p(u))
        return u

    def fft_columns(self, cols, inverse=False):
        """The hot path's hand-written FFT engine on rows of `cols` (ncols, D)."""
        d = np.ascontiguousarray(cols, dtype=np.complex128).copy()
        nc, D = d.shape
        self._call(_load().fse_cuda_fft_columns, int(D), int(nc), d.ctypes.data_as(_dp),
                   int(inverse))
        return d

    def xscale_probe(self, cfg, kind, green, seed, ky, kz):
        """Diagnostics (fse_cuda_xscale_probe): the hot path's fused x pass on a
        pseudo-random spectrum; returns (out (np, 3, Mt) complex, gcol (np, D))."""
        ky = np.ascontiguousarray(ky, dtype=np.int32)
        kz = np.ascontiguousarray(kz, dtype=np.int32)
        npb = ky.shape[0]
        out = np.empty((npb, 3, cfg.Mtilde), np.complex128)
        gcol = np.empty((npb, cfg.D))
        ip = C.POINTER(C.c_int)
        self._call(_load().fse_cuda_xscale_probe, C.byref(cfg), int(kind),
                   green.handle if green is not None else None, int(seed), npb,
                   ky.ctypes.data_as(ip), kz.ctypes.data_as(ip), out.ctypes.data_as(_dp), _p(gcol))
        return out, gcol

    # -- partitioned multi-GPU evaluation (fse_dist)
    def dist_virtual_total_sum(self, system: SourceSystem, kind, cfg, targets, green, nranks,
                               targets_are_sources=False, profile=None):
        """The partitioned algorithm (ownership, ghost exchange, distributed FFT,
        partial-sum return) with `nranks` virtual ranks on this device; u in
        caller order.  profile: optional (nranks, 6, 2) float64 array receiving
        per rank and step (classify, pack, forward, scale, inverse, finish) the
        step time in ms with the rank alone on the device and the bytes sent."""
        t = system.positions if targets_are_sources else _f64(targets, (-1, 3))
        n, nt = system.size(), t.shape[0]
        ptrs = []
        try:
            def up(a):
                p = self.dev_alloc(max(a.nbytes, 8))
                ptrs.append(p)
                if a.nbytes:
                    self.memcpy(p, a.ctypes.data, a.nbytes)
                return p
            dp, ds = up(system.positions), up(system.strengths)
            dt = dp if targets_are_sources else up(t)
            du = self.dev_alloc(max(24 * nt, 8))
            ptrs.append(du)
            self._call(_load().fse_cuda_dist_virtual_total_sum, int(nranks), C.byref(cfg),
                       int(kind), C.c_void_p(dp), C.c_void_p(ds), n, C.c_void_p(dt), nt,
                       int(bool(targets_are_sources)), green.handle, C.c_void_p(du),
                       profile.ctypes.data_as(C.c_void_p) if profile is not None else None)
            u = np.empty((nt, 3))
            if nt:
                self.memcpy(u.ctypes.data, du, u.nbytes)
            return u
        finally:
            for p in ptrs:
                self.dev_free(p)

    def dist_create(self, rank: int, nranks: int, unique_id: bytes):
        """NCCL rank of the partitioned evaluation (fse_cuda_dist_create)."""
        h = C.c_void_p()
        idb = C.create_string_buffer(bytes(unique_id), 128)
        self._call(_load().fse_cuda_dist_create, int(rank), int(nranks), idb, C.byref(h))
        return h

    def dist_total_sum(self, dist, cfg, kind, d_pos, d_str, n_own, n_total, d_tgt, nt_own, tas,
                       green, d_u):
        """fse_cuda_dist_total_sum on device pointers (this rank's owned points)."""
        st = _load().fse_cuda_dist_total_sum(dist, C.byref(cfg), int(kind), C.c_void_p(d_pos),
                                             C.c_void_p(d_str), int(n_own), int(n_total),
                                             C.c_void_p(d_tgt), int(nt_own), int(bool(tas)),
                                             green.handle, C.c_void_p(d_u))
        if st != 0:
            _raise(st, _load().fse_cuda_last_error(self.handle).decode())

    def fft3d(self, data, inverse=False):
        d = np.ascontiguousarray(data, dtype=np.complex128).copy()
        n0, n1, n2 = d.shape
        self._call(_load().fse_cuda_fft3d, d.ctypes.data_as(_dp), n0, n1, n2, int(inverse))
        return d

    # -- device memory helpers (bench)
    def dev_alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        self._call(_load().fse_cuda_dev_alloc, int(nbytes), C.byref(p))
        return p.value

    def dev_free(self, ptr: int):
        _load().fse_cuda_dev_free(self._h, C.c_void_p(ptr))

    def host_alloc(self, shape, dtype=np.float64) -> np.ndarray:
        """Pinned host array; the pinned block is released (fse_cuda_host_free) when
        the array and every view of it are garbage collected."""
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        self._call(_load().fse_cuda_host_alloc, n, C.byref(p))
        buf = (C.c_char * max(n, 1)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
        weakref.finalize(buf, _load().fse_cuda_host_free, C.c_void_p(p.value))
        return arr

    def memcpy(self, dst: int, src: int, nbytes: int):
        self._call(_load().fse_cuda_memcpy, C.c_void_p(dst), C.c_void_p(src), int(nbytes))

    def mark(self):
        self._call(_load().fse_cuda_mark)

    def elapsed_ms(self) -> float:
        v = C.c_double()
        self._call(_load().fse_cuda_elapsed_ms, C.byref(v))
        return v.value


# ---------------------------------------------------------- default context
_default = None
_default_lock = threading.Lock()


def default_context() -> Context:
    global _default
    with _default_lock:
        if _default is None:
            _default = Context(int(os.environ.get("FSE_CUDA_DEVICE", "0")))
        return _default


def precompute_mollified_green(kind, Ltilde, Mtilde, sf) -> MollifiedGreen:
    return default_context().precompute_mollified_green(kind, Ltilde, Mtilde, sf)


def spread(system, cfg, kind, use_fgg=True):
    return default_context().spread(system, cfg, kind, use_fgg)


def kspace_scale(ghat, cfg, kind, green):
    return default_context().kspace_scale(ghat, cfg, kind, green)


def fourier_sum(system, cfg, kind, targets, green, timings=None):
    return default_context().fourier_sum(system, cfg, kind, targets, green, timings)


def total_sum(system, kind, cfg, targets, green, timings=None):
    return default_context().total_sum(system, kind, cfg, targets, green, timings)


def real_space_sum(system, kind, xi, rc, targets):
    return default_context().real_space_sum(system, kind, xi, rc, targets)


def freespace_solve(green, rhs):  # greens.hpp:76
    return green._ctx.freespace_solve(green, rhs)


def build_cell_list(system, rc, domain_pad=0.0):
    return default_context().build_cell_list(system, rc, domain_pad)


def direct_sum(system, kind, targets, exclude_self):
    return default_context().direct_sum(system, kind, targets, exclude_self)


def fft3d_forward(data):
    return default_context().fft3d(data, inverse=False)


def fft3d_inverse(data):
    return default_context().fft3d(data, inverse=True)


def save_mollified_green(green, path):
    green._ctx.save_mollified_green(green, path)


def load_mollified_green(path):
    return default_context().load_mollified_green(path)


# ---------------------------------------------------------- host helpers
def self_interaction(xi, f, kind):  # kernels.cpp:84-89
    if not xi > 0:
        raise InvalidArgument("self_interaction: xi must be positive")
    if int(kind) != KernelKind.Stokeslet:
        return np.zeros(3)
    return (-4.0 * xi / np.sqrt(np.pi)) * np.asarray(f, dtype=np.float64)[:3]


def rms_error(u, u_ref, relative):  # kernels.cpp:91-103
    u, u_ref = np.asarray(u, dtype=np.float64), np.asarray(u_ref, dtype=np.float64)
    if u.shape != u_ref.shape:
        raise InvalidArgument("rms_error: length mismatch")
    num = float(((u - u_ref) ** 2).sum())
    den = float((u_ref ** 2).sum())
    n = u.shape[0]
    ab = np.sqrt(num / n)
    if not relative:
        return ab
    if den == 0:
        raise DomainError("rms_error: relative error of zero reference")
    return ab / np.sqrt(den / n)


def strength_quadratic_sum(system: SourceSystem) -> float:  # kernels.cpp:105-110
    """Sequential sum of c_i^2 in the reference's order (bit-identical Q)."""
    st = system.strengths
    return float(np.cumsum((st * st).ravel())[-1]) if st.size else 0.0


def generate_system(kind, n, L, seed) -> SourceSystem:
    """fse::generate_system (harness.cpp:47-66), bit-identical stream."""
    pos = np.empty((n, 3))
    st = np.empty((n, strength_arity(kind)))
    if _load().fse_generate_system(int(kind), int(n), float(L), int(seed), _p(pos), _p(st)):
        raise InvalidArgument("generate_system: need N >= 1, L > 0")
    return SourceSystem(pos, st, float(L))


WL_UNIFORM, WL_SPHERE, WL_CLUSTERED, WL_UNIFORM_TARGETS = 1, 3, 4, 5


class MultiContext:
    """Several GPUs in one process (fse_cuda_multi_*): total_sum with host buffers,
    partitioned over the devices with NCCL inside the library."""

    def __init__(self, devices):
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        st = _load().fse_cuda_multi_create(devs, len(devices), C.byref(h))
        if st != 0:
            _raise(st, "fse_cuda_multi_create failed")
        self._h = h

    def close(self):
        if self._h:
            _load().fse_cuda_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def total_sum(self, system: SourceSystem, kind, cfg, targets, green_full=None,
                  targets_are_sources: int = -1):
        t = _f64(targets, (-1, 3))
        u = np.empty((t.shape[0], 3))
        gp = None
        if green_full is not None:
            green_full = _f64(green_full)
            gp = green_full.ctypes.data_as(C.c_void_p)
        st = _load().fse_cuda_multi_total_sum(self._h, C.byref(cfg), int(kind),
                                              _p(system.positions), _p(system.strengths),
                                              system.size(), float(system.box_side), _p(t),
                                              t.shape[0], int(targets_are_sources), gp, _p(u),
                                              None)
        if st != 0:
            _raise(st, _load().fse_cuda_multi_last_error(self._h).decode())
        return u


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 makes it; the caller broadcasts it)."""
    b = C.create_string_buffer(128)
    st = _load().fse_cuda_nccl_unique_id(b)
    if st != 0:
        raise FseRuntimeError("ncclGetUniqueId failed")
    return b.raw


def dist_owner(cfg: EwaldConfig, nranks: int, positions) -> np.ndarray:
    """Owner slab of every point (fse_dist_owner; host)."""
    p = _f64(positions, (-1, 3))
    out = np.empty(p.shape[0], np.int32)
    st = _load().fse_dist_owner(C.byref(cfg), int(nranks), _p(p), p.shape[0],
                                out.ctypes.data_as(C.POINTER(C.c_int32)))
    if st != 0:
        raise InvalidArgument("dist_owner: bad arguments")
    return out


def dist_masks(cfg: EwaldConfig, nranks: int, positions, targets: bool) -> np.ndarray:
    """Bit masks of the ranks that need each point (fse_dist_masks; host)."""
    p = _f64(positions, (-1, 3))
    out = np.empty(p.shape[0], np.uint32)
    st = _load().fse_dist_masks(C.byref(cfg), int(nranks), _p(p), p.shape[0], int(bool(targets)),
                                out.ctypes.data_as(C.POINTER(C.c_uint32)))
    if st != 0:
        raise InvalidArgument("dist_masks: bad arguments")
    return out


def generate_workload(which: int, n: int, seed: int):
    """SURVEY.md 8(d) generators; returns (SourceSystem, targets or None)."""
    a = 9 if which == WL_SPHERE else 3
    pos = np.empty((n, 3))
    st = np.empty((n, a))
    tgt = np.empty((n, 3)) if which == WL_UNIFORM_TARGETS else None
    if _load().fse_generate_workload(int(which), int(n), int(seed), _p(pos), _p(st), _p(tgt)):
        raise InvalidArgument("generate_workload: bad arguments")
    return SourceSystem(pos, st, 1.0), tgt
