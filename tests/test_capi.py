"""CPU checks of the product library without a GPU: it loads, exports every
symbol include/*.h declares, and its host-only pieces (make_config, the
EwaldConfig mirror, the generators) match the reference bit for bit."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("fse_cuda.h", "fse_host.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(fse_\w+)\s*\(", src):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol(fse):
    lib = ctypes.CDLL(fse.library_path())
    syms = declared_symbols()
    assert len(syms) > 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_arity(fse):
    lib = fse.api.lib()
    assert lib.fse_cuda_abi_version() == 1
    assert [lib.fse_arity(k) for k in (0, 1, 2)] == [3, 9, 3]


def test_config_layout_mirrors_ewaldconfig(fse):
    C = fse.EwaldConfig
    assert ctypes.sizeof(C) == 120
    assert C.Mtilde.offset == 80 and C.kinf.offset == 88 and C.deterministic.offset == 112


@pytest.mark.parametrize("args", [(2.0, 7.0, 0.63, 48, 16), (2.0, 30.0, 0.2, 48, 16),
                                  (1.0, 110.0, 0.045, 288, 24), (1.0, 28.0, 0.15, 80, 16),
                                  (1.0, 40.0, 0.12, 128, 20), (1.0, 220.0, 0.022, 576, 24),
                                  (1.0, 6.0, 0.3, 12, 8, 3.5)])
def test_make_config_bitwise(fse, oracle, args):
    a = fse.make_config(*args)
    b = oracle.make_config(*args)
    for k in ("L", "xi", "rc", "M", "P", "h", "d", "m", "eta", "deltaL", "Ltilde", "Mtilde",
              "kinf", "R", "sf"):
        assert getattr(a, k) == getattr(b, k), k


def test_make_config_bitwise_vs_reference(fse, ref):
    for args in [(1.0, 110.0, 0.045, 288, 24), (2.0, 7.0, 0.58, 38, 16)]:
        a, b = fse.make_config(*args), ref.make_config(*args)
        assert (a.h, a.eta, a.deltaL, a.Mtilde, a.kinf, a.R) == (b.h, b.eta, b.deltaL, b.Mtilde,
                                                                 b.kinf, b.R)


def test_make_config_errors(fse):
    for bad in [(2.0, 7.0, 0.63, 48, 15), (2.0, 7.0, 0.63, 0, 16), (-1.0, 7.0, 0.63, 48, 16),
                (2.0, 7.0, 0.63, 48, 16, 1.5), (1.0, 7.0, -0.1, 48, 16), (1.0, 7.0, 0.1, 48, 0)]:
        with pytest.raises(fse.InvalidArgument):
            fse.make_config(*bad)


def test_generate_system_matches_reference_harness(fse, ref):
    for kind in (0, 1, 2):
        s = fse.generate_system(kind, 777, 2.0, 2026 + kind)
        p, q = ref.generate_system(kind, 777, 2.0, 2026 + kind)
        assert np.array_equal(s.positions, p) and np.array_equal(s.strengths, q)


def test_workload_generators(fse):
    s, t = fse.generate_workload(fse.WL_UNIFORM, 5000, 1)
    assert t is None and s.positions.min() >= 0 and s.positions.max() < 1
    assert abs(s.strengths.mean()) < 0.05 and abs(s.strengths.std() - 1) < 0.05
    s, t = fse.generate_workload(fse.WL_SPHERE, 2000, 2)
    r = np.linalg.norm(s.positions - 0.5, axis=1)
    assert np.allclose(r, 0.5, atol=1e-12) and s.strengths.shape == (2000, 9)
    n = (s.positions - 0.5) / 0.5
    f = s.strengths.reshape(-1, 3, 3)
    q = f[:, 0, :] / n[:, :1]  # f_lm = n_l q_m
    assert np.allclose(f, n[:, :, None] * q[:, None, :], rtol=1e-9, atol=1e-12)
    s, t = fse.generate_workload(fse.WL_CLUSTERED, 6400, 3)
    assert s.positions.max() < 1.0 and s.positions.min() >= 0.0
    s, t = fse.generate_workload(fse.WL_UNIFORM_TARGETS, 100, 4)
    assert t.shape == (100, 3)
    a, _ = fse.generate_workload(fse.WL_UNIFORM, 100, 9)
    b, _ = fse.generate_workload(fse.WL_UNIFORM, 100, 9)
    assert np.array_equal(a.positions, b.positions)


def test_missing_library_fails_loudly(fse, monkeypatch, tmp_path):
    api = fse.api
    monkeypatch.setattr(api, "LIB_PATH", str(tmp_path / "absent.so"))
    monkeypatch.setattr(api, "_lib", None)
    with pytest.raises(ImportError):
        api.lib()


def test_rms_error_and_self_interaction(fse):
    u = np.array([[1.0, 0, 0], [0, 1.0, 0]])
    assert fse.rms_error(u, u, True) == 0
    with pytest.raises(fse.DomainError):
        fse.rms_error(u, np.zeros_like(u), True)
    v = fse.self_interaction(2.0, [1.0, 2.0, 3.0], fse.KernelKind.Stokeslet)
    assert np.allclose(v, -8.0 / np.sqrt(np.pi) * np.array([1, 2, 3]))
    assert np.all(fse.self_interaction(2.0, [1.0, 2.0, 3.0], fse.KernelKind.Rotlet) == 0)


def test_fft_planner_verdicts_without_a_gpu(fse):
    """fse_fft_plan_query (host only): every BASELINE grid and tolerance-consistent
    variant has an engine -- including cfg5t's D = 1730 = 2 x 5 x 173 (Stockham with a
    generic first stage) -- and a grid beyond the engines is refused with
    invalid_argument, the status total_sum returns before allocating anything."""
    lib = ctypes.CDLL(fse.library_path())
    lib.fse_fft_plan_query.restype = ctypes.c_int
    lib.fse_fft_plan_query.argtypes = [ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]

    def query(D, kind=0):
        e, g = ctypes.c_int(-1), ctypes.c_int(-1)
        st = lib.fse_fft_plan_query(D, kind, ctypes.byref(e), ctypes.byref(g))
        return st, e.value, g.value

    assert query(624) == (0, 1, 0)       # cfg2 / cfg4: register engine 24 x 26
    assert query(1200) == (0, 2, 0)      # cfg5: 30 x 40
    assert query(704) == (0, 3, 0)       # cfg4t
    assert query(242) == (0, 4, 0)       # cfg1t
    for D in (194, 298):                 # cfg1, cfg3: Bluestein engines (primes 97, 149)
        st, e, g = query(D, 1)
        assert st == 0 and e in (5, 6, 7) and g == 0
    assert query(348, 1) == (0, 0, 1)    # cfg3t = 12 x 29: generic stage beats Bluestein
    assert query(888) == (0, 0, 1)       # cfg2t: generic stage of radix 37
    assert query(1730) == (0, 0, 1)      # cfg5t: generic stage of radix 173
    assert query(2018)[0] == 1           # 2 x 1009: FSE_EINVAL
    assert query(623)[0] == 1 and query(624, 7)[0] == 1
