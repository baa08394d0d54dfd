"""Error estimates and parameter selection, CPU only.

The restatement (csrc/cpp/fse_estimates.cpp via the C-ABI of
include/fse_host.h) is pinned to the reference compiled from its own sources
(oracle/_ref, estimates.cpp:13-126): same formulas and libm calls, so the
results are compared bit for bit.  Also the reference's own known answers
(test_estimates.cpp:84-108): the criterion-2 workload selection and the
degenerate / infeasible / invalid branches.
"""
import numpy as np
import pytest


def _cfg_fields(c):
    return (c.L, c.xi, c.rc, c.M, c.P, c.h, c.d, c.m, c.eta, c.deltaL, c.Ltilde, c.Mtilde,
            c.kinf, c.R, c.sf)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_estimators_match_reference(fse, ref, kind):
    rng = np.random.default_rng(7 + kind)
    for _ in range(200):
        L = rng.uniform(0.5, 3.0)
        xi = rng.uniform(1.0, 60.0)
        M = int(rng.integers(8, 128))
        P = int(rng.choice([8, 12, 16, 20, 24]))
        rc = rng.uniform(0.02, 0.5) * L
        Q = rng.uniform(0.1, 1e4)
        try:
            cfg = fse.make_config(L, xi, rc, M, P)
        except fse.InvalidArgument:
            continue
        b = fse.error_budget(kind, cfg, Q)
        rr, rf = ref.error_budget(kind, L, xi, rc, M, P, Q)
        assert b.predicted_real_rms == rr and b.predicted_fourier_rms == rf
        assert b.predicted_real_rms == fse.real_error_estimate(kind, Q, xi, rc, L)
        assert b.predicted_fourier_rms == fse.fourier_error_estimate(kind, Q, xi, cfg.kinf, L,
                                                                     cfg.R)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_select_parameters_matches_reference(fse, ref, kind):
    rng = np.random.default_rng(100 + kind)
    for _ in range(60):
        N = int(rng.integers(10, 200000))
        L = rng.uniform(0.5, 3.0)
        Q = rng.uniform(1.0, 1e5)
        xi = rng.uniform(2.0, 40.0) / L
        tol = 10.0 ** rng.uniform(-13, -3)
        try:
            want, wfeas = ref.select_parameters(kind, N, L, Q, xi, tol)
        except Exception:
            with pytest.raises(fse.InvalidArgument):
                fse.select_parameters(kind, N, L, Q, xi, tol)
            continue
        got, feas = fse.select_parameters(kind, N, L, Q, xi, tol)
        assert feas == wfeas
        assert _cfg_fields(got) == tuple(getattr(want, k) for k in (
            "L", "xi", "rc", "M", "P", "h", "d", "m", "eta", "deltaL", "Ltilde", "Mtilde",
            "kinf", "R", "sf"))


def test_select_parameters_known_answers(fse):
    # test_estimates.cpp:84-93: the criterion-2 workload (L = 2, xi = 7, tol 5e-9) picks
    # P = 16 and an even M
    s = fse.generate_system(0, 20000, 2.0, 2026)
    Q = float((s.strengths ** 2).sum())
    cfg, feas = fse.select_parameters(0, 20000, 2.0, Q, 7.0, 0.5e-8)
    assert feas and cfg.P == 16 and cfg.M % 2 == 0
    b = fse.error_budget(0, cfg, Q)
    ref_rms = fse.reference_velocity_rms(0, Q, 2.0, 20000)
    assert b.predicted_real_rms <= 0.25 * 0.5e-8 * ref_rms * 1.0000001
    assert b.predicted_fourier_rms <= 0.25 * 0.5e-8 * ref_rms * 1.0000001
    # test_estimates.cpp:95-108: loose tolerance -> rc = 1/xi; hopeless -> infeasible;
    # invalid arguments raise
    loose, ok = fse.select_parameters(0, 100, 1.0, 100.0, 8.0, 0.5)
    assert ok and loose.rc == 1.0 / 8.0
    hard, ok = fse.select_parameters(0, 100, 1.0, 100.0, 0.05, 1e-300)
    assert not ok and hard.rc == np.sqrt(3.0)
    with pytest.raises(fse.InvalidArgument):
        fse.select_parameters(0, 100, 1.0, 100.0, 8.0, -1.0)
    with pytest.raises(fse.InvalidArgument):
        fse.real_error_estimate(0, -1.0, 8.0, 0.1, 1.0)
