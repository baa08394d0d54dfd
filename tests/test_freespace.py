"""fse::freespace_solve on the GPU (greens.cpp:115-139).

Pinned three ways: a numpy restatement of greens.cpp:115-139 on the same
Green's table (zero-pad, FFT, multiply, inverse FFT, window); the reference
test suite's analytic Gaussian oracles (test_greens.cpp: conv(1/r, Gaussian) =
erf(sqrt(a) r)/r and the biharmonic closed form, < 1e-10 at M~ = 48, spectral
convergence over M~); linearity, zero rhs and the extents check.
"""
import numpy as np
import pytest
from math import erf, sqrt, pi, exp

pytestmark = pytest.mark.gpu

KA = 200.0  # Gaussian sharpness of the analytic oracles (test_greens.cpp)


def gaussian_rhs(M, Lt, c):
    h = Lt / M
    x = np.arange(M) * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    r2 = (X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2
    return (KA / pi) ** 1.5 * np.exp(-KA * r2), np.sqrt(r2)


def exact(kind, r):
    if kind == 0:
        return np.where(r < 1e-12, 2 * sqrt(KA / pi),
                        np.vectorize(lambda t: erf(sqrt(KA) * t) / max(t, 1e-300))(r))
    rr = np.maximum(r, 1e-12)
    return ((rr + 1 / (2 * KA * rr)) * np.vectorize(lambda t: erf(sqrt(KA) * t))(rr)
            + np.exp(-KA * rr * rr) / sqrt(pi * KA))


def solve_error(fse, ctx, kind, M, sf=2.7320508075688772):
    g = ctx.precompute_mollified_green(kind, 1.0, M, sf)
    rhs, r = gaussian_rhs(M, 1.0, (0.5, 0.5, 0.5))
    phi = ctx.freespace_solve(g, rhs)
    ref = exact(kind, r)
    return np.abs(phi - ref).max() / np.abs(ref).max()


@pytest.mark.parametrize("kind", [0, 1])
def test_gaussian_oracle(fse, ctx, kind):
    assert solve_error(fse, ctx, kind, 48) < 1e-10


@pytest.mark.parametrize("kind", [0, 1])
def test_spectral_convergence(fse, ctx, kind):
    prev = -1
    for M in (16, 24, 32, 48):
        err = solve_error(fse, ctx, kind, M)
        if prev > 1e-12:
            assert prev / err > 10.0
        prev = err
    assert prev < 1e-12


@pytest.mark.parametrize("kind,M", [(0, 12), (1, 20), (0, 37), (1, 48)])
def test_matches_numpy_restatement(fse, ctx, rng, kind, M):
    g = ctx.precompute_mollified_green(kind, 1.3, M, 2.7320508075688772 if kind == 0 else 3.0)
    rhs = rng.standard_normal((M, M, M))
    D = 2 * M
    buf = np.zeros((D, D, D), dtype=complex)
    buf[:M, :M, :M] = rhs
    want = np.fft.ifftn(np.fft.fftn(buf) * g.fourier)[:M, :M, :M].real
    got = ctx.freespace_solve(g, rhs)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_linearity_zero_and_extents(fse, ctx, rng):
    M = 12
    g = ctx.precompute_mollified_green(0, 1.0, M, 2.7320508075688772)
    assert np.all(ctx.freespace_solve(g, np.zeros((M, M, M))) == 0)
    f1, _ = gaussian_rhs(M, 1.0, (0.4, 0.5, 0.55))
    f2, _ = gaussian_rhs(M, 1.0, (0.6, 0.45, 0.5))
    u1, u2, us = (ctx.freespace_solve(g, f) for f in (f1, f2, f1 + f2))
    assert np.allclose(us, u1 + u2, rtol=1e-12, atol=1e-12 * np.abs(us).max())
    with pytest.raises(fse.InvalidArgument):
        ctx.freespace_solve(g, np.zeros((M - 1, M, M)))
