"""The fused x pass of the hot path (k_xscale / k_xscale2: forward x-FFT ->
k-space multiplier -> inverse x-FFT, in place on the pruned spectrum) against
a numpy restatement, column by column, on EVERY FFT engine the BASELINE
configurations and their tolerance-consistent variants select (register
engines 624, 1200, 704, 242; Bluestein 194 (cfg1), 298 (cfg3), 422; Stockham with
a generic first stage 348 (cfg3t), 888 (cfg2t), 1730 (cfg5t)) and all three kernels, including the stresslet's nine input
columns on the 1200- and 704-point engines.

The input spectrum and (by default) the Green's table are pseudo-random
(splitmix64, fse_cuda_xscale_probe), so the check is size-independent: the
multiplier is the reference's kspace_scale (ewald.cpp:216-293) with the
Nyquist-exact Hermitian average A_eff(k) = (A(k) + A(k~)) / 2,
1/D^3 folded in, applied between an unnormalised forward and inverse DFT of
length D = 2 Mtilde over the zero-padded x < Mtilde input; the window keeps
x < Mtilde.  One case runs with the real mollified Green's table."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from xpass_numpy import expected, splitmix_u


def columns(cfg, rng, n=20):
    D = cfg.D
    h = D // 2
    fixed = [(0, 0), (h, 0), (0, h), (h, h), (1, h), (h, 1), (D - 1, 1), (3, 0)]
    ky = list(rng.integers(0, D, n - len(fixed)))
    kz = list(rng.integers(0, h + 1, n - len(fixed)))
    return (np.array([f[0] for f in fixed] + ky, np.int32),
            np.array([f[1] for f in fixed] + kz, np.int32))


# (label, make_config args, expected D, kinds): every engine the BASELINE configs and
# their select_parameters variants use, plus the 422 Bluestein-1024 engine
CASES = [
    ("cfg2/cfg4 624", (1.0, 110.0, 0.045, 288, 24), 624, (0, 1, 2)),
    ("cfg5 1200", (1.0, 220.0, 0.022, 576, 24), 1200, (0, 1, 2)),
    ("cfg4t 704", (1.0, 110.0, 0.043375, 328, 24), 704, (0, 1, 2)),
    ("cfg1t 242", (1.0, 28.0, 0.15276, 96, 16), 242, (0, 1, 2)),
    ("cfg3 298 (Bluestein)", (1.0, 40.0, 0.12, 128, 20), 298, (0, 1, 2)),
    ("cfg3t 348", (1.0, 40.0, 0.11451, 146, 16), 348, (0, 1, 2)),
    ("422 (Bluestein-1024)", (1.0, 110.0, 0.045, 187, 24), 422, (0, 1, 2)),
    ("cfg2t 888", (1.0, 110.0, 0.042896, 414, 24), 888, (0, 2)),
    ("cfg1 194", (1.0, 28.0, 0.15, 80, 16), 194, (0, 1, 2)),
    # cfg5's tolerance-consistent grid: generic Stockham stage of radix 173, one CTA
    # per SM at the 227 KB shared-memory maximum (~90 GB of spectra: stokeslet only)
    ("cfg5t 1730", (1.0, 220.0, 0.021279, 834, 24), 1730, (0,)),
]


@pytest.mark.parametrize("label,args,D,kinds", CASES, ids=[c[0] for c in CASES])
def test_xpass_matches_numpy(fse, ctx, label, args, D, kinds):
    cfg = fse.make_config(*args)
    assert cfg.D == D
    rng = np.random.default_rng(D)
    ky, kz = columns(cfg, rng)
    for kind in kinds:
        seed = 1000 * D + kind
        got, gcol = ctx.xscale_probe(cfg, kind, None, seed, ky, kz)
        # the synthetic table is what the kernel read
        Dh = D // 2 + 1
        q = (np.arange(D, dtype=np.uint64)[None, :] * np.uint64(D) + ky[:, None].astype(np.uint64)) \
            * np.uint64(Dh) + kz[:, None].astype(np.uint64)
        assert np.array_equal(gcol, 0.5 + splitmix_u(np.uint64(seed ^ 0x5DEECE66D) + q))
        want = expected(cfg, kind, seed, ky, kz, gcol)
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err <= 1e-12, (label, kind, err)
    ctx.trim()


def test_xpass_too_large_is_refused_cleanly(fse, ctx):
    """D = 2018 = 2 x 1009 exceeds every FFT engine (Bluestein would need a
    >= 4035-point register engine, three generic-Stockham columns more than 227 KB
    of shared memory): the call fails with invalid_argument before any buffer is
    allocated instead of computing garbage."""
    cfg = fse.make_config(1.0, 220.0, 0.02, 968, 24)
    assert cfg.D == 2018
    with pytest.raises(fse.InvalidArgument):
        ctx.xscale_probe(cfg, 0, None, 1, np.array([0], np.int32), np.array([0], np.int32))
    ctx.trim()


def test_xpass_real_green_cfg2(fse, ctx):
    """Same check with the real mollified Green's table of cfg2 (D = 624)."""
    cfg = fse.make_config(1.0, 110.0, 0.045, 288, 24)
    g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    ky, kz = columns(cfg, np.random.default_rng(3))
    got, gcol = ctx.xscale_probe(cfg, 0, g, 77, ky, kz)
    want = expected(cfg, 0, 77, ky, kz, gcol)
    assert np.abs(got - want).max() / np.abs(want).max() <= 1e-12
    full_row = g.fourier[:, ky[5], kz[5]]
    assert np.array_equal(gcol[5], full_row)
