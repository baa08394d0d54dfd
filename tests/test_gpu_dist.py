"""The partitioned multi-GPU evaluation (fse_dist): particles
split by x-slab owner, ghost sources (spread supports crossing slab faces,
real-space neighbours within rc) and ghost targets (quadrature shares)
exchanged, the FFT distributed by two spectrum transposes, ghost partial sums
returned to the owners -- run as G virtual ranks on one GPU with device-copy
exchanges (fse_cuda_dist_virtual_total_sum; a kernel never waits on another
rank).  It must reproduce the one-GPU total_sum for every kernel, for
targets == sources (self term on the owner) and distinct targets, uniform and
clustered inputs, uneven and empty slabs (G = 5, 8, 16 at small Mtilde)."""
import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu


def system(fse, rng, kind, n, clustered=False):
    if clustered:
        c = rng.uniform(0.3, 0.7, (4, 3))
        pos = np.clip(c[np.arange(n) % 4] + 0.05 * rng.standard_normal((n, 3)), 0,
                      np.nextafter(1, 0))
    else:
        pos = rng.uniform(0, 1, (n, 3))
    return fse.SourceSystem(pos, rng.standard_normal((n, fse.strength_arity(kind))), 1.0)


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("G", [1, 2, 3, 5])
@pytest.mark.parametrize("distinct", [False, True])
def test_virtual_ranks_match_one_gpu(fse, ctx, rng, kind, G, distinct):
    cfg = fse.make_config(1.0, 12.0, 0.25, 48, 16)
    s = system(fse, rng, kind, 3000)
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(kind)), cfg.Ltilde, cfg.Mtilde,
                                       cfg.sf)
    tgt = rng.uniform(0, 1, (2000, 3)) if distinct else s.positions
    want = ctx.total_sum(s, kind, cfg, tgt, g, targets_are_sources=0 if distinct else 1)
    got = ctx.dist_virtual_total_sum(s, kind, cfg, tgt, g, G, targets_are_sources=not distinct)
    assert rel_max(got, want) <= 1e-12


@pytest.mark.parametrize("G", [2, 8, 16])
def test_virtual_ranks_clustered_and_empty_slabs(fse, ctx, rng, G):
    # Mtilde = 72 with G = 16: 8-plane slabs, the last ones empty
    cfg = fse.make_config(1.0, 20.0, 0.15, 56, 16)
    s = system(fse, rng, 0, 6000, clustered=True)
    g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    want = ctx.total_sum(s, 0, cfg, s.positions, g, targets_are_sources=1)
    got = ctx.dist_virtual_total_sum(s, 0, cfg, s.positions, g, G, targets_are_sources=True)
    assert rel_max(got, want) <= 1e-12


def test_virtual_ranks_cfg2_full_size(fse, ctx):
    """cfg2 (N = 1e6, D = 624) split over 4 virtual ranks."""
    s, _ = fse.generate_workload(fse.WL_UNIFORM, 1_000_000, 20260101)
    cfg = fse.make_config(1.0, 110.0, 0.045, 288, 24)
    g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    want = ctx.total_sum(s, 0, cfg, s.positions, g, targets_are_sources=1)
    got = ctx.dist_virtual_total_sum(s, 0, cfg, s.positions, g, 4, targets_are_sources=True)
    assert rel_max(got, want) <= 1e-12
    ctx.trim()


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_multi_device_context_one_gpu(fse, ctx, rng, kind):
    """fse_cuda_multi_* (one process, ncclCommInitAll, a host thread per device,
    host buffers in and out) on the one GPU the pool provides: the partition,
    the NCCL steps and the scatter back to caller order, against total_sum;
    with the caller's Green's table uploaded and with the per-device precompute."""
    cfg = fse.make_config(1.0, 12.0, 0.25, 48, 16)
    s = system(fse, rng, kind, 3000)
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(kind)), cfg.Ltilde, cfg.Mtilde,
                                       cfg.sf)
    want = ctx.total_sum(s, kind, cfg, s.positions, g)
    m = fse.MultiContext([0])
    got = m.total_sum(s, kind, cfg, s.positions)
    assert rel_max(got, want) <= 1e-12
    got2 = m.total_sum(s, kind, cfg, s.positions, green_full=g.fourier)
    assert rel_max(got2, want) <= 1e-12
    tgt = rng.uniform(0, 1, (500, 3))
    want_t = ctx.total_sum(s, kind, cfg, tgt, g)
    assert rel_max(m.total_sum(s, kind, cfg, tgt), want_t) <= 1e-12
    bad = fse.SourceSystem(np.vstack([s.positions, [[0.5, 0.5, 7.0]]]),
                           np.vstack([s.strengths, s.strengths[:1]]), 1.0)
    with pytest.raises(fse.InvalidArgument):
        m.total_sum(bad, kind, cfg, bad.positions)
    m.close()
