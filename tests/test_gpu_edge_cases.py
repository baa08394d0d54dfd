"""Edge cases of the hot path against the C oracle (GPU): a single source and
target, points on the box faces (0 and L, the support clamp at the grid
edge), an empty target set, coincident sources (r = 0 pairs are excluded
from the real-space sum, realspace.cpp:140), every point in one cell (the
largest real-space work item), and targets placed exactly on grid nodes and
half-nodes (support-start ties)."""
import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu

ARGS = (1.0, 8.0, 0.3, 24, 16)


def _green(fse, ctx, oracle, kind, cfg):
    gk = int(fse.green_kind_for(kind))
    table = oracle.precompute_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    return ctx.upload_mollified_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, table), table


def _check(fse, ctx, oracle, kind, pos, st, tgt, tol=1e-11):
    cfg = fse.make_config(*ARGS)
    ocfg = oracle.make_config(*ARGS)
    g, table = _green(fse, ctx, oracle, kind, cfg)
    s = fse.SourceSystem(pos, st, 1.0)
    got = ctx.total_sum(s, kind, cfg, tgt, g)
    want = oracle.total_sum(ocfg, kind, s.positions, s.strengths, tgt, table)
    assert got.shape == want.shape
    assert np.isfinite(got).all()
    if want.size:
        assert rel_max(got, want) <= tol, rel_max(got, want)
    return got


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_single_source_single_target(fse, ctx, oracle, rng, kind):
    a = fse.strength_arity(kind)
    _check(fse, ctx, oracle, kind, [[0.4, 0.55, 0.6]], rng.standard_normal((1, a)),
           np.array([[0.45, 0.5, 0.62]]))


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_points_on_box_faces(fse, ctx, oracle, rng, kind):
    n = 200
    pos = rng.uniform(0, 1, (n, 3))
    pos[: n // 4, 0] = 0.0
    pos[n // 4: n // 2, 1] = 1.0
    pos[n // 2: 3 * n // 4, 2] = 0.0
    pos[-5:] = [[0, 0, 0], [1, 1, 1], [0, 1, 0], [1, 0, 1], [0.5, 0.0, 1.0]]
    _check(fse, ctx, oracle, kind, pos, rng.standard_normal((n, fse.strength_arity(kind))), pos)


def test_empty_targets(fse, ctx, oracle, rng):
    pos = rng.uniform(0, 1, (50, 3))
    got = _check(fse, ctx, oracle, 0, pos, rng.standard_normal((50, 3)), np.zeros((0, 3)))
    assert got.shape == (0, 3)


@pytest.mark.parametrize("kind", [0, 2])
def test_coincident_sources(fse, ctx, oracle, rng, kind):
    base = rng.uniform(0.2, 0.8, (40, 3))
    pos = np.concatenate([base, base[:10], base[:3]])
    st = rng.standard_normal((pos.shape[0], 3))
    _check(fse, ctx, oracle, kind, pos, st, pos)


def test_all_points_in_one_cell(fse, ctx, oracle, rng):
    # rc = 0.3 -> cells of side 1/3; 700 points inside one cell and its targets
    pos = rng.uniform(0.34, 0.66, (700, 3))
    _check(fse, ctx, oracle, 0, pos, rng.standard_normal((700, 3)), pos)


def test_targets_on_grid_nodes_and_half_nodes(fse, ctx, oracle, rng):
    cfg = fse.make_config(*ARGS)
    nodes = (np.arange(4, cfg.M - 4) * cfg.h)[:, None] * np.ones((1, 3))
    half = nodes + 0.5 * cfg.h
    tgt = np.concatenate([nodes, half])
    pos = rng.uniform(0, 1, (300, 3))
    _check(fse, ctx, oracle, 0, pos, rng.standard_normal((300, 3)), tgt)


def test_total_sum_into_pinned_output(fse, ctx, oracle, rng):
    """total_sum(out=...) writes the same velocities into a caller's (pinned)
    array; a wrong shape/dtype is rejected before any work."""
    cfg = fse.make_config(*ARGS)
    g, _ = _green(fse, ctx, oracle, 0, cfg)
    pos = rng.random((300, 3))
    s = fse.SourceSystem(pos, rng.standard_normal((300, 3)), 1.0)
    want = ctx.total_sum(s, 0, cfg, pos, g)
    hu = ctx.host_alloc((300, 3))
    got = ctx.total_sum(s, 0, cfg, pos, g, out=hu)
    assert got is hu
    assert np.array_equal(hu, want)
    with pytest.raises(fse.InvalidArgument):
        ctx.total_sum(s, 0, cfg, pos, g, out=np.empty((299, 3)))
