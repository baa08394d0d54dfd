"""Golden vectors written by the reference itself (tests/golden/make_golden.py,
oracle/_ref).  CPU: the C oracle reproduces them.  GPU (-m gpu): the CUDA
path through the C-ABI reproduces them, with no reference present at run time."""
import os

import numpy as np
import pytest

from conftest import rel_max

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_small.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _cfg(mod, gold):
    a = gold["args"]
    return mod.make_config(float(a[0]), float(a[1]), float(a[2]), int(a[3]), int(a[4]))


# --------------------------------------------------------------- CPU: oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_oracle_matches_golden(oracle, gold, kind):
    cfg = _cfg(oracle, gold)
    gk = oracle.green_kind_for(kind)
    G = oracle.precompute_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    assert rel_max(G, gold[f"green_{gk}"]) <= 1e-14
    pos, st, tgt = gold[f"pos_{kind}"], gold[f"str_{kind}"], gold[f"tgt_{kind}"]
    assert rel_max(oracle.total_sum(cfg, kind, pos, st, pos, G), gold[f"total_{kind}"]) <= 1e-14
    assert rel_max(oracle.fourier_sum(cfg, kind, pos, st, tgt, G),
                   gold[f"fourier_tgt_{kind}"]) <= 1e-14
    assert np.array_equal(oracle.real_space_sum(kind, pos, st, 1.0, cfg.xi, cfg.rc, pos),
                          gold[f"real_{kind}"])
    assert rel_max(oracle.spread(cfg, kind, pos, st), gold[f"spread_{kind}"]) <= 1e-14
    assert rel_max(oracle.direct_sum(kind, pos, st, pos, True), gold[f"direct_{kind}"]) <= 1e-15


def test_oracle_cell_list_golden(oracle, gold):
    cl = oracle.build_cell_list(gold["pos_0"], 1.0, 0.1)
    assert np.array_equal(cl["bstart"], gold["bstart_c"])
    assert np.array_equal(cl["perm"], gold["perm_c"])


# --------------------------------------------------------------- GPU: product
@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_gpu_matches_golden(fse, ctx, gold, kind):
    cfg = _cfg(fse, gold)
    gk = int(fse.green_kind_for(kind))
    green = ctx.precompute_mollified_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    assert rel_max(green.fourier, gold[f"green_{gk}"]) <= 1e-13
    s = fse.SourceSystem(gold[f"pos_{kind}"], gold[f"str_{kind}"], 1.0)
    tgt = gold[f"tgt_{kind}"]
    assert rel_max(ctx.total_sum(s, kind, cfg, s.positions, green), gold[f"total_{kind}"]) <= 1e-11
    assert rel_max(ctx.fourier_sum(s, cfg, kind, s.positions, green),
                   gold[f"fourier_{kind}"]) <= 1e-11
    assert rel_max(ctx.fourier_sum(s, cfg, kind, tgt, green), gold[f"fourier_tgt_{kind}"]) <= 1e-11
    ur = ctx.real_space_sum(s, kind, cfg.xi, cfg.rc, s.positions)
    want = gold[f"real_{kind}"]
    assert np.all(np.linalg.norm(ur - want, axis=1) <= 1e-13 * (1 + np.linalg.norm(want, axis=1)))
    assert rel_max(ctx.spread(s, cfg, kind), gold[f"spread_{kind}"]) <= 1e-13
    assert rel_max(ctx.direct_sum(s, kind, s.positions, True), gold[f"direct_{kind}"]) <= 1e-13


@pytest.mark.gpu
def test_gpu_cell_list_golden(fse, ctx, gold):
    cl = ctx.build_cell_list(fse.SourceSystem(gold["pos_0"], gold["str_0"], 1.0), 0.1)
    assert np.array_equal(cl.bstart, gold["bstart_c"])
    assert np.array_equal(cl.perm, gold["perm_c"])
