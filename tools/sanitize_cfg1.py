"""One small total_sum per kernel (cfg1-like sizes) for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_cfg1.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_04808_b200 as fse  # noqa: E402

ctx = fse.Context(0)
rng = np.random.default_rng(3)
for kind, args in ((0, (1.0, 28.0, 0.15, 80, 16)), (1, (1.0, 20.0, 0.2, 40, 16)),
                   (2, (1.0, 28.0, 0.15, 48, 16))):
    n = 3000
    s = fse.SourceSystem(rng.random((n, 3)), rng.standard_normal((n, fse.strength_arity(kind))))
    cfg = fse.make_config(*args)
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(kind)), cfg.Ltilde, cfg.Mtilde, cfg.sf)
    u = ctx.total_sum(s, kind, cfg, s.positions, g)
    v = ctx.dist_virtual_total_sum(s, kind, cfg, s.positions, g, 3, targets_are_sources=True)
    print(kind, float(np.abs(u - v).max() / np.abs(u).max()))
print("sanitize run done")
