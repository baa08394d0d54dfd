"""cfg5's tolerance-consistent variant on the GPU: select_parameters(xi = 220,
tol = 1e-10) -> M = 834, D = 1730 = 2 x 5 x 173 (generic Stockham stage of radix
173, ~135 GB of HBM).  Prints timings and the relative RMS error against the
O(N^2) direct sum on sampled targets.  Usage: python tools/cfg5t_probe.py [nsample]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_04808_b200 as fse


def main():
    ns = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    ctx = fse.Context(0)
    s, tgt = fse.generate_workload(fse.WL_UNIFORM_TARGETS, 8_000_000, 20260101)
    Q = fse.strength_quadratic_sum(s)
    cfg, feasible = fse.select_parameters(0, s.size(), 1.0, Q, 220.0, 1e-10)
    print("cfg5t", dict(M=cfg.M, P=cfg.P, rc=cfg.rc, D=cfg.D, feasible=feasible), flush=True)
    t0 = time.time()
    g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    print("green precompute s", time.time() - t0, flush=True)
    out = {}
    for rep in range(2):
        t0 = time.time()
        tm = fse.StageTimings()
        u = ctx.total_sum(s, 0, cfg, tgt, g, timings=tm)
        out = dict(wall_s=time.time() - t0, spread=tm.spread, fft=tm.fft, scale=tm.scale,
                   quadrature=tm.quadrature, realspace=tm.realspace, total=tm.total)
        print("call", rep, out, flush=True)
    idx = np.sort(np.random.default_rng(4).choice(tgt.shape[0], ns, replace=False))
    ref = ctx.direct_sum(s, 0, tgt[idx], False)
    err = fse.rms_error(u[idx], ref, True)
    out.update(rel_rms_vs_direct=err, nsample=ns, M=cfg.M, D=cfg.D, rc=cfg.rc, P=cfg.P)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
