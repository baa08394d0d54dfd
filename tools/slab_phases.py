"""Per-rank phase times of the z-slab decomposition, measured as G virtual
ranks in sequence on one GPU (no exchange cost): what one rank of a G-GPU run
spends in its local phases.

    python tools/slab_phases.py [cfg2] [G ...]
    python tools/slab_phases.py cfg2 8:3      (only rank 3 of 8, once: for ncu)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1607_04808_b200 as fse  # noqa: E402
from paper_1607_04808_b200.slabs import SlabSum  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    args = sys.argv[2:] or ["1", "2", "4", "8"]
    only = None
    if len(args) == 1 and ":" in args[0]:
        G, r = (int(v) for v in args[0].split(":"))
        args, only = [str(G)], r
    Gs = [int(v) for v in args]
    w = bench.WORKLOADS[name]
    ctx = fse.Context(0)
    s, tgt = fse.generate_workload(w["wl"], w["n"], bench.SEED)
    t = s.positions if tgt is None else tgt
    tas = tgt is None
    cfg = fse.make_config(1.0, w["xi"], w["rc"], w["M"], w["P"])
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(w["kind"])), cfg.Ltilde,
                                       cfg.Mtilde, cfg.sf)
    n, nt = s.size(), t.shape[0]
    d_pos = ctx.dev_alloc(s.positions.nbytes)
    d_str = ctx.dev_alloc(s.strengths.nbytes)
    d_tgt = d_pos if tas else ctx.dev_alloc(t.nbytes)
    d_u = ctx.dev_alloc(24 * nt)
    ctx.memcpy(d_pos, s.positions.ctypes.data, s.positions.nbytes)
    ctx.memcpy(d_str, s.strengths.ctypes.data, s.strengths.nbytes)
    if not tas:
        ctx.memcpy(d_tgt, t.ctypes.data, t.nbytes)
    for G in Gs:
        worst = {"forward": 0.0, "scale": 0.0, "inverse": 0.0}
        tot = []
        for r in (range(G) if only is None else [only]):
            ss = SlabSum(ctx, cfg, w["kind"], r, G)
            for rep in range(2 if only is None else 1):  # warm, then timed
                ph = {}
                t0 = time.perf_counter()
                ss.forward(d_pos, d_str, n)
                ph["forward"] = time.perf_counter() - t0
                t0 = time.perf_counter()
                ss.scale(g)
                ph["scale"] = time.perf_counter() - t0
                t0 = time.perf_counter()
                ss.inverse(d_pos, d_str, n, d_tgt, nt, tas, d_u)
                ph["inverse"] = time.perf_counter() - t0
            ss.free()
            for k in worst:
                worst[k] = max(worst[k], ph[k])
            tot.append(sum(ph.values()))
        print(f"G={G}: slowest rank {1e3 * max(tot):.2f} ms (phases max "
              + ", ".join(f"{k} {1e3 * v:.2f}" for k, v in worst.items())
              + f"), mean rank {1e3 * np.mean(tot):.2f} ms", flush=True)
        ctx.trim()


if __name__ == "__main__":
    main()
