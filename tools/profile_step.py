"""One warm-up + N steps of the hot path on a BASELINE workload, for ncu.

    python tools/profile_step.py [cfg2] [steps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1607_04808_b200 as fse  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    w = bench.WORKLOADS[name]
    ctx = fse.Context(0)
    s, tgt = fse.generate_workload(w["wl"], w["n"], bench.SEED)
    cfg = fse.make_config(1.0, w["xi"], w["rc"], w["M"], w["P"])
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(w["kind"])), cfg.Ltilde,
                                       cfg.Mtilde, cfg.sf)
    t = s.positions if tgt is None else tgt
    for _ in range(1 + steps):
        u = ctx.total_sum(s, w["kind"], cfg, t, g, targets_are_sources=1 if tgt is None else 0)
    print(name, "ok", u[0], ctx.kernel_ms())


if __name__ == "__main__":
    main()
