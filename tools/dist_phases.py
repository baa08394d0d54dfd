"""Per-rank work of the partitioned multi-GPU evaluation, measured on ONE GPU:
G virtual ranks run in sequence (fse_cuda_dist_virtual_total_sum with a
profile), each step timed with its rank alone on the device, plus the bytes
each rank sends per step.  A G-GPU step is then estimated as
    sum over steps of max over ranks (time) + max over ranks (bytes) / BW
(BW = 700 GB/s per GPU and direction, NVLink 5 through NVSwitch, derated from
900).  No kernel waits on another rank here (B200_PROFILING.md: never emulate
ranks that wait on each other on one GPU).

    python tools/dist_phases.py cfg2 [1 2 4 8]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1607_04808_b200 as fse  # noqa: E402

STEPS = ["classify", "pack", "forward", "scale", "inverse", "finish"]
BW = 700e9


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    Gs = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    w = bench.WORKLOADS[name]
    ctx = fse.Context(0)
    s, tgt = fse.generate_workload(w["wl"], w["n"], bench.SEED)
    cfg = bench.workload_config(w, s.strengths, fse)
    g = ctx.precompute_mollified_green(int(fse.green_kind_for(w["kind"])), cfg.Ltilde, cfg.Mtilde,
                                       cfg.sf)
    t = s.positions if tgt is None else tgt
    tas = tgt is None
    ctx.dist_virtual_total_sum(s, w["kind"], cfg, t, g, 1, targets_are_sources=tas)  # warm
    out = {}
    for G in Gs:
        prof = np.zeros((G, 6, 2))
        ctx.dist_virtual_total_sum(s, w["kind"], cfg, t, g, G, targets_are_sources=tas,
                                   profile=prof)
        prof = np.zeros((G, 6, 2))
        ctx.dist_virtual_total_sum(s, w["kind"], cfg, t, g, G, targets_are_sources=tas,
                                   profile=prof)
        tmax = prof[:, :, 0].max(axis=0)
        bmax = prof[:, :, 1].max(axis=0)
        est = tmax.sum() + (bmax.sum() / BW) * 1e3
        out[G] = {"step_ms_max_over_ranks": dict(zip(STEPS, np.round(tmax, 3).tolist())),
                  "bytes_max_over_ranks": dict(zip(STEPS, bmax.tolist())),
                  "compute_ms": round(float(tmax.sum()), 3),
                  "exchange_ms_at_700GBs": round(float(bmax.sum() / BW * 1e3), 3),
                  "estimated_step_ms": round(float(est), 3)}
        print(G, json.dumps(out[G]), flush=True)
        if os.environ.get("FSE_PHASES_VERBOSE"):
            for r in range(G):
                print("  rank", r, "ms", np.round(prof[r, :, 0], 2).tolist(), "MB",
                      np.round(prof[r, :, 1] / 1e6, 1).tolist(), flush=True)
        ctx.trim()
    base = out[Gs[0]]["estimated_step_ms"] * Gs[0]
    for G in Gs:
        print(f"G={G}: estimated {out[G]['estimated_step_ms']:.2f} ms, "
              f"strong-scaling efficiency vs G={Gs[0]}: "
              f"{base / (G * out[G]['estimated_step_ms']):.2f}")


if __name__ == "__main__":
    main()
