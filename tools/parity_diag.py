"""Where does GPU-vs-reference disagreement come from?  Splits total_sum into
its parts at a BASELINE config and compares each with the reference
(oracle/_ref): Green's table, fourier_sum (GPU table and reference table
uploaded), real_space_sum.  Diagnostics only (needs the GPU and oracle/_ref).
    python tools/parity_diag.py cfg1 [cfg2 ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1607_04808_b200 as fse  # noqa: E402
from oracle import refimpl as R  # noqa: E402

CFG = {"cfg1": (0, 1, 10_000, (1.0, 28.0, 0.15, 80, 16)),
       "cfg2": (0, 1, 1_000_000, (1.0, 110.0, 0.045, 288, 24)),
       "cfg2s": (0, 1, 100_000, (1.0, 110.0, 0.045, 288, 24)),
       "cfg4": (2, 4, 1_000_000, (1.0, 110.0, 0.045, 288, 24))}


def rel(a, b, scale):
    return float(np.abs(a - b).max() / scale)


def main():
    ctx = fse.Context(0)
    R.set_threads(os.cpu_count() or 1)
    for name in sys.argv[1:]:
        kind, wl, n, args = CFG[name]
        pos, st, _ = R.generate_workload(wl, n, 20260101)
        rng = np.random.default_rng(1)
        rows = np.sort(rng.choice(n, min(n, 4000), replace=False))
        tgt = pos[rows]
        cfg = fse.make_config(*args)
        rcfg = R.make_config(*args)
        gk = int(fse.green_kind_for(kind))
        G_ref = R.precompute_green(gk, rcfg.Ltilde, rcfg.Mtilde, rcfg.sf)
        g_gpu = ctx.precompute_mollified_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.sf)
        G_gpu = g_gpu.fourier
        print(f"{name}: green max-rel {rel(G_gpu, G_ref, np.abs(G_ref).max()):.3e}", flush=True)
        g_up = ctx.upload_mollified_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, G_ref)
        s = fse.SourceSystem(pos, st, 1.0)
        uF_ref = R.fourier_sum(rcfg, kind, pos, st, tgt, G_ref)
        uF_gpu = ctx.fourier_sum(s, cfg, kind, tgt, g_gpu)
        uF_gpu_rt = ctx.fourier_sum(s, cfg, kind, tgt, g_up)
        uR_ref = R.real_space_sum(kind, pos, st, 1.0, cfg.xi, cfg.rc, tgt)
        uR_gpu = ctx.real_space_sum(s, kind, cfg.xi, cfg.rc, tgt)
        scale = np.abs(uF_ref + uR_ref).max()
        print(f"  fourier (gpu table)  max-rel {rel(uF_gpu, uF_ref, scale):.3e}")
        print(f"  fourier (ref table)  max-rel {rel(uF_gpu_rt, uF_ref, scale):.3e}")
        print(f"  real space           max-rel {rel(uR_gpu, uR_ref, scale):.3e}")
        print(f"  |uF|max {np.abs(uF_ref).max():.3e} |uR|max {np.abs(uR_ref).max():.3e}",
              flush=True)


if __name__ == "__main__":
    main()
