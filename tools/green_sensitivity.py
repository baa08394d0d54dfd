"""How sensitive is fourier_sum to rounding-level noise in the Green's table?
Uploads the reference's own table (oracle/_ref) and the same table with
relative-to-max noise of a few ulp added, and compares the GPU fourier sums.
Diagnostics only.   python tools/green_sensitivity.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1607_04808_b200 as fse  # noqa: E402
from oracle import refimpl as R  # noqa: E402

ctx = fse.Context(0)
R.set_threads(os.cpu_count() or 1)
args = (1.0, 110.0, 0.045, 288, 24)
pos, st, _ = R.generate_workload(1, 100_000, 20260101)
tgt = pos[:4000]
cfg = fse.make_config(*args)
rcfg = R.make_config(*args)
G = R.precompute_green(1, rcfg.Ltilde, rcfg.Mtilde, rcfg.sf)
s = fse.SourceSystem(pos, st, 1.0)
g0 = ctx.upload_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, G)
u0 = ctx.fourier_sum(s, cfg, 0, tgt, g0)
scale = np.abs(u0).max()
rng = np.random.default_rng(0)
gmax = np.abs(G).max()
for eps in (1e-17, 1e-16, 4e-16):
    Gp = G + eps * gmax * rng.standard_normal(G.shape)
    gp = ctx.upload_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, Gp)
    u = ctx.fourier_sum(s, cfg, 0, tgt, gp)
    print(f"absolute table noise {eps:.0e} x max|G|: fourier max-rel change "
          f"{np.abs(u - u0).max() / scale:.3e}", flush=True)
    gp.free()
# relative (per-entry) noise instead: the same ulps relative to each entry
for eps in (1e-16, 1e-15):
    Gp = G * (1.0 + eps * rng.standard_normal(G.shape))
    gp = ctx.upload_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, Gp)
    u = ctx.fourier_sum(s, cfg, 0, tgt, gp)
    print(f"relative table noise {eps:.0e}: fourier max-rel change "
          f"{np.abs(u - u0).max() / scale:.3e}", flush=True)
    gp.free()
g1 = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
G1 = g1.fourier
d = np.abs(G1 - G)
for lo, hi in ((0, 100), (100, 200), (200, 312)):
    kk = np.arange(624)
    kk = np.minimum(kk, 624 - kk)
    m = (kk[:, None, None] >= lo) & (kk[:, None, None] < hi)
    m = m & (kk[None, :, None] < hi) & (kk[None, None, :] < hi)
    sel = np.broadcast_to(m, G.shape)
    print(f"|kx| in [{lo},{hi}): max |dG| {d[sel].max():.3e}, max |G| {np.abs(G[sel]).max():.3e},"
          f" median rel {np.median(d[sel] / np.abs(G[sel])):.3e}")
