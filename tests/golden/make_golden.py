"""Regenerate tests/golden/golden_small.npz from the REFERENCE itself
(oracle/_ref/libfse_ref.so = /root/reference/proj/src compiled unmodified by
oracle/Makefile).  Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

Fixture contents (all float64 unless noted), config make_config(1, 6, 0.3, 12, 8)
(Mtilde 20, D 40), N = 200 seeded points, for each kind k in {0, 1, 2}:
  pos_k, str_k           inputs (targets = sources)
  tgt_k                  60 distinct targets
  total_k, fourier_k     fse::total_sum / fourier_sum at the sources
  fourier_tgt_k          fourier_sum at the distinct targets
  real_k                 real_space_sum(xi=6, rc=0.3) at the sources
  direct_k               direct_sum(exclude_self)
  spread_k               spread() grid (deterministic=true)
  i0_k (int32)           not from the reference (its support index is internal)
plus green_0 / green_1 (harmonic / biharmonic tables, 40^3) and the cell list
bstart_c / perm_c (int64) of pos_0 at rc = 0.1.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refimpl as R  # noqa: E402

ARGS = (1.0, 6.0, 0.3, 12, 8)
N, NT = 200, 60


def main():
    rng = np.random.default_rng(1607_04808)
    cfg = R.make_config(*ARGS)
    out = {"args": np.array(ARGS)}
    greens = {g: R.precompute_green(g, cfg.Ltilde, cfg.Mtilde, cfg.sf) for g in (0, 1)}
    out["green_0"], out["green_1"] = greens[0], greens[1]
    for k in (0, 1, 2):
        pos = rng.uniform(0.02, 0.98, (N, 3))
        st = rng.standard_normal((N, R.arity(k)))
        tgt = rng.uniform(0, 1, (NT, 3))
        G = greens[R.green_kind_for(k)]
        out[f"pos_{k}"], out[f"str_{k}"], out[f"tgt_{k}"] = pos, st, tgt
        out[f"total_{k}"] = R.total_sum(cfg, k, pos, st, pos, G)
        out[f"fourier_{k}"] = R.fourier_sum(cfg, k, pos, st, pos, G)
        out[f"fourier_tgt_{k}"] = R.fourier_sum(cfg, k, pos, st, tgt, G)
        out[f"real_{k}"] = R.real_space_sum(k, pos, st, 1.0, cfg.xi, cfg.rc, pos)
        out[f"direct_{k}"] = R.direct_sum(k, pos, st, 1.0, pos, True)
        out[f"spread_{k}"] = R.spread(cfg, k, pos, st, deterministic=True)
    cl = R.build_cell_list(out["pos_0"], 1.0, 0.1)
    out["bstart_c"], out["perm_c"] = cl["bstart"], cl["perm"]
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_small.npz"))


if __name__ == "__main__":
    main()
