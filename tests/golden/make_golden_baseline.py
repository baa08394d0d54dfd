"""Golden velocities at the BASELINE.json configurations, written by the
REFERENCE itself (oracle/_ref/libfse_ref.so = /root/reference/proj/src compiled
unmodified by oracle/Makefile; FFTs through oracle/fftw_shim).  Run in the
build container (needs /root/reference and ~45 GB of host RAM for cfg4t):

    python tests/golden/make_golden_baseline.py [case ...]

Inputs are the SURVEY 8(d) workload streams from the reference-side generator
(oracle/ref_capi.cpp ref_generate_workload, seed 20260101 = bench.py's SEED);
tests/test_oracle_generators.py shows the product generator reproduces them
bit for bit, and each fixture stores sha256 digests of the inputs so the GPU
test proves it evaluated the same system.

For each case the reference's fse::total_sum (ewald.cpp:394-415) runs over ALL
targets (= the sources, so the stokeslet self term is applied exactly as in
production) with the reference's own precomputed Green's table
(greens.cpp:48-113).  Stored (baseline_<case>.npz):
  rows (int64)        seeded subset of target indices (all targets for cfg1)
  u_rows              total_sum velocities at those targets
  umax                max |u| over ALL targets (the max-rel denominator)
  usum                column sums of u over all targets (a checksum)
  drows, u_direct     1024 sampled targets and the reference's O(N^2) direct_sum
                      there (kernels.cpp:59-82; coincident self pair excluded)
  u_drows             total_sum velocities at drows
  dims, cell_side, bstart_sha, perm_sha
                      build_cell_list(sources, rc) (realspace.cpp:65-84):
                      sha256 of the int64 bucket starts and bucket-ordered indices
  pos_sha, str_sha    sha256 of the float64 inputs
  timings             the reference's StageTimings for this call (s, 8 threads)
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refimpl as R  # noqa: E402

SEED = 20260101
# name: (kind, workload, n, xi, rc, M, P, tol, subset rows)
#   rc = None -> the reference's select_parameters at (xi, tol) (estimates.cpp:81-126):
#   the tolerance-consistent variants of SURVEY 8(d)
CASES = {
    "cfg1": (0, 1, 10_000, 28.0, 0.15, 80, 16, 1e-8, None),
    "cfg2": (0, 1, 1_000_000, 110.0, 0.045, 288, 24, 1e-10, 8192),
    "cfg3": (1, 3, 100_000, 40.0, 0.12, 128, 20, 1e-8, 8192),
    "cfg4": (2, 4, 1_000_000, 110.0, 0.045, 288, 24, 1e-10, 8192),
    "cfg1t": (0, 1, 10_000, 28.0, None, None, None, 1e-8, None),
    "cfg3t": (1, 3, 100_000, 40.0, None, None, None, 1e-8, 8192),
    "cfg4t": (2, 4, 1_000_000, 110.0, None, None, None, 1e-10, 8192),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def quadratic_sum(st):
    """strength_quadratic_sum (kernels.cpp:105-110): sequential sum of c_i^2."""
    return float(np.cumsum((st * st).ravel())[-1])


def direct_at(kind, pos, st, rows):
    """direct_sum at targets pos[rows] with each target's own source excluded:
    the other sources as one system, plus the subset's own points with
    exclude_self (index match) -- direct_sum is linear in the sources."""
    mask = np.ones(pos.shape[0], bool)
    mask[rows] = False
    tgt = pos[rows]
    u = R.direct_sum(kind, pos[mask], st[mask], 1.0, tgt, False)
    u += R.direct_sum(kind, pos[rows], st[rows], 1.0, tgt, True)
    return u


def make(name):
    kind, wl, n, xi, rc, M, P, tol, nrows = CASES[name]
    pos, st, _ = R.generate_workload(wl, n, SEED)
    if rc is None:
        cfg, feas = R.select_parameters(kind, n, 1.0, quadratic_sum(st), xi, tol)
        assert feas, name
    else:
        cfg = R.make_config(1.0, xi, rc, M, P)
    t0 = time.time()
    green = R.precompute_green(R.green_kind_for(kind), cfg.Ltilde, cfg.Mtilde, cfg.sf)
    tg = time.time() - t0
    tm = {}
    u = R.total_sum(cfg, kind, pos, st, pos, green, timings=tm)
    del green
    rng = np.random.default_rng(SEED + n)
    rows = np.arange(n) if nrows is None else np.sort(rng.choice(n, nrows, replace=False))
    drows = np.sort(rng.choice(n, min(1024, n), replace=False))
    t1 = time.time()
    ud = direct_at(kind, pos, st, drows)
    td = time.time() - t1
    cl = R.build_cell_list(pos, 1.0, cfg.rc)
    out = dict(
        kind=kind, workload=wl, n=n, seed=SEED, tol=tol,
        args=np.array([1.0, cfg.xi, cfg.rc, cfg.M, cfg.P]),
        Mtilde=cfg.Mtilde,
        rows=rows.astype(np.int64), u_rows=u[rows], umax=np.abs(u).max(), usum=u.sum(axis=0),
        drows=drows.astype(np.int64), u_direct=ud, u_drows=u[drows],
        dims=cl["dims"].astype(np.int64), cell_side=cl["cell_side"],
        bstart_sha=sha(cl["bstart"].astype(np.int64)), perm_sha=sha(cl["perm"].astype(np.int64)),
        pos_sha=sha(pos), str_sha=sha(st),
        timings=np.array([tm[k] for k in ("spread", "fft", "scale", "quadrature", "realspace",
                                          "total")]),
    )
    path = os.path.join(HERE, f"baseline_{name}.npz")
    np.savez_compressed(path, **out)
    err = np.sqrt(((u[drows] - ud) ** 2).sum() / (ud ** 2).sum())
    print(f"{name}: D={2 * cfg.Mtilde} rc={cfg.rc:.6g} M={cfg.M} green {tg:.1f}s total_sum "
          f"{tm['total']:.1f}s direct {td:.1f}s  rel-rms vs direct {err:.3e} -> {path}",
          flush=True)


def main():
    names = sys.argv[1:] or list(CASES)
    R.set_threads(os.cpu_count() or 1)
    for nm in names:
        make(nm)


if __name__ == "__main__":
    main()
