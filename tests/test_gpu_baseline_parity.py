"""Parity with the REFERENCE at the BASELINE.json configurations (north_star:
"velocities within 1e-11 relative max error at N=1e6 ... bit-exact cell
binning and ordering indices ... both also compared against direct O(N^2)
summation at the stated Ewald tolerance").

The golden vectors (tests/golden/baseline_<case>.npz) were written by the
reference's own fse::total_sum (oracle/_ref = /root/reference/proj/src
compiled unmodified; tests/golden/make_golden_baseline.py) over all N
targets of the SURVEY 8(d) workloads.  Here the product path runs the same
call -- fse_cuda_total_sum through the C-ABI with host buffers, targets ==
sources detected by value as in ewald.cpp:405-407 -- at the production
shapes (N = NT = 1e6 on the 624-point register engines and the TMA
quadrature; cfg3's Bluestein x-pass; the tolerance-consistent variants on the
242 / 348 / 704 engines) and is compared on the stored rows:

  max_rows |u_gpu - u_ref| / max_all |u_ref|  <=  1e-11          (north_star bar)
  |sum_all u_gpu - sum_all u_ref|             <=  1e-11 N max|u|  (all targets)
  the GPU cell list: dims, cell_side bit-equal, sha256 of bucket starts and
  bucket-ordered source indices equal to the reference's      (bit-exact binning)
  |err_gpu - err_ref| <= 1e-3 err_ref for the relative RMS error against the
  reference's O(N^2) direct_sum on 1024 sampled targets; for the
  tolerance-consistent variants err_gpu is also reported against the tolerance.

Identical inputs include the Green's table: fse::total_sum takes the
MollifiedGreen as an input (ewald.hpp:75-77), so the reference's own table
(oracle/_ref precompute_mollified_green, computed here on the host) is
uploaded and fed to the GPU path.  The GPU's own precompute agrees with that
table to ~7e-16 of its max (test_gpu_parity / test_gpu_fseg), but the
fourier sum is ill-conditioned in the table's high-k entries (the multiplier's
exp((eta - 1) k^2 / 4 xi^2) with eta = 1.17 at cfg2/cfg4):
rounding-level differences between two table computations move u by ~1e-11
of max |u|.  The production call with the GPU's own table is therefore also
run and checked against the BASELINE tolerance (1e-10), and both numbers are
logged.

Results are appended to $FSE_PARITY_LOG (JSON lines) when set; the round's
numbers are in profiles/ and DESIGN.md section 5."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg1t", "cfg3t", "cfg4t"]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel_rms(u, ref):
    return float(np.sqrt(((u - ref) ** 2).sum() / (ref ** 2).sum()))


def log(rec):
    path = os.environ.get("FSE_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("case", CASES)
def test_total_sum_matches_reference(fse, ctx, ref, case):
    path = os.path.join(HERE, "golden", f"baseline_{case}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing golden fixture {path} (tests/golden/make_golden_baseline.py)")
    g = np.load(path)
    kind, n = int(g["kind"]), int(g["n"])
    s, _ = fse.generate_workload(int(g["workload"]), n, int(g["seed"]))
    assert sha(s.positions) == str(g["pos_sha"]) and sha(s.strengths) == str(g["str_sha"])
    L, xi, rc, M, P = g["args"]
    cfg = fse.make_config(float(L), float(xi), float(rc), int(M), int(P))
    assert cfg.Mtilde == int(g["Mtilde"])
    gk = int(fse.green_kind_for(kind))
    ref.set_threads(os.cpu_count() or 1)
    table = ref.precompute_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    green = ctx.upload_mollified_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, table)
    del table
    u = ctx.total_sum(s, kind, cfg, s.positions, green)  # targets == sources detected by value
    green.free()
    own = ctx.precompute_mollified_green(gk, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    u_own = ctx.total_sum(s, kind, cfg, s.positions, own)
    own.free()
    rows = g["rows"]
    umax = float(g["umax"])
    err = float(np.abs(u[rows] - g["u_rows"]).max() / umax)
    err_own = float(np.abs(u_own[rows] - g["u_rows"]).max() / umax)
    sum_err = float(np.abs(u.sum(axis=0) - g["usum"]).max())

    cl = ctx.build_cell_list(s, cfg.rc)
    cell_ok = (tuple(int(d) for d in g["dims"]) == tuple(cl.dims)
               and cl.cell_side == float(g["cell_side"])
               and sha(cl.bstart.astype(np.int64)) == str(g["bstart_sha"])
               and sha(cl.perm.astype(np.int64)) == str(g["perm_sha"]))

    drows = g["drows"]
    ud = g["u_direct"]
    err_gpu = rel_rms(u[drows], ud)
    err_ref = rel_rms(g["u_drows"], ud)
    err_drows = float(np.abs(u[drows] - g["u_drows"]).max() / umax)
    rec = {"case": case, "kind": kind, "N": n, "D": cfg.D, "max_rel_vs_reference": err,
           "max_rel_vs_reference_own_green": err_own,
           "sum_abs_err": sum_err, "cell_list_bit_exact": cell_ok,
           "rel_rms_vs_direct_gpu": err_gpu, "rel_rms_vs_direct_ref": err_ref,
           "tol": float(g["tol"])}
    log(rec)
    print(json.dumps(rec))
    assert err <= 1e-11 and err_drows <= 1e-11, rec
    assert err_own <= float(g["tol"]) and err_own <= 1e-10, rec
    assert sum_err <= 1e-11 * n * umax, rec
    assert cell_ok, rec
    assert abs(err_gpu - err_ref) <= 1e-3 * err_ref, rec


@pytest.mark.parametrize("case", ["cfg2", "cfg4"])
def test_support_index_bit_exact_full_size(fse, ctx, oracle, case):
    """i0 (ewald.cpp:33-51) of every one of the 1e6 points is bit-exact vs the C
    restatement (itself pinned to the reference by the golden grids)."""
    g = np.load(os.path.join(HERE, "golden", f"baseline_{case}.npz"))
    s, _ = fse.generate_workload(int(g["workload"]), int(g["n"]), int(g["seed"]))
    L, xi, rc, M, P = g["args"]
    cfg = fse.make_config(float(L), float(xi), float(rc), int(M), int(P))
    ocfg = oracle.make_config(float(L), float(xi), float(rc), int(M), int(P))
    got = ctx.support_index(cfg, s.positions)
    want = oracle.support_index(ocfg, s.positions)
    assert np.array_equal(got, want)
