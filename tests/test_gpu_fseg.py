"""FSEG Green's-table cache (greens.cpp:141-203) on the GPU path
(fse_cuda_green_save / fse_cuda_green_load), after the reference suite's
round-trip test (proj/tests/test_greens.cpp:180-206) plus cross-loads in both
directions with the reference's own save/load (oracle/_ref):

- a file written by the reference (tests/golden/fseg_ref_*_Mt10.bin) loads with
  the same header fields; the device keeps the half table D x D x (D/2+1)
  (the hot path's layout), so the payload comes back bit-exact on kz <= D/2 and
  the other half is the even extension (the reference's table is even to
  ~6e-17 relative, not bitwise: it is the real part of a forward FFT);
- GPU save -> GPU load -> GPU save is byte-identical (the reference's round
  trip);
- the reference loads a GPU-written file and gets the GPU table;
- the GPU precompute agrees with the reference table at 1e-13 of its max;
- malformed files raise the runtime error the reference raises
  (std::runtime_error), and an unknown kind byte is rejected."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SF = 1.0 + math.sqrt(3.0)


def ref_file(nm):
    return os.path.join(HERE, "golden", f"fseg_ref_{nm}_Mt10.bin")


@pytest.mark.parametrize("nm,gk", [("harm", 0), ("biharm", 1)])
def test_load_reference_written_file(fse, ctx, ref, nm, gk):
    g = ctx.load_mollified_green(ref_file(nm))
    k2, Lt, h, R, Mt, want = ref.load_green(ref_file(nm))
    assert (int(g.kind), g.Ltilde, g.h, g.R, g.Mtilde) == (k2, Lt, h, R, Mt)
    got = g.fourier
    D = 2 * Mt
    assert np.array_equal(got[:, :, : D // 2 + 1], want[:, :, : D // 2 + 1])
    assert np.abs(got - want).max() <= 1e-15 * np.abs(want).max()


@pytest.mark.parametrize("gk", [0, 1])
def test_round_trip_and_reference_reads_gpu_file(fse, ctx, ref, tmp_path, gk):
    g = ctx.precompute_mollified_green(gk, 1.25, 10, SF)
    table = g.fourier
    k2, Lt, h, R, Mt, want = ref.load_green(ref_file("harm" if gk == 0 else "biharm"))
    assert np.abs(table - want).max() <= 1e-13 * np.abs(want).max()
    p1, p2 = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    ctx.save_mollified_green(g, p1)
    g2 = ctx.load_mollified_green(p1)
    assert np.array_equal(g2.fourier, table)
    ctx.save_mollified_green(g2, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    k3, Lt3, h3, R3, Mt3, back = ref.load_green(p1)
    assert (k3, Lt3, h3, R3, Mt3) == (gk, g.Ltilde, g.h, g.R, 10)
    assert np.array_equal(back, table)


def test_malformed_files_raise(fse, ctx, tmp_path):
    good = open(ref_file("biharm"), "rb").read()
    cases = {
        "magic": b"FSEX" + good[4:],
        "version": good[:4] + (2).to_bytes(4, "little") + good[8:],
        "kind": good[:8] + bytes([7]) + good[9:],
        "truncated": good[:-8],
        "extents": good[:33] + (21).to_bytes(8, "little") + good[41:],
    }
    for nm, blob in cases.items():
        p = str(tmp_path / f"{nm}.bin")
        open(p, "wb").write(blob)
        with pytest.raises(fse.FseRuntimeError):
            ctx.load_mollified_green(p)
    with pytest.raises(fse.FseRuntimeError):
        ctx.load_mollified_green(str(tmp_path / "missing.bin"))
