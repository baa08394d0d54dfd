"""FSEG cache files (greens.cpp:141-203), CPU side: the reference-written
fixtures (tests/golden/make_fseg.py) parse with the documented layout -- magic
"FSEG", u32 version 1, u8 kind, f64 Ltilde / h / R, three u64 extents, then the
(2 Mtilde)^3 doubles -- and the reference's own loader returns that payload."""
import math
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def parse(path):
    b = open(path, "rb").read()
    assert b[:4] == b"FSEG"
    version, kind = struct.unpack_from("<IB", b, 4)
    Lt, h, R = struct.unpack_from("<3d", b, 9)
    d = struct.unpack_from("<3Q", b, 33)
    payload = np.frombuffer(b, dtype="<f8", offset=57)
    return version, kind, Lt, h, R, d, payload


@pytest.mark.parametrize("nm,gk", [("harm", 0), ("biharm", 1)])
def test_reference_fseg_layout(ref, nm, gk):
    path = os.path.join(HERE, "golden", f"fseg_ref_{nm}_Mt10.bin")
    version, kind, Lt, h, R, d, payload = parse(path)
    assert (version, kind, Lt, d) == (1, gk, 1.25, (20, 20, 20))
    assert h == 1.25 / 10 and R == math.sqrt(3.0) * 1.25
    assert payload.size == 20 ** 3
    k2, Lt2, h2, R2, Mt2, table = ref.load_green(path)
    assert (k2, Lt2, h2, R2, Mt2) == (gk, Lt, h, R, 10)
    assert np.array_equal(table.ravel(), payload)
    want = ref.precompute_green(gk, 1.25, 10, 1.0 + math.sqrt(3.0))
    assert np.array_equal(want.ravel(), payload)
