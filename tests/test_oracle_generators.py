"""The reference-side workload generator (oracle/ref_capi.cpp
ref_generate_workload, used by bench.py's reference arm and by
tests/golden/make_golden_baseline.py) and the product's
fse_generate_workload produce the same SURVEY 8(d) streams bit for bit, so
the golden vectors' inputs are the GPU tests' inputs."""
import numpy as np
import pytest

from oracle import refimpl as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("which", [1, 3, 4, 5])
@pytest.mark.parametrize("n", [1, 33, 4096])
def test_generators_bit_identical(fse, which, n):
    pos, st, tgt = R.generate_workload(which, n, 20260101 + n)
    sysm, t2 = fse.generate_workload(which, n, 20260101 + n)
    assert np.array_equal(pos, sysm.positions)
    assert np.array_equal(st, sysm.strengths)
    if which == 5:
        assert np.array_equal(tgt, t2)
    else:
        assert tgt is None and t2 is None
