"""The hand-written fp64 FFT engine of the hot path (k_fft.cu) against
numpy.fft, at the FFT sizes of every BASELINE config (D = 2 Mtilde: 194 =
2*97, 298 = 2*149, 624 = 2^4*3*13, 1200 = 2^4*3*5^2) and the tolerance-consistent
variants (242, 348, 704, 888), plus radix edge cases.  Also the cuFFT-backed
fft3d seam (fft.hpp:11,14)."""
import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("D", [2, 8, 12, 26, 30, 154, 194, 242, 298, 348, 624, 704, 888, 1200,
                               17 * 2, 97, 1730])
def test_fft_engine_matches_numpy(ctx, D):
    rng = np.random.default_rng(D)
    x = rng.standard_normal((7, D)) + 1j * rng.standard_normal((7, D))
    assert rel_max(ctx.fft_columns(x), np.fft.fft(x, axis=1)) <= 2e-15 * max(1, np.log2(D))
    assert rel_max(ctx.fft_columns(x, inverse=True), np.fft.ifft(x, axis=1) * D) <= \
        2e-15 * max(1, np.log2(D))


def test_fft3d_seam(ctx):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((12, 10, 14)) + 1j * rng.standard_normal((12, 10, 14))
    assert rel_max(ctx.fft3d(x), np.fft.fftn(x)) <= 1e-14
    assert rel_max(ctx.fft3d(x, inverse=True), np.fft.ifftn(x)) <= 1e-14
