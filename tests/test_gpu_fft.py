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


def test_three_level_engine_opt_in(tmp_path):
    """The opt-in three-level engine (1200 = 10 x 12 x 10, FSE_FFT_1200_3L=1; the
    engine is chosen once per plan, so a fresh process) against numpy, and a
    fourier_sum through it against the default two-level engine."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1607_04808_b200 as fse
ctx = fse.Context(0)
rng = np.random.default_rng(1)
x = rng.standard_normal((5, 1200)) + 1j * rng.standard_normal((5, 1200))
e = np.abs(ctx.fft_columns(x) - np.fft.fft(x, axis=1)).max() / np.abs(np.fft.fft(x, axis=1)).max()
cfg = fse.make_config(1.0, 220.0, 0.022, 576, 24)
g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
s = fse.SourceSystem(rng.random((2000, 3)), rng.standard_normal((2000, 3)))
u = ctx.fourier_sum(s, cfg, 0, s.positions, g)
np.save({str(tmp_path / 'u.npy')!r}, u)
print(e)
"""
    outs = []
    for flag in ("1", None):
        env = dict(os.environ)
        env.pop("FSE_FFT_1200_3L", None)
        if flag:
            env["FSE_FFT_1200_3L"] = flag
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        assert float(r.stdout.split()[-1]) <= 2e-15 * np.log2(1200)
        outs.append(np.load(tmp_path / "u.npy"))
    assert rel_max(outs[0], outs[1]) <= 1e-11
