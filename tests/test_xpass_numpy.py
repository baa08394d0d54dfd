"""Pins the numpy multiplier of tests/xpass_numpy.py (used as the oracle of
the GPU x-pass test) to the reference's own kspace_scale (oracle/_ref,
ewald.cpp:216-293) on a small full C2C grid: at every k off the Nyquist
planes the reference output equals A(k) ghat(k)."""
import numpy as np
import pytest

from xpass_numpy import multiplier


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_numpy_multiplier_matches_reference(ref, kind):
    cfg = ref.make_config(1.0, 8.0, 0.3, 4, 4)
    D = cfg.D
    rng = np.random.default_rng(kind)
    a = 9 if kind == 1 else 3
    ghat = rng.standard_normal((a, D, D, D)) + 1j * rng.standard_normal((a, D, D, D))
    green = rng.uniform(0.5, 1.5, (D, D, D))
    out = ref.kspace_scale(cfg, kind, green, ghat)
    dk = np.pi / cfg.Ltilde
    ax = dk * np.where(np.arange(D) < D // 2, np.arange(D), np.arange(D) - D)
    I, J, L = np.meshgrid(np.arange(D), np.arange(D), np.arange(D), indexing="ij")
    k = np.stack([ax[I].ravel(), ax[J].ravel(), ax[L].ravel()])
    A = multiplier(kind, k, green.ravel(), cfg)
    want = np.einsum("pqn,qn->pn", A, ghat.reshape(a, -1)).reshape(3, D, D, D)
    assert np.abs(out - want).max() <= 1e-13 * np.abs(want).max()
