"""Pins the C restatement (oracle/fse_oracle.c) to the reference compiled
from its own sources (oracle/_ref) on fresh seeded inputs, and the FFTW shim
to numpy.fft.  Skipped where oracle/_ref cannot be built (no /root/reference)."""
import numpy as np
import pytest

from conftest import rel_max


@pytest.mark.parametrize("shape", [(4, 6, 8), (97, 2, 13), (6, 149, 4), (61, 2, 2), (12, 9, 10),
                                   (1, 1, 1), (26, 26, 26)])
def test_fft_shim_matches_numpy(oracle, shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    assert rel_max(oracle.fft3d(x), np.fft.fftn(x)) <= 1e-14
    assert rel_max(oracle.fft3d(x, inverse=True), np.fft.ifftn(x)) <= 1e-14


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("args", [(1.0, 8.0, 0.3, 24, 16), (1.5, 5.0, 0.5, 20, 10)])
def test_restated_equals_reference(oracle, ref, kind, args):
    rng = np.random.default_rng(100 * kind + args[3])
    L = args[0]
    n = 250
    pos = rng.uniform(0, L, (n, 3))
    st = rng.standard_normal((n, ref.arity(kind)))
    tgt = rng.uniform(0, L, (90, 3))
    c_o, c_r = oracle.make_config(*args), ref.make_config(*args)
    assert c_o == c_r
    gk = ref.green_kind_for(kind)
    G = ref.precompute_green(gk, c_r.Ltilde, c_r.Mtilde, c_r.sf)
    assert np.array_equal(oracle.precompute_green(gk, c_r.Ltilde, c_r.Mtilde, c_r.sf), G)
    for t in (pos, tgt):
        assert rel_max(oracle.total_sum(c_o, kind, pos, st, t, G, box_side=L),
                       ref.total_sum(c_r, kind, pos, st, t, G)) <= 1e-14
    assert np.array_equal(oracle.real_space_sum(kind, pos, st, L, args[1], args[2], tgt),
                          ref.real_space_sum(kind, pos, st, L, args[1], args[2], tgt))
    D = c_r.D
    gh = rng.standard_normal((ref.arity(kind), D, D, D)) + 1j * rng.standard_normal(
        (ref.arity(kind), D, D, D))
    assert rel_max(oracle.kspace_scale(c_o, kind, G, gh), ref.kspace_scale(c_r, kind, G, gh)) <= 1e-15
    cl_o = oracle.build_cell_list(pos, L, args[2], 0.1)
    cl_r = ref.build_cell_list(pos, L, args[2], 0.1)
    for k in ("bstart", "perm", "dims"):
        assert np.array_equal(cl_o[k], cl_r[k])
    assert rel_max(oracle.direct_sum(kind, pos, st, tgt, False),
                   ref.direct_sum(kind, pos, st, L, tgt, False)) == 0.0


def test_reference_errors_match(oracle, ref):
    for bad in [(2.0, 7.0, 0.63, 48, 15), (2.0, 7.0, 0.63, 0, 16), (2.0, 7.0, 0.63, 48, 16, 1.5)]:
        with pytest.raises(ValueError):
            ref.make_config(*bad)
        with pytest.raises(ValueError):
            oracle.make_config(*bad)
