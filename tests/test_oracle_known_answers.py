"""The reference's own known-answer tests, restated against the C oracle
(oracle/fse_oracle.c).  Each test cites the reference test it restates
(/root/reference/proj/tests/...); the golden numbers recorded in
proj/test_output.txt are checked in test_oracle_recorded.py.  CPU only."""
import math

import numpy as np
import pytest

KINDS = [0, 1, 2]


def rnd_system(rng, kind, n, L):
    pos = rng.uniform(0, L, (n, 3))
    st = rng.uniform(-1, 1, (n, 9 if kind == 1 else 3))
    return pos, st


# test_spectral.cpp:17-42
def test_make_config_reference_values(oracle):
    c = oracle.make_config(2.0, 7.0, 0.63, 48, 16)
    assert c.h == pytest.approx(1.0 / 24, rel=1e-15)
    assert c.d == pytest.approx(2.0 / 3, rel=1e-15)
    assert c.m == pytest.approx(0.976 * math.sqrt(16.0 * math.pi), rel=1e-15)
    assert c.m == pytest.approx(6.921, rel=1e-3)
    assert c.eta == pytest.approx(0.4546, rel=1e-3)
    assert c.Ltilde == pytest.approx(c.h * c.Mtilde, rel=1e-14)
    assert c.kinf == pytest.approx(math.pi * c.Mtilde / c.Ltilde, rel=1e-14)
    assert c.R == pytest.approx(math.sqrt(3.0) * c.Ltilde, rel=1e-14)
    assert c.deltaL / c.h == pytest.approx(round(c.deltaL / c.h), rel=1e-12)
    c2 = oracle.make_config(2.0, 30.0, 0.2, 48, 16)
    assert c2.eta >= 1.0 and c2.deltaL == pytest.approx(c2.d, rel=1e-14)
    for bad in [(2.0, 7.0, 0.63, 48, 15), (2.0, 7.0, 0.63, 0, 16), (-1.0, 7.0, 0.63, 48, 16)]:
        with pytest.raises(ValueError):
            oracle.make_config(*bad)
    with pytest.raises(ValueError):
        oracle.make_config(2.0, 7.0, 0.63, 48, 16, 1.5)


# test_spectral.cpp:44-82
def test_spread_node_centered_source_is_sampled_gaussian(oracle):
    cfg = oracle.make_config(1.0, 6.0, 0.3, 16, 8)
    ox = -cfg.deltaL / 2
    x0 = ox + 12 * cfg.h
    pos = np.array([[x0, x0, x0]])
    g = oracle.spread(cfg, 0, pos, np.array([[1.0, 0, 0]]))
    alpha = 2 * cfg.xi ** 2 / cfg.eta
    pref = (2 * cfg.xi ** 2 / (math.pi * cfg.eta)) ** 1.5
    idx = np.arange(cfg.Mtilde)
    inside1 = (idx - 12 >= -cfg.P // 2) & (idx - 12 <= cfg.P // 2 - 1)
    node = ox + idx * cfg.h
    d2 = ((node - x0) ** 2)
    expect = pref * np.exp(-alpha * (d2[:, None, None] + d2[None, :, None] + d2[None, None, :]))
    mask = inside1[:, None, None] & inside1[None, :, None] & inside1[None, None, :]
    assert np.all(g[0][~mask] == 0.0)
    assert np.all(np.abs(g[0][mask] - expect[mask]) <= 1e-12 * expect[mask] + pref * 1e-14)
    assert np.all(g[1] == 0.0)


# test_spectral.cpp:84-100
@pytest.mark.parametrize("kind", KINDS)
def test_spread_conserves_strength(oracle, kind):
    rng = np.random.default_rng(271)
    pos, st = rnd_system(rng, kind, 20, 1.0)
    cfg = oracle.make_config(1.0, 8.0, 0.3, 24, 16)
    g = oracle.spread(cfg, kind, pos, st)
    tol = 10 * math.exp(-cfg.m ** 2 / 2) + 1e-12
    mass = g.reshape(g.shape[0], -1).sum(axis=1) * cfg.h ** 3
    want = st.sum(axis=0)
    assert np.all(np.abs(mass - want) <= tol * (1 + np.abs(want)))


# test_spectral.cpp:102-122 (FGG = naive; 200 random cases here)
def test_fgg_equals_naive(oracle):
    rng = np.random.default_rng(515)
    for it in range(200):
        kind = KINDS[it % 3]
        n = 1 + int(rng.integers(12))
        L = rng.uniform(0.5, 2.0)
        xi = rng.uniform(3.0, 12.0)
        M = 8 + 2 * int(rng.integers(5))
        P = 4 + 2 * int(rng.integers(3))
        pos, st = rnd_system(rng, kind, n, L)
        cfg = oracle.make_config(L, xi, 0.2 * L, M, P)
        a = oracle.spread(cfg, kind, pos, st, use_fgg=True)
        b = oracle.spread(cfg, kind, pos, st, use_fgg=False)
        scale = np.abs(b[0]).max()
        assert np.all(np.abs(a - b) <= 1e-13 * (scale + np.abs(b)))


# test_spectral.cpp:124-155
def test_kspace_stokeslet_zero_mode_and_incompressibility(oracle):
    cfg = oracle.make_config(1.0, 6.0, 0.3, 12, 8)
    G = oracle.precompute_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    D = cfg.D
    rng = np.random.default_rng(3)
    gh = rng.uniform(-1, 1, (3, D, D, D)) + 1j * rng.uniform(-1, 1, (3, D, D, D))
    out = oracle.kspace_scale(cfg, 0, G, gh)
    assert np.all(out[:, 0, 0, 0] == 0)
    dk = math.pi / cfg.Ltilde
    kof = lambda a: dk * (a if a < D // 2 else a - D)  # noqa: E731
    for _ in range(200):
        i, j, l = (int(v) for v in rng.integers(D, size=3))
        if i == j == l == 0:
            continue
        div = kof(i) * out[0, i, j, l] + kof(j) * out[1, i, j, l] + kof(l) * out[2, i, j, l]
        mag = np.abs(out[:, i, j, l]).sum()
        assert abs(div) <= 1e-10 * (1 + mag * (abs(kof(i)) + abs(kof(j)) + abs(kof(l))))


# test_spectral.cpp:157-183
def test_kspace_rotlet_axis_mode(oracle):
    cfg = oracle.make_config(1.0, 6.0, 0.3, 12, 8)
    G = oracle.precompute_green(0, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    D = cfg.D
    gh = np.zeros((3, D, D, D), np.complex128)
    g1, g2, g3 = 0.3 - 0.4j, 1.1 + 0.2j, -0.7 + 0.9j
    gh[:, 3, 0, 0] = [g1, g2, g3]
    out = oracle.kspace_scale(cfg, 2, G, gh)
    kappa = math.pi / cfg.Ltilde * 3
    rem = math.exp(-(1 - cfg.eta) * kappa ** 2 / (4 * cfg.xi ** 2))
    e1 = 1j * G[3, 0, 0] * rem * (-kappa * g3)
    e2 = 1j * G[3, 0, 0] * rem * (kappa * g2)
    assert abs(out[0, 3, 0, 0]) < 1e-14
    assert abs(out[1, 3, 0, 0] - e1) < 1e-12 * abs(e1)
    assert abs(out[2, 3, 0, 0] - e2) < 1e-12 * abs(e2)


# test_spectral.cpp:185-196
@pytest.mark.parametrize("kind", KINDS)
def test_total_sum_two_sources_matches_direct(oracle, kind):
    rng = np.random.default_rng(42 + kind)
    pos, st = rnd_system(rng, kind, 2, 1.0)
    cfg = oracle.make_config(1.0, 6.0, 1.0, 28, 32)
    G = oracle.precompute_green(oracle.green_kind_for(kind), cfg.Ltilde, cfg.Mtilde, cfg.sf)
    u = oracle.total_sum(cfg, kind, pos, st, pos, G)
    ref = oracle.direct_sum(kind, pos, st, pos, True)
    rel = math.sqrt(((u - ref) ** 2).sum() / (ref ** 2).sum())
    assert rel < 1e-12


# test_spectral.cpp:198-212
def test_total_sum_linear(oracle):
    rng = np.random.default_rng(68)
    pos, st = rnd_system(rng, 0, 15, 1.0)
    cfg = oracle.make_config(1.0, 7.0, 0.6, 24, 16)
    G = oracle.precompute_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    u1 = oracle.total_sum(cfg, 0, pos, st, pos, G)
    u2 = oracle.total_sum(cfg, 0, pos, -2.5 * st, pos, G)
    assert np.all(np.linalg.norm(u2 + 2.5 * u1, axis=1) <= 1e-13 * (1 + np.linalg.norm(u2, axis=1)))


# test_spectral.cpp:233-251
def test_fourier_reciprocity(oracle):
    cfg = oracle.make_config(1.0, 7.0, 0.5, 24, 16)
    G = oracle.precompute_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    x1, x2 = np.array([[0.31, 0.47, 0.62]]), np.array([[0.68, 0.55, 0.33]])
    f1, f2 = np.array([[0.4, -0.8, 0.2]]), np.array([[-0.3, 0.5, 0.9]])
    ua = oracle.fourier_sum(cfg, 0, x1, f1, x2, G)
    ub = oracle.fourier_sum(cfg, 0, x2, f2, x1, G)
    assert float(ua[0] @ f2[0]) == pytest.approx(float(ub[0] @ f1[0]), rel=1e-12)


# test_spectral.cpp:253-268
def test_fourier_sum_errors(oracle):
    cfg = oracle.make_config(1.0, 6.0, 0.3, 12, 8)
    G = oracle.precompute_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
    with pytest.raises(ValueError):
        oracle.fourier_sum(cfg, 0, [[0.5, 0.5, 0.5]], [[1, 0, 0]], [[1.5, 0.5, 0.5]], G)


# test_realspace.cpp:33-56
def test_real_kernel_limits_and_pinned(oracle):
    f = np.array([0.4, -0.2, 0.9])
    r = np.array([0.3, 0.5, -0.2])
    a = oracle.eval_real_kernel(0, r, 1e-12, f)
    b = oracle.eval_kernel(0, r, f)
    assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b)
    big = oracle.eval_real_kernel(0, r, 8.0 / np.linalg.norm(r), f)
    assert np.linalg.norm(big) < 1e-26 * np.linalg.norm(f) / np.linalg.norm(r)
    w = oracle.eval_real_kernel(2, [0, 0, 1.0], 1.0, [0, 1.0, 0])
    expect = math.erfc(1.0) + 2.0 / math.sqrt(math.pi) * math.exp(-1.0)
    assert w[0] == pytest.approx(expect, rel=1e-14) and w[1] == 0 and w[2] == 0
    with pytest.raises(ArithmeticError):
        oracle.eval_real_kernel(2, [0, 0, 0.0], 1.0, f)


# test_core.cpp:35-54
def test_bare_kernel_pinned(oracle):
    assert oracle.eval_kernel(0, [1, 0, 0.0], [1, 0, 0.0])[0] == pytest.approx(2.0, rel=1e-15)
    f11 = np.zeros(9)
    f11[0] = 1
    assert oracle.eval_kernel(1, [1, 0, 0.0], f11)[0] == pytest.approx(-6.0, rel=1e-15)
    assert oracle.eval_kernel(2, [0, 0, 1.0], [0, 1.0, 0])[0] == pytest.approx(1.0, rel=1e-15)


# test_realspace.cpp:89-131 (cell list basics + lattice coverage)
def test_cell_list_basics_and_lattice(oracle):
    cl = oracle.build_cell_list([[0.3, 0.4, 0.5]], 1.0, 0.2)
    assert (np.diff(cl["bstart"]) > 0).sum() == 1 and cl["bstart"][-1] == 1
    whole = oracle.build_cell_list([[0.3, 0.4, 0.5]], 1.0, 1.0)
    assert tuple(whole["dims"]) == (1, 1, 1)
    g = (np.arange(10) + 0.5) / 10
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    cl = oracle.build_cell_list(pos, 1.0, 0.1)
    assert cl["bstart"][-1] == len(pos)
    d = int(cl["dims"][0])

    def cell(x):
        return min(max(int(math.floor((x - cl["origin"]) / cl["cell_side"])), 0), d - 1)
    owner = np.empty(len(pos), int)
    for b in range(d ** 3):
        owner[cl["perm"][cl["bstart"][b]:cl["bstart"][b + 1]]] = b
    for m in range(0, len(pos), 37):
        ci = [cell(v) for v in pos[m]]
        near = np.where(np.linalg.norm(pos - pos[m], axis=1) <= 0.1)[0]
        for q in near:
            b = owner[q]
            qi = (b // (d * d), (b // d) % d, b % d)
            assert all(abs(qi[k] - ci[k]) <= 1 for k in range(3))


# test_realspace.cpp:166-205 (cell list == brute force; 200 random cases)
def test_real_space_equals_brute(oracle):
    rng = np.random.default_rng(404)
    for it in range(200):
        kind = KINDS[it % 3]
        n = 2 + int(rng.integers(60))
        L = rng.uniform(0.5, 3.0)
        xi = rng.uniform(0.5, 6.0)
        rc = rng.uniform(0.05 * L, 1.2 * L)
        pos, st = rnd_system(rng, kind, n, L)
        tgt = pos if it % 5 else rng.uniform(0, L, (8, 3))
        fast = oracle.real_space_sum(kind, pos, st, L, xi, rc, tgt)
        ref = np.zeros_like(fast)
        for m in range(len(tgt)):
            for q in range(n):
                r = tgt[m] - pos[q]
                d2 = float(r @ r)
                if d2 == 0 or d2 > rc * rc:
                    continue
                ref[m] += oracle.eval_real_kernel(kind, r, xi, st[q])
        assert np.all(np.linalg.norm(fast - ref, axis=1) <= 1e-13 * (1 + np.linalg.norm(ref, axis=1)))
    # rc far below the minimum spacing: exactly zero
    pos, st = rnd_system(rng, 0, 30, 1.0)
    assert np.all(oracle.real_space_sum(0, pos, st, 1.0, 2.0, 1e-9, pos) == 0.0)


# test_greens.cpp:67-83
def test_green_transforms_pinned(oracle):
    assert oracle.hhat(0.0, 2.0) == pytest.approx(8 * math.pi, rel=1e-14)
    assert abs(oracle.hhat(2 * math.pi / 3, 3.0)) < 1e-13
    assert oracle.hhat(math.pi, 1.0) == pytest.approx(8 / math.pi, rel=1e-13)
    assert oracle.bhat(0.0, 1.0) == pytest.approx(math.pi, rel=1e-14)
    assert oracle.bhat(0.0, 2.0) == pytest.approx(16 * math.pi, rel=1e-14)
    assert oracle.bhat(1e-4, 1.0) == pytest.approx(3.141592650099134736, rel=1e-13)
    assert oracle.bhat(0.3, 1.0) == pytest.approx(3.110282574231583346, rel=1e-13)
    assert oracle.bhat(0.4999999, 1.0) == pytest.approx(oracle.bhat(0.5000001, 1.0), rel=1e-7)


# test_greens.cpp:171-178
def test_green_zero_mode(oracle):
    g = oracle.precompute_green(0, 1.0, 32, 1 + math.sqrt(3))
    assert g[0, 0, 0] == pytest.approx(9.5203, rel=2e-3)
    with pytest.raises(ValueError):
        oracle.precompute_green(0, 1.0, 8, 2.0)
