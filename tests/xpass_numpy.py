"""numpy restatement of the hot path's fused x pass (test helper for
tests/test_gpu_xpass_oracle.py; pinned to the reference's kspace_scale by
tests/test_xpass_numpy.py)."""
import numpy as np

def splitmix_u(x):
    """k_misc.cu probe_u: splitmix64 finaliser, (z >> 11) 2^-53."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def multiplier(kind, k, G, cfg):
    """ewald.cpp:216-293 as a per-k linear map: returns the (3, a) complex
    matrix A(k) G(k) rem(k) for k of shape (3, n)."""
    k2 = k[0] * k[0] + k[1] * k[1] + k[2] * k[2]
    inv4 = 1.0 / (4.0 * cfg.xi * cfg.xi)
    rem = np.exp(-(1.0 - cfg.eta) * k2 * inv4)
    n = k.shape[1]
    if kind == 0:   # stokeslet: b (k^2 g - k (k.g)), b = -G (1 + k^2/4xi^2) rem
        b = -G * (1.0 + k2 * inv4) * rem
        A = np.zeros((3, 3, n), complex)
        for p in range(3):
            for q in range(3):
                A[p, q] = b * ((k2 if p == q else 0.0) - k[p] * k[q])
        return A
    if kind == 2:   # rotlet: -i G rem (g x k)
        c = -1j * G * rem
        A = np.zeros((3, 3, n), complex)
        A[0, 1], A[0, 2] = c * k[2], -c * k[1]
        A[1, 2], A[1, 0] = c * k[0], -c * k[2]
        A[2, 0], A[2, 1] = c * k[1], -c * k[0]
        return A
    # stresslet: -i b [k^2 (a_p + bt_p + k_p tr) - 2 k_p (k.g.k)], b = G (1 + k^2/4xi^2) rem,
    # a_p = sum_q g_pq k_q, bt_p = sum_l k_l g_lp, tr = sum g_pp; g_pq at slot 3p+q
    b = -1j * G * (1.0 + k2 * inv4) * rem
    A = np.zeros((3, 9, n), complex)
    for p in range(3):
        for l in range(3):
            for m in range(3):
                coef = 0.0
                if l == p:
                    coef = coef + k2 * k[m]          # a_p
                if m == p:
                    coef = coef + k2 * k[l]          # bt_p
                if l == m:
                    coef = coef + k2 * k[p]          # k_p tr
                coef = coef - 2.0 * k[p] * k[l] * k[m]
                A[p, 3 * l + m] = b * coef
    return A


def expected(cfg, kind, seed, ky, kz, gcol):
    Mt, D = cfg.Mtilde, cfg.D
    Dh = D // 2 + 1
    a = 9 if kind == 1 else 3
    dk = np.pi / cfg.Ltilde
    kax = dk * np.where(np.arange(D) < D // 2, np.arange(D), np.arange(D) - D)
    half = D // 2
    out = np.zeros((len(ky), 3, Mt), complex)
    x = np.arange(Mt, dtype=np.uint64)
    for p, (y, z) in enumerate(zip(ky, kz)):
        col = np.zeros((a, D), complex)
        for c in range(a):
            idx = ((np.uint64(c) * np.uint64(Mt) + x) * np.uint64(D) + np.uint64(y)) \
                * np.uint64(Dh) + np.uint64(z)
            s2 = np.uint64(seed) + np.uint64(2) * idx
            col[c, :Mt] = (splitmix_u(s2) - 0.5) + 1j * (splitmix_u(s2 + np.uint64(1)) - 0.5)
        gh = np.fft.fft(col, axis=1)
        kx = np.arange(D)
        k = np.stack([kax[kx], np.full(D, kax[y]), np.full(D, kax[z])])
        A = multiplier(kind, k, gcol[p], cfg)
        kt = k.copy()   # k~: components at the Nyquist index negated
        kt[0, kx == half] *= -1
        if y == half:
            kt[1] *= -1
        if z == half:
            kt[2] *= -1
        A = 0.5 * (A + multiplier(kind, kt, gcol[p], cfg))
        res = np.einsum("pqn,qn->pn", A, gh) / float(D) ** 3
        out[p] = (np.fft.ifft(res, axis=1) * D)[:, :Mt]
    return out
