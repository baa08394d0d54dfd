// k_realspace.cu -- screened real-space pair sum (realspace.cpp:86-149) with
// the screened kernels of realspace.cpp:13-58.
//
// Work item = (target cell, up to 128 of its targets); one thread per target.
// The 27 neighbour buckets (lexicographic (di,dj,dk), sources in bucket order
// -- the reference's summation order) are concatenated virtually and
// streamed through shared memory in chunks of 128 sources shared by all
// targets of the item.  Each thread first tests its target against the whole
// chunk (exact closed-ball test 0 < d2 <= rc2 with d2 = (x*x + y*y) + z*z
// rounded like the reference) into a 128-bit mask, then evaluates only the
// accepted pairs in ascending order.  This keeps the pair evaluation off the
// ~85% of candidates that fail the test, instead of predicating the whole
// warp on every candidate.
//
// Pair math: with x = xi r and inv = 1/r (rsqrt), every screened kernel is a
// power of inv times smooth functions of x alone (s = 2/sqrt(pi)):
//   stokeslet: a - b = inv Ahat(x), a = inv Chat(x),
//              Ahat = erfc x - s x e^{-x^2},  Chat = erfc x + s x e^{-x^2}
//   rotlet:    c = inv^2 Chat(x)
//   stresslet: c1 = -2 inv^2 Dhat(x), c2 = xi^2 Ehat(x),
//              Dhat = 3 erfc x + s x (3 + 2x^2) e^{-x^2},  Ehat = 2 s x e^{-x^2}
// Those are tabulated on [0, 6.5) as piecewise degree-12 Chebyshev fits
// (monomial in the local t), computed on the host in long double from
// erfcl/expl, so a pair costs one rsqrt and two 12-term Horner evaluations
// instead of erfc + exp + divisions.  Absolute fit error < 1e-17 of the
// functions' O(1) scale.  x >= 6.5 (only for xi rc > 6.5) uses erfc/exp.
//
// Roofline: FP64 (pair work).
#include <cmath>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int TPB = 128, CH = 128;
constexpr double kInvSqrtPi = 0.5641895835477562869;

constexpr int kNI = 32, kDeg = 12;
constexpr double kXMax = 6.5;
constexpr int kNumFn = 4;  // Ahat, Chat, Dhat, Ehat
__constant__ double c_fn[kNumFn][kDeg + 1][kNI];

struct Tab {
    double c[kDeg + 1][kNI];
};

__device__ __forceinline__ double horner(const Tab& tb, int iv, double t) {
    double acc = tb.c[kDeg][iv];
#pragma unroll
    for (int j = kDeg - 1; j >= 0; --j) acc = fma(acc, t, tb.c[j][iv]);
    return acc;
}

// exact functions (fallback beyond the table)
__device__ __forceinline__ void fn_exact(int which, double x, double* out) {
    const double e = exp(-x * x), ec = erfc(x), s = 2.0 * kInvSqrtPi;
    switch (which) {
        case 0: *out = ec - s * x * e; break;
        case 1: *out = ec + s * x * e; break;
        case 2: *out = 3.0 * ec + s * x * (3.0 + 2.0 * x * x) * e; break;
        default: *out = 2.0 * s * x * e; break;
    }
}

__device__ __forceinline__ double exact_d2(double rx, double ry, double rz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz));
}

// tab0/tab1: the two functions this kernel needs (stokeslet: Ahat, Chat;
// rotlet: Chat; stresslet: Dhat, Ehat)
template <int KIND>
__device__ __forceinline__ void pair(double rx, double ry, double rz, double r2, double xi,
                                     const double* f, const Tab& tab0, const Tab& tab1,
                                     double acc[3]) {
    const double inv = rsqrt(r2);
    const double rn = r2 * inv;
    const double xr = xi * rn;
    double F0, F1 = 0.0;
    if (xr < kXMax) {
        const double uu = xr * (kNI / kXMax);
        const int iv = min(static_cast<int>(uu), kNI - 1);
        const double t = 2.0 * (uu - iv) - 1.0;
        F0 = horner(tab0, iv, t);
        if (KIND != FSE_ROTLET) F1 = horner(tab1, iv, t);
    } else {
        fn_exact(KIND == FSE_STOKESLET ? 0 : (KIND == FSE_ROTLET ? 1 : 2), xr, &F0);
        if (KIND != FSE_ROTLET) fn_exact(KIND == FSE_STOKESLET ? 1 : 3, xr, &F1);
    }
    const double rh[3] = {inv * rx, inv * ry, inv * rz};
    if (KIND == FSE_STOKESLET) {
        const double amb = inv * F0;  // a - b
        const double a = inv * F1;
        const double s = a * (rh[0] * f[0] + rh[1] * f[1] + rh[2] * f[2]);
#pragma unroll
        for (int j = 0; j < 3; ++j) acc[j] += amb * f[j] + s * rh[j];
    } else if (KIND == FSE_STRESSLET) {
        const double c1 = -2.0 * inv * inv * F0;
        const double c2 = xi * xi * F1;
        double rfr = 0, f_r[3] = {0, 0, 0}, r_f[3] = {0, 0, 0};
#pragma unroll
        for (int l = 0; l < 3; ++l)
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                rfr += rh[l] * f[3 * l + m] * rh[m];
                f_r[l] += f[3 * l + m] * rh[m];
                r_f[m] += rh[l] * f[3 * l + m];
            }
        const double trf = f[0] + f[4] + f[8];
        const double s = c1 * rfr + c2 * trf;
#pragma unroll
        for (int j = 0; j < 3; ++j) acc[j] += s * rh[j] + c2 * (f_r[j] + r_f[j]);
    } else {
        const double c = inv * inv * F0;
        acc[0] += c * (f[1] * rh[2] - f[2] * rh[1]);
        acc[1] += c * (f[2] * rh[0] - f[0] * rh[2]);
        acc[2] += c * (f[0] * rh[1] - f[1] * rh[0]);
    }
}

template <int KIND>
__global__ void __launch_bounds__(TPB) k_realspace(
    int dim, const double* __restrict__ spx, const double* __restrict__ spy,
    const double* __restrict__ spz, const double* __restrict__ sfs,
    const int32_t* __restrict__ bstart, const double* __restrict__ tpx,
    const double* __restrict__ tpy, const double* __restrict__ tpz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ items,
    const uint32_t* __restrict__ tperm, const int32_t* __restrict__ nitems_dev, double xi,
    double rc2, double* __restrict__ u) {
    constexpr int A = KIND == FSE_STRESSLET ? 9 : 3;
    constexpr int F0 = KIND == FSE_STOKESLET ? 0 : (KIND == FSE_ROTLET ? 1 : 2);
    constexpr int F1 = KIND == FSE_STOKESLET ? 1 : 3;
    __shared__ double sx[CH], sy[CH], sz[CH];
    __shared__ double sf[CH][A];
    __shared__ int nb_start[27], nb_pref[28];
    __shared__ Tab tab0, tab1;
    for (int e = threadIdx.x; e < (kDeg + 1) * kNI; e += blockDim.x) {
        tab0.c[e / kNI][e % kNI] = c_fn[F0][e / kNI][e % kNI];
        if (KIND != FSE_ROTLET) tab1.c[e / kNI][e % kNI] = c_fn[F1][e / kNI][e % kNI];
    }

    if (static_cast<int>(blockIdx.x) >= *nitems_dev) return;  // grid is an upper bound
    const int cell = items[2 * blockIdx.x];
    const int sub = items[2 * blockIdx.x + 1];
    const int tid = threadIdx.x;
    const int ck = cell % dim, cj = (cell / dim) % dim, ci = cell / (dim * dim);
    if (tid == 0) {
        int acc = 0, r = 0;
        for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj)
                for (int dk = -1; dk <= 1; ++dk) {
                    const int i = ci + di, j = cj + dj, k = ck + dk;
                    int len = 0, st = 0;
                    if (i >= 0 && i < dim && j >= 0 && j < dim && k >= 0 && k < dim) {
                        const int b = (i * dim + j) * dim + k;
                        st = bstart[b];
                        len = bstart[b + 1] - st;
                    }
                    nb_start[r] = st;
                    nb_pref[r] = acc;
                    acc += len;
                    ++r;
                }
        nb_pref[27] = acc;
    }
    const int q = tstart[cell] + sub * TPB + tid;
    const bool valid = q < tstart[cell + 1];
    double x = 0, y = 0, z = 0;
    if (valid) {
        x = tpx[q];
        y = tpy[q];
        z = tpz[q];
    }
    double acc[3] = {0.0, 0.0, 0.0};
    __syncthreads();
    const int total = nb_pref[27];
    int r = 0;  // neighbour cursor for the cooperative load (monotone in v)
    for (int base = 0; base < total; base += CH) {
        const int v = base + tid;
        if (v < total) {
            while (nb_pref[r + 1] <= v) ++r;
            const int sidx = nb_start[r] + (v - nb_pref[r]);
            sx[tid] = spx[sidx];
            sy[tid] = spy[sidx];
            sz[tid] = spz[sidx];
#pragma unroll
            for (int c = 0; c < A; ++c) sf[tid][c] = sfs[static_cast<int64_t>(sidx) * A + c];
        }
        __syncthreads();
        const int cnt = min(CH, total - base);
        uint32_t mask[CH / 32];
#pragma unroll
        for (int wd = 0; wd < CH / 32; ++wd) {
            uint32_t m = 0;
            const int lim = min(32, cnt - wd * 32);
            for (int b = 0; b < lim; ++b) {
                const int j = wd * 32 + b;
                const double d2 = exact_d2(x - sx[j], y - sy[j], z - sz[j]);
                const bool pass = (d2 != 0.0) && !(d2 > rc2);  // realspace.cpp:140
                m |= static_cast<uint32_t>(pass) << b;
            }
            mask[wd] = valid ? m : 0u;
        }
#pragma unroll
        for (int wd = 0; wd < CH / 32; ++wd) {
            uint32_t m = mask[wd];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int j = wd * 32 + b;
                const double rx = x - sx[j], ry = y - sy[j], rz = z - sz[j];
                pair<KIND>(rx, ry, rz, exact_d2(rx, ry, rz), xi, sf[j], tab0, tab1, acc);
            }
        }
        __syncthreads();
    }
    if (valid) {
        const int64_t m = tperm[q];
        u[3 * m] = acc[0];
        u[3 * m + 1] = acc[1];
        u[3 * m + 2] = acc[2];
    }
}

__global__ void k_item_counts(const int32_t* __restrict__ start, int64_t ncell, int per,
                              int32_t* __restrict__ cnt) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c < ncell) cnt[c] = (start[c + 1] - start[c] + per - 1) / per;
    if (c == ncell) cnt[c] = 0;
}

__global__ void k_fill_items(const int32_t* __restrict__ off, int64_t ncell,
                             int32_t* __restrict__ items) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= ncell) return;
    for (int32_t it = off[c]; it < off[c + 1]; ++it) {
        items[2 * it] = static_cast<int32_t>(c);
        items[2 * it + 1] = it - off[c];
    }
}

// long-double screened functions of x (see the header comment)
long double fn_ld(int which, long double x) {
    const long double s = 2.0L / sqrtl(3.141592653589793238462643383279502884L);
    const long double e = expl(-x * x), ec = erfcl(x);
    switch (which) {
        case 0: return ec - s * x * e;
        case 1: return ec + s * x * e;
        case 2: return 3.0L * ec + s * x * (3.0L + 2.0L * x * x) * e;
        default: return 2.0L * s * x * e;
    }
}

// Chebyshev fit on each interval, converted to monomials in t in [-1, 1]
void build_tables(double out[kNumFn][kDeg + 1][kNI]) {
    const int n = kDeg + 1;
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int fnid = 0; fnid < kNumFn; ++fnid)
        for (int iv = 0; iv < kNI; ++iv) {
            const long double a = kXMax * iv / static_cast<long double>(kNI);
            const long double b = kXMax * (iv + 1) / static_cast<long double>(kNI);
            long double fv[n], cheb[n];
            for (int k = 0; k < n; ++k) {
                const long double t = cosl(PI * (k + 0.5L) / n);
                fv[k] = fn_ld(fnid, 0.5L * (a + b) + 0.5L * (b - a) * t);
            }
            for (int j = 0; j < n; ++j) {
                long double sum = 0;
                for (int k = 0; k < n; ++k) sum += fv[k] * cosl(PI * j * (k + 0.5L) / n);
                cheb[j] = sum * 2.0L / n;
            }
            cheb[0] *= 0.5L;
            long double mono[n] = {}, Tprev[n] = {}, Tcur[n] = {}, Tnext[n];
            Tprev[0] = 1;
            Tcur[1] = 1;
            for (int j = 0; j < n; ++j) mono[j] += cheb[0] * Tprev[j] + cheb[1] * Tcur[j];
            for (int d = 2; d < n; ++d) {
                for (int j = 0; j < n; ++j) Tnext[j] = -Tprev[j] + (j > 0 ? 2 * Tcur[j - 1] : 0);
                for (int j = 0; j < n; ++j) mono[j] += cheb[d] * Tnext[j];
                for (int j = 0; j < n; ++j) {
                    Tprev[j] = Tcur[j];
                    Tcur[j] = Tnext[j];
                }
            }
            for (int j = 0; j < n; ++j) out[fnid][j][iv] = static_cast<double>(mono[j]);
        }
}

void ensure_tables() {
    static bool ready[64] = {};
    int dev = 0;
    FSE_CU(cudaGetDevice(&dev));
    if (dev < 64 && ready[dev]) return;
    static double tab[kNumFn][kDeg + 1][kNI];
    static bool built = false;
    if (!built) {
        build_tables(tab);
        built = true;
    }
    FSE_CU(cudaMemcpyToSymbol(c_fn, tab, sizeof tab));
    if (dev < 64) ready[dev] = true;
}

}  // namespace

void launch_item_counts(const Launch& L, const int32_t* start, int64_t ncell, int per,
                        int32_t* cnt) {
    k_item_counts<<<static_cast<unsigned>((ncell + 256) / 256), 256, 0, L.s>>>(start, ncell, per,
                                                                             cnt);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_fill_items(const Launch& L, const int32_t* start, const int32_t* off, int64_t ncell,
                       int per, int32_t* items) {
    (void)start;
    (void)per;
    k_fill_items<<<static_cast<unsigned>((ncell + 255) / 256), 256, 0, L.s>>>(off, ncell, items);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_realspace(const Launch& L, int kind, const CellGrid& cg, const double* spx,
                      const double* spy, const double* spz, const double* sfs, int64_t ns,
                      const int32_t* bstart, const double* tpx, const double* tpy,
                      const double* tpz, const int32_t* tcell_start, const int32_t* items,
                      int64_t max_items, const int32_t* nitems_dev, const uint32_t* tperm,
                      double xi, double rc, double* uR) {
    (void)ns;
    if (max_items <= 0) return;
    ensure_tables();
    const double rc2 = rc * rc;
    const unsigned b = static_cast<unsigned>(max_items);
    if (kind == FSE_STOKESLET)
        k_realspace<FSE_STOKESLET><<<b, TPB, 0, L.s>>>(cg.dim, spx, spy, spz, sfs, bstart, tpx,
                                                       tpy, tpz, tcell_start, items, tperm,
                                                       nitems_dev, xi, rc2, uR);
    else if (kind == FSE_STRESSLET)
        k_realspace<FSE_STRESSLET><<<b, TPB, 0, L.s>>>(cg.dim, spx, spy, spz, sfs, bstart, tpx,
                                                       tpy, tpz, tcell_start, items, tperm,
                                                       nitems_dev, xi, rc2, uR);
    else
        k_realspace<FSE_ROTLET><<<b, TPB, 0, L.s>>>(cg.dim, spx, spy, spz, sfs, bstart, tpx, tpy,
                                                    tpz, tcell_start, items, tperm, nitems_dev,
                                                    xi, rc2, uR);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
