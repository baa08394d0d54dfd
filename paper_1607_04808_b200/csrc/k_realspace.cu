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
// accepted pairs in ascending order.  This keeps the erfc/exp-heavy pair
// evaluation off the ~85% of candidates that fail the test, instead of
// predicating the whole warp on every candidate.
//
// Roofline: FP64 (transcendental-heavy pair work).
#include <cmath>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int TPB = 128, CH = 128;
constexpr double kInvSqrtPi = 0.5641895835477562869;

// erfc(x) = exp(-x^2) erfcx(x); erfcx on [0, kErfXMax) from a piecewise
// Chebyshev fit (kErfNI intervals, degree kErfDeg, monomial in the local
// t in [-1, 1]) computed on the host in long double from erfcl/expl
// (|error| < 1e-17 relative).  One exp + a degree-12 Horner replace CUDA's
// range-branched erfc (~190 SASS instructions) plus the separate exp.
constexpr int kErfNI = 32, kErfDeg = 12;
constexpr double kErfXMax = 6.5;
__constant__ double c_erfcx[kErfDeg + 1][kErfNI];

__device__ __forceinline__ double erfcx_tab(double x, const double (*tab)[kErfNI]) {
    const double u = x * (kErfNI / kErfXMax);
    const int iv = min(static_cast<int>(u), kErfNI - 1);
    const double t = 2.0 * (u - iv) - 1.0;
    double acc = tab[kErfDeg][iv];
#pragma unroll
    for (int j = kErfDeg - 1; j >= 0; --j) acc = fma(acc, t, tab[j][iv]);
    return acc;
}

// screened pair kernels of realspace.cpp:13-58, rearranged around
// inv = 1/r (rsqrt) and erfc = gauss * erfcx: no divisions
template <int KIND>
__device__ __forceinline__ void pair(double rx, double ry, double rz, double r2, double xi,
                                     const double* f, const double (*tab)[kErfNI], double acc[3]) {
    const double inv = rsqrt(r2);
    const double rn = r2 * inv;
    const double xr = xi * rn;
    const double gauss = exp(-xr * xr);
    const double erfc_xr = xr < kErfXMax ? gauss * erfcx_tab(xr, tab) : erfc(xr);
    const double rh[3] = {inv * rx, inv * ry, inv * rz};
    const double cg = 2.0 * xi * kInvSqrtPi * gauss;  // 2 xi e^{-x^2} / sqrt(pi)
    if (KIND == FSE_STOKESLET) {
        // a = 2 (xi g/sqrt(pi) + erfc/(2r)), b = 4 xi g/sqrt(pi)
        const double e_r = erfc_xr * inv;
        const double a = cg + e_r;
        const double amb = e_r - cg;
        const double s = a * (rh[0] * f[0] + rh[1] * f[1] + rh[2] * f[2]);
#pragma unroll
        for (int j = 0; j < 3; ++j) acc[j] += amb * f[j] + s * rh[j];
    } else if (KIND == FSE_STRESSLET) {
        const double c1 = -2.0 * inv * (3.0 * erfc_xr * inv + cg * (3.0 + 2.0 * xr * xr));
        const double c2 = 2.0 * xi * xi * cg * rn;  // 4 xi^3 g r / sqrt(pi)
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
        const double c = (erfc_xr * inv + cg) * inv;  // erfc/r^2 + 2 xi g/(sqrt(pi) r)
        acc[0] += c * (f[1] * rh[2] - f[2] * rh[1]);
        acc[1] += c * (f[2] * rh[0] - f[0] * rh[2]);
        acc[2] += c * (f[0] * rh[1] - f[1] * rh[0]);
    }
}

__device__ __forceinline__ double exact_d2(double rx, double ry, double rz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz));
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
    __shared__ double sx[CH], sy[CH], sz[CH];
    __shared__ double sf[CH][A];
    __shared__ int nb_start[27], nb_pref[28];
    __shared__ double tab[kErfDeg + 1][kErfNI];
    for (int e = threadIdx.x; e < (kErfDeg + 1) * kErfNI; e += blockDim.x)
        tab[e / kErfNI][e % kErfNI] = c_erfcx[e / kErfNI][e % kErfNI];

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
                pair<KIND>(rx, ry, rz, exact_d2(rx, ry, rz), xi, sf[j], tab, acc);
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

// Chebyshev fit of erfcx on each interval, long double, converted to
// monomial coefficients in the local variable t in [-1, 1]
void build_erfcx_table(double out[kErfDeg + 1][kErfNI]) {
    const int n = kErfDeg + 1;
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int iv = 0; iv < kErfNI; ++iv) {
        const long double a = kErfXMax * iv / static_cast<long double>(kErfNI);
        const long double b = kErfXMax * (iv + 1) / static_cast<long double>(kErfNI);
        long double fv[n], cheb[n];
        for (int k = 0; k < n; ++k) {
            const long double t = cosl(PI * (k + 0.5L) / n);
            const long double x = 0.5L * (a + b) + 0.5L * (b - a) * t;
            fv[k] = expl(x * x) * erfcl(x);
        }
        for (int j = 0; j < n; ++j) {
            long double sum = 0;
            for (int k = 0; k < n; ++k) sum += fv[k] * cosl(PI * j * (k + 0.5L) / n);
            cheb[j] = sum * 2.0L / n;
        }
        cheb[0] *= 0.5L;
        // sum_j cheb_j T_j(t) -> sum_j mono_j t^j
        long double mono[n] = {}, Tprev[n] = {}, Tcur[n] = {}, Tnext[n];
        Tprev[0] = 1;            // T0
        Tcur[1] = 1;             // T1
        for (int j = 0; j < n; ++j) mono[j] += cheb[0] * Tprev[j];
        for (int j = 0; j < n; ++j) mono[j] += cheb[1] * Tcur[j];
        for (int d = 2; d < n; ++d) {
            for (int j = 0; j < n; ++j) Tnext[j] = -Tprev[j] + (j > 0 ? 2 * Tcur[j - 1] : 0);
            for (int j = 0; j < n; ++j) mono[j] += cheb[d] * Tnext[j];
            for (int j = 0; j < n; ++j) {
                Tprev[j] = Tcur[j];
                Tcur[j] = Tnext[j];
            }
        }
        for (int j = 0; j < n; ++j) out[j][iv] = static_cast<double>(mono[j]);
    }
}

void ensure_erfcx_table() {
    static bool ready[64] = {};
    int dev = 0;
    FSE_CU(cudaGetDevice(&dev));
    if (dev < 64 && ready[dev]) return;
    static double tab[kErfDeg + 1][kErfNI];
    static bool built = false;
    if (!built) {
        build_erfcx_table(tab);
        built = true;
    }
    FSE_CU(cudaMemcpyToSymbol(c_erfcx, tab, sizeof tab));
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
    const int64_t nitems = max_items;
    if (nitems <= 0) return;
    ensure_erfcx_table();
    const double rc2 = rc * rc;
    const unsigned b = static_cast<unsigned>(nitems);
    if (kind == FSE_STOKESLET)
        k_realspace<FSE_STOKESLET><<<b, TPB, 0, L.s>>>(cg.dim, spx, spy, spz, sfs, bstart, tpx,
                                                       tpy, tpz, tcell_start, items, tperm, nitems_dev,
                                                       xi, rc2, uR);
    else if (kind == FSE_STRESSLET)
        k_realspace<FSE_STRESSLET><<<b, TPB, 0, L.s>>>(cg.dim, spx, spy, spz, sfs, bstart, tpx,
                                                       tpy, tpz, tcell_start, items, tperm, nitems_dev,
                                                       xi, rc2, uR);
    else
        k_realspace<FSE_ROTLET><<<b, TPB, 0, L.s>>>(cg.dim, spx, spy, spz, sfs, bstart, tpx, tpy,
                                                    tpz, tcell_start, items, tperm, nitems_dev, xi, rc2, uR);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
