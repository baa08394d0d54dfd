// k_misc.cu -- epilogue of total_sum (ewald.cpp:403-410), the O(N NT)
// direct sum (kernels.cpp:27-82), and the GPU precompute of the mollified
// Green's function (greens.cpp:22-113).
#include <algorithm>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int TPB = 256;

inline unsigned blocks_for(int64_t n, int tpb = TPB) {
    return static_cast<unsigned>((n + tpb - 1) / tpb);
}

// u = (uF + uR) + self, in the reference's order (ewald.cpp:403, 408-410)
__global__ void k_epilogue(int64_t nt, const double* __restrict__ uF,
                           const double* __restrict__ uR, const double* __restrict__ str,
                           double coef, double* __restrict__ u) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= 3 * nt) return;
    double v = uF ? uF[q] : 0.0;
    if (uR) v += uR[q];
    if (str) v += coef * str[q];
    u[q] = v;
}

// ---------------------------------------------------------------- direct sum
template <int KIND>
__device__ __forceinline__ void bare(double rx, double ry, double rz, const double* f,
                                     double acc[3]) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double rn = sqrt(r2);
    if (KIND == FSE_STOKESLET) {
        const double rf = rx * f[0] + ry * f[1] + rz * f[2];
        const double a = 1.0 / rn, b = rf / (r2 * rn);
        acc[0] += a * f[0] + b * rx;
        acc[1] += a * f[1] + b * ry;
        acc[2] += a * f[2] + b * rz;
    } else if (KIND == FSE_STRESSLET) {
        const double r[3] = {rx, ry, rz};
        double rfr = 0;
#pragma unroll
        for (int l = 0; l < 3; ++l)
#pragma unroll
            for (int m = 0; m < 3; ++m) rfr += r[l] * f[3 * l + m] * r[m];
        const double c = -6.0 * rfr / (r2 * r2 * rn);
        acc[0] += c * rx;
        acc[1] += c * ry;
        acc[2] += c * rz;
    } else {
        const double inv_r3 = 1.0 / (r2 * rn);
        acc[0] += (f[1] * rz - f[2] * ry) * inv_r3;
        acc[1] += (f[2] * rx - f[0] * rz) * inv_r3;
        acc[2] += (f[0] * ry - f[1] * rx) * inv_r3;
    }
}

template <int KIND>
__global__ void __launch_bounds__(TPB) k_direct(const double* __restrict__ pos,
                                                const double* __restrict__ str, int64_t n,
                                                const double* __restrict__ tgt, int64_t nt,
                                                int exclude_self, double* __restrict__ u,
                                                int* flags) {
    constexpr int A = KIND == FSE_STRESSLET ? 9 : 3;
    __shared__ double sp[TPB][3];
    __shared__ double sf[TPB][A];
    const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const bool valid = m < nt;
    double x = 0, y = 0, z = 0;
    if (valid) {
        x = tgt[3 * m];
        y = tgt[3 * m + 1];
        z = tgt[3 * m + 2];
    }
    double acc[3] = {0, 0, 0};
    bool coincident = false;
    for (int64_t base = 0; base < n; base += TPB) {
        const int64_t s = base + threadIdx.x;
        if (s < n) {
            sp[threadIdx.x][0] = pos[3 * s];
            sp[threadIdx.x][1] = pos[3 * s + 1];
            sp[threadIdx.x][2] = pos[3 * s + 2];
#pragma unroll
            for (int c = 0; c < A; ++c) sf[threadIdx.x][c] = str[s * A + c];
        }
        __syncthreads();
        const int cnt = static_cast<int>(n - base < TPB ? n - base : TPB);
        if (valid)
            for (int j = 0; j < cnt; ++j) {
                if (exclude_self && base + j == m) continue;
                const double rx = x - sp[j][0], ry = y - sp[j][1], rz = z - sp[j][2];
                if (rx == 0 && ry == 0 && rz == 0) {
                    coincident = true;
                    continue;
                }
                bare<KIND>(rx, ry, rz, sf[j], acc);
            }
        __syncthreads();
    }
    if (coincident) atomicOr(flags, FLAG_COINCIDENT);
    if (valid) {
        u[3 * m] = acc[0];
        u[3 * m + 1] = acc[1];
        u[3 * m + 2] = acc[2];
    }
}

// ------------------------------------------------------------------- Green
__device__ double d_sinc(double x) {
    if (fabs(x) < 1e-8) return 1.0 - x * x / 6.0;
    return sin(x) / x;
}

// greens.cpp:22-26
__device__ double d_hhat(double k, double R) {
    const double s = d_sinc(0.5 * R * k);
    return 2.0 * M_PI * R * R * s * s;
}

// greens.cpp:28-46.  The reference evaluates Rk >= 0.5 in x87 long double;
// there is no long double on the GPU, so 0.5 <= Rk < 2 uses the convergent
// alternating series  Bhat/(pi R^4) = sum_m c_m (Rk)^{2m},
//   c_m = 4 (-1)^m (2m+3)(2m+2)/(2m+4)!  (c_0..c_6 are the reference's own
// coefficients), which has no cancellation there, and Rk >= 2 the closed form
// in double (cancellation <= 2 bits).  Rk < 0.5 is the reference's series.
__device__ double d_bhat(double k, double R) {
    const double t = R * k;
    const double piR4 = M_PI * R * R * R * R;
    if (t < 0.5) {
        const double t2 = t * t;
        return piR4 * (1.0 + t2 * (-1.0 / 9.0 + t2 * (1.0 / 240.0 +
                       t2 * (-1.0 / 12600.0 + t2 * (1.0 / 1088640.0 +
                       t2 * (-1.0 / 139708800.0 + t2 / 24908083200.0))))));
    }
    if (t < 2.0) {
        constexpr int NT = 16;
        double c[NT];
        c[0] = 1.0;
        for (int m = 0; m + 1 < NT; ++m)
            c[m + 1] = -c[m] * (2.0 * m + 4.0) / ((2.0 * m + 2.0) * (2.0 * m + 3.0) * (2.0 * m + 6.0));
        const double t2 = t * t;
        double acc = c[NT - 1];
        for (int m = NT - 2; m >= 0; --m) acc = acc * t2 + c[m];
        return piR4 * acc;
    }
    // The reference forms R k in long double: at large Rk the rounding of the
    // double product (~1e-16 Rk absolute) would move cos/sin by ~1e-13 and
    // the stresslet multiplier amplifies that.  Carry the exact product as
    // th + tl (FMA two-product) and correct cos/sin to first order in tl.
    const double th = R * k;
    const double tl = fma(R, k, -th);
    double sn, cs;
    sincos(th, &sn, &cs);
    const double c = cs - sn * tl, s = sn + cs * tl;
    const double t2 = fma(th, th, 2.0 * th * tl);
    const double num = (2.0 - t2) * c + 2.0 * th * s + 2.0 * tl * s - 2.0;
    const double t4 = t2 * t2;
    return 4.0 * M_PI * num / t4 * (R * R * R * R);
}

// octant of the sM^3 wavenumber grid (greens.cpp:62-79): index q <= sM/2 has
// n_a = q (q = sM/2 is n = -sM/2, same k2), k = sqrt((k2(i) + k2(j)) + k2(l)) in
// the reference's summation order
__global__ void k_green_octant(int gkind, int sM, double dk, double R, double* __restrict__ oct) {
    const int nq = sM / 2 + 1;
    const int64_t tot = static_cast<int64_t>(nq) * nq * nq;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < tot;
         q += stride) {
        const int l = static_cast<int>(q % nq);
        const int j = static_cast<int>((q / nq) % nq);
        const int i = static_cast<int>(q / (static_cast<int64_t>(nq) * nq));
        auto sgn = [&](int a) { return a < sM / 2 ? a : a - sM; };
        const double ki = dk * sgn(i), kj = dk * sgn(j), kl = dk * sgn(l);
        const double k2ij = ki * ki + kj * kj;
        const double k = sqrt(k2ij + kl * kl);
        oct[q] = gkind == FSE_HARMONIC ? d_hhat(k, R) : d_bhat(k, R);
    }
}

// half[kx][ky][kz] = T[fold(kx)][fold(ky)][kz], fold(k) = min(k, D - k)
__global__ void k_green_unfold(int Mt, const double* __restrict__ T, double* __restrict__ half) {
    const int D = 2 * Mt, Dh = Mt + 1;
    const int64_t tot = static_cast<int64_t>(D) * D * Dh;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < tot;
         q += stride) {
        const int l = static_cast<int>(q % Dh);
        const int j = static_cast<int>((q / Dh) % D);
        const int i = static_cast<int>(q / (static_cast<int64_t>(Dh) * D));
        const int fi = i <= Mt ? i : D - i, fj = j <= Mt ? j : D - j;
        half[q] = T[(static_cast<int64_t>(fi) * Dh + fj) * Dh + l];
    }
}

__global__ void k_full_to_half(int D, const double* __restrict__ full, double* __restrict__ half) {
    const int Dh = D / 2 + 1;
    const int64_t tot = static_cast<int64_t>(D) * D * Dh;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < tot;
         q += stride) {
        const int64_t l = q % Dh, ij = q / Dh;
        half[q] = full[ij * D + l];
    }
}

// the table is even in k, so entries with l > D/2 mirror (-i, -j, -l)
__global__ void k_half_to_full(int D, const double* __restrict__ half, double* __restrict__ full) {
    const int Dh = D / 2 + 1;
    const int64_t tot = static_cast<int64_t>(D) * D * D;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < tot;
         q += stride) {
        int l = static_cast<int>(q % D);
        int j = static_cast<int>((q / D) % D);
        int i = static_cast<int>(q / (static_cast<int64_t>(D) * D));
        if (l >= Dh) {
            l = D - l;
            j = (D - j) % D;
            i = (D - i) % D;
        }
        full[q] = half[(static_cast<int64_t>(i) * D + j) * Dh + l];
    }
}

// DFMA throughput probe (roofline denominator for the FP64-bound stages):
// 8 independent FMA chains per thread, no memory traffic.
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double seed) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
    const double m = 0.999999999, c = 1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

unsigned grid_stride_blocks(int64_t n) {
    int64_t b = (n + TPB - 1) / TPB;
    const int64_t cap = 148 * 32;
    return static_cast<unsigned>(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

double measure_dfma_tflops(const Launch& L, double* scratch) {
    int sms = 148;
    int dev = 0;
    FSE_CU(cudaGetDevice(&dev));
    FSE_CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned blocks = static_cast<unsigned>(sms) * 8;
    const int iters = 1 << 14;
    cudaEvent_t a, b;
    FSE_CU(cudaEventCreate(&a));
    FSE_CU(cudaEventCreate(&b));
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
        FSE_CU(cudaEventRecord(a, L.s));
        k_dfma_peak<<<blocks, 256, 0, L.s>>>(scratch, iters, 1.0 + rep);
        FSE_CU(cudaEventRecord(b, L.s));
        FSE_CU(cudaEventSynchronize(b));
        float ms = 0;
        FSE_CU(cudaEventElapsedTime(&ms, a, b));
        const double flops = 2.0 * 8.0 * iters * 256.0 * blocks;
        if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *L.launches += 4;
    return best;
}

void launch_epilogue(const Launch& L, int64_t nt, const double* uF, const double* uR,
                     const double* str_self, double self_coef, double* u) {
    if (nt <= 0) return;
    k_epilogue<<<blocks_for(3 * nt), TPB, 0, L.s>>>(nt, uF, uR, str_self, self_coef, u);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_direct(const Launch& L, int kind, const double* pos, const double* str, int64_t n,
                   const double* tgt, int64_t nt, int exclude_self, double* u, int* flags) {
    if (nt <= 0) return;
    const unsigned b = blocks_for(nt);
    if (kind == FSE_STOKESLET)
        k_direct<FSE_STOKESLET><<<b, TPB, 0, L.s>>>(pos, str, n, tgt, nt, exclude_self, u, flags);
    else if (kind == FSE_STRESSLET)
        k_direct<FSE_STRESSLET><<<b, TPB, 0, L.s>>>(pos, str, n, tgt, nt, exclude_self, u, flags);
    else
        k_direct<FSE_ROTLET><<<b, TPB, 0, L.s>>>(pos, str, n, tgt, nt, exclude_self, u, flags);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_green_octant(const Launch& L, int gkind, int sM, double dk, double R, double* oct) {
    const int64_t nq = sM / 2 + 1;
    k_green_octant<<<grid_stride_blocks(nq * nq * nq), TPB, 0, L.s>>>(gkind, sM, dk, R, oct);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_green_unfold(const Launch& L, int Mt, const double* T, double* half) {
    const int64_t D = 2 * Mt;
    k_green_unfold<<<grid_stride_blocks(D * D * (Mt + 1)), TPB, 0, L.s>>>(Mt, T, half);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_green_full_to_half(const Launch& L, int D, const double* full, double* half) {
    const int64_t n = static_cast<int64_t>(D) * D * (D / 2 + 1);
    k_full_to_half<<<grid_stride_blocks(n), TPB, 0, L.s>>>(D, full, half);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_green_half_to_full(const Launch& L, int D, const double* half, double* full) {
    const int64_t n = static_cast<int64_t>(D) * D * D;
    k_half_to_full<<<grid_stride_blocks(n), TPB, 0, L.s>>>(D, half, full);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

// ---------------------------------------------------------------- x-pass probe
// Diagnostics for fse_cuda_xscale_probe: deterministic pseudo-random spectra
// and Green's tables from splitmix64(seed + index), u = (z >> 11) 2^-53
// (tests/test_gpu_xpass_oracle.py regenerates the same values in numpy).
__device__ __forceinline__ double probe_u(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return static_cast<double>(x >> 11) * 0x1.0p-53;
}

__global__ void k_probe_fill(double2* C, int64_t n, uint64_t seed) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        C[q] = make_double2(probe_u(seed + 2 * q) - 0.5, probe_u(seed + 2 * q + 1) - 0.5);
}

__global__ void k_probe_green(double* G, int64_t n, uint64_t seed) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        G[q] = 0.5 + probe_u(seed + q);
}

// out[p][c][x] = C[c][x][ky_p][kz_p] (c < 3, x < Mt); gcol[p][kx] = G[kx][ky_p][kz_p]
__global__ void k_probe_extract(const double2* C, const double* G, int Mt, int D, int nprobe,
                                const int* ky, const int* kz, double2* out, double* gcol) {
    const int Dh = D / 2 + 1;
    const int64_t n = static_cast<int64_t>(nprobe) * 3 * Mt;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(q / (3 * Mt));
        const int r = static_cast<int>(q - static_cast<int64_t>(p) * 3 * Mt);
        const int c = r / Mt, x = r - c * Mt;
        out[q] = C[((static_cast<int64_t>(c) * Mt + x) * D + ky[p]) * Dh + kz[p]];
    }
    const int64_t m = static_cast<int64_t>(nprobe) * D;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < m;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(q / D), kx = static_cast<int>(q - static_cast<int64_t>(p) * D);
        gcol[q] = G[(static_cast<int64_t>(kx) * D + ky[p]) * Dh + kz[p]];
    }
}

void launch_probe_fill(const Launch& L, double2* C, int64_t n, uint64_t seed) {
    k_probe_fill<<<grid_stride_blocks(n), TPB, 0, L.s>>>(C, n, seed);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_probe_green(const Launch& L, double* G, int64_t n, uint64_t seed) {
    k_probe_green<<<grid_stride_blocks(n), TPB, 0, L.s>>>(G, n, seed);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_probe_extract(const Launch& L, const double2* C, const double* G, int Mt, int D,
                          int nprobe, const int* ky, const int* kz, double2* out, double* gcol) {
    const int64_t n = static_cast<int64_t>(nprobe) * (3 * Mt > D ? 3 * Mt : D);
    k_probe_extract<<<grid_stride_blocks(n), TPB, 0, L.s>>>(C, G, Mt, D, nprobe, ky, kz, out,
                                                            gcol);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
