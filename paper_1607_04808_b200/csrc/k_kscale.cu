// k_kscale.cu -- pointwise k-space scaling (ewald.cpp:216-293).
//
// The fse::kspace_scale drop-in: the reference multiplier verbatim on D^3
// C2C planes.  The hot path does not use it: there the multiplier is fused
// into the x pass (k_fft.cu k_xscale*) in its Nyquist-exact half-spectrum form
//     A_eff(k) = (A(k) + A(k~)) / 2,
// k~ = k with every component on the Nyquist index (D/2, assigned -dk D/2 by
// the reference, ewald.cpp:235) negated.  The reference keeps Re(IFFT) of the
// full spectrum (ewald.cpp:343), which is the C2R inverse of the Hermitian part
// of A(k) ghat(idx) = A_eff(k) ghat(idx) for the transform of real data
// (SURVEY.md 8a A7).
#include "fse_internal.cuh"

namespace fsecu {

namespace {

struct C2 {
    double re, im;
};

template <int KIND>
__device__ __forceinline__ void apply(const double k[3], double k2, double gval, double rem,
                                      double inv4xi2, const C2* g, C2* out) {
    if (KIND == FSE_STOKESLET) {
        // -(k^2 I - k k)(1 + k^2/4xi^2) Bhat
        const double b = -gval * (1.0 + k2 * inv4xi2) * rem;
        const double kgr = k[0] * g[0].re + k[1] * g[1].re + k[2] * g[2].re;
        const double kgi = k[0] * g[0].im + k[1] * g[1].im + k[2] * g[2].im;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            out[p].re = b * (k2 * g[p].re - k[p] * kgr);
            out[p].im = b * (k2 * g[p].im - k[p] * kgi);
        }
    } else if (KIND == FSE_STRESSLET) {
        const double b = gval * (1.0 + k2 * inv4xi2) * rem;
        double ar[3] = {0, 0, 0}, ai[3] = {0, 0, 0}, br[3] = {0, 0, 0}, bi[3] = {0, 0, 0};
        double trr = 0, tri = 0, kgkr = 0, kgki = 0;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            trr += g[3 * p + p].re;
            tri += g[3 * p + p].im;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                ar[p] += g[3 * p + q].re * k[q];
                ai[p] += g[3 * p + q].im * k[q];
                br[q] += k[p] * g[3 * p + q].re;
                bi[q] += k[p] * g[3 * p + q].im;
            }
        }
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            kgkr += k[p] * ar[p];
            kgki += k[p] * ai[p];
        }
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const double vr = k2 * (ar[p] + br[p] + k[p] * trr) - 2.0 * k[p] * kgkr;
            const double vi = k2 * (ai[p] + bi[p] + k[p] * tri) - 2.0 * k[p] * kgki;
            out[p].re = b * vi;  // (0, -b) (vr + i vi)
            out[p].im = -b * vr;
        }
    } else {
        // -i Hhat (ghat x k)
        const double cm = -gval * rem;
        const double vr[3] = {g[1].re * k[2] - g[2].re * k[1], g[2].re * k[0] - g[0].re * k[2],
                              g[0].re * k[1] - g[1].re * k[0]};
        const double vi[3] = {g[1].im * k[2] - g[2].im * k[1], g[2].im * k[0] - g[0].im * k[2],
                              g[0].im * k[1] - g[1].im * k[0]};
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            out[p].re = -cm * vi[p];
            out[p].im = cm * vr[p];
        }
    }
}

__device__ __forceinline__ double kax(int q, int D, double dk) {
    return dk * (q < D / 2 ? q : q - D);
}

template <int KIND>
__global__ void __launch_bounds__(256) k_kscale_full(GridParams g, const double* __restrict__ G,
                                                     const double2* __restrict__ gh_in,
                                                     double2* __restrict__ out) {
    constexpr int A = KIND == FSE_STRESSLET ? 9 : 3;
    const int64_t T = static_cast<int64_t>(g.D) * g.D * g.D;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < T;
         idx += stride) {
        const int l = static_cast<int>(idx % g.D);
        const int j = static_cast<int>((idx / g.D) % g.D);
        const int i = static_cast<int>(idx / (static_cast<int64_t>(g.D) * g.D));
        const double k[3] = {kax(i, g.D, g.dk), kax(j, g.D, g.dk), kax(l, g.D, g.dk)};
        const double k2 = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
        const double rem = exp(-(1.0 - g.eta) * k2 * g.inv4xi2);
        C2 gh[A];
#pragma unroll
        for (int c = 0; c < A; ++c) {
            const double2 v = gh_in[c * T + idx];
            gh[c].re = v.x;
            gh[c].im = v.y;
        }
        C2 o[3];
        apply<KIND>(k, k2, G[idx], rem, g.inv4xi2, gh, o);
#pragma unroll
        for (int p = 0; p < 3; ++p) out[p * T + idx] = make_double2(o[p].re, o[p].im);
    }
}

__global__ void k_scale_complex(double2* d, int64_t n, double s) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
         q += stride) {
        const double2 v = d[q];
        d[q] = make_double2(v.x * s, v.y * s);
    }
}

unsigned grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    const int64_t cap = 148 * 16;
    return static_cast<unsigned>(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

void launch_kscale_full(const Launch& L, const GridParams& g, int kind, const double* Gfull,
                        const double2* ghat, double2* out) {
    const int64_t T = static_cast<int64_t>(g.D) * g.D * g.D;
    const unsigned b = grid_for(T);
    if (kind == FSE_STOKESLET)
        k_kscale_full<FSE_STOKESLET><<<b, 256, 0, L.s>>>(g, Gfull, ghat, out);
    else if (kind == FSE_STRESSLET)
        k_kscale_full<FSE_STRESSLET><<<b, 256, 0, L.s>>>(g, Gfull, ghat, out);
    else
        k_kscale_full<FSE_ROTLET><<<b, 256, 0, L.s>>>(g, Gfull, ghat, out);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_scale_complex(const Launch& L, double2* data, int64_t n, double s) {
    k_scale_complex<<<grid_for(n), 256, 0, L.s>>>(data, n, s);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
