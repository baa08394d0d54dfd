// k_fft.cuh -- the hand-written fp64 FFT engine (k_fft.cu) interface.
#pragma once

#include <vector>

#include "fse_internal.cuh"

namespace fsecu {

constexpr int kFftMaxStages = 16;

// division by an invariant 32-bit divisor d via multiply-high (n < 2^31):
// q = (umulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1
struct FDiv {
    uint32_t d, m, l;
};

inline __host__ __device__ FDiv make_fdiv(uint32_t d) {
#ifdef __CUDA_ARCH__
    // kernels build these per CTA: clz instead of the loop, and the 64-bit
    // quotient from one double division (numerator (2^l - d) 2^32 is exact in
    // double; the rounded-toward-zero quotient is at most one off) instead of
    // the ~100-instruction u64 division routine
    const uint32_t l = d <= 1u ? 0u : 32u - static_cast<uint32_t>(__clz(d - 1u));
    const uint64_t num = ((1ull << l) - d) << 32;
    uint64_t q = static_cast<uint64_t>(__ddiv_rz(static_cast<double>(num), static_cast<double>(d)));
    const int64_t r = static_cast<int64_t>(num - q * d);
    if (r < 0) --q;
    else if (r >= static_cast<int64_t>(d)) ++q;
    return FDiv{d, static_cast<uint32_t>(q + 1), l};
#else
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
    return FDiv{d, static_cast<uint32_t>(m), l};
#endif
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FDiv& f) {
    return (__umulhi(n, f.m) + n) >> f.l;
}
__device__ __forceinline__ uint32_t fmod_(uint32_t n, uint32_t q, const FDiv& f) { return n - q * f.d; }
#endif

// device-side plan of a length-D transform (passed by value to kernels)
struct FftPlan {
    int D;
    int nst;
    int p[kFftMaxStages];   // radix of each stage
    int Ns[kFftMaxStages];  // product of the earlier radices
    int tw[kFftMaxStages];  // offset of the stage's twiddle table (double2 units)
    FDiv dnb[kFftMaxStages];   // D / p
    FDiv dNs[kFftMaxStages];   // Ns
    FDiv dP[kFftMaxStages];    // p
    FDiv dNsP[kFftMaxStages];  // Ns p
    FDiv dD;                   // D
    int tw_elems;           // twiddle table length (copied to shared memory)
    const double2* wd;      // three-level engine: W_D^t, t < D, in global memory
    int two_bufs;           // a generic stage needs a second column buffer
    int buf_elems;          // padded column-buffer length (set per launch)
};

struct HostFftPlan {
    FftPlan dev;
    std::vector<double2> tw;  // concatenated twiddle tables (copied to shared memory)
    std::vector<int> radices;
    bool generic = false;     // a non-register (generic DFT) stage is present
    int eng = 0;              // 0: shared-memory Stockham; >0: two-level register engine
    bool blue = false;        // Bluestein over an Mb = D1 D2 register engine (eng 5..7)
    int D1 = 0, D2 = 0;       // D = D1 * D2 for eng > 0 (three-level: D = D1 D2 D3)
    int D3 = 1;
    int tw_staged = -1;       // leading entries of tw staged in shared memory (-1: all)
};

HostFftPlan make_fft_plan(int D);

// diagnostics: FFT of ncols contiguous columns of length D (in place, device)
void fft_test_columns(const Launch& L, const HostFftPlan& h, const double2* d_tw, double2* data,
                      int ncols, int inverse);

// R (a x nx x Mt^2 real, this slab's planes) -> B (a x nx x Mt x Dh) -> C (slab-blocked
// send layout, see spec_row in k_fft.cu; one GPU: a x Mt x D x Dh)
// peers: destinations of the spectrum blocks (peer-direct exchange); null =
// the local exchange buffer C
void launch_fft_forward_zy(const Launch& L, const HostFftPlan& h, const double2* d_tw,
                           const GridParams& g, int ncomp, const double* R, double2* B,
                           double2* C, const BlockDest* peers = nullptr);
// C (receive layout, ky rows [ky_lo, ky_lo + nky)): forward x-FFT, multiply by
// A_eff(k) G(k) / D^3, inverse x-FFT, in place (3 comps out)
// peers: where the results of each x block go (peer-direct exchange); null =
// in place
// d_ex: scratch for the D per-axis exp factors of the multiplier
void fft_xscale_check(const HostFftPlan& h, int kind);
void launch_fft_xscale(const Launch& L, const HostFftPlan& h, const double2* d_tw,
                       const GridParams& g, int kind, const double* G, double2* C,
                       double* d_ex, const BlockDest* peers = nullptr);
// C (send layout, 3 comps in blocks of A) -> B (j < Mt) -> W (3 x nx x Mt^2 real)
void launch_fft_inverse_yz(const Launch& L, const HostFftPlan& h, const double2* d_tw,
                           const GridParams& g, int A, double2* C, double2* B, double* W,
                           int ncomp = 3);
// x-pass multiplier kind of fse::freespace_solve (one component, times G only)
constexpr int KIND_SCALAR_X = 3;

}  // namespace fsecu
