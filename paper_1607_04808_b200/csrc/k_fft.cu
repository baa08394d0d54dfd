// k_fft.cu -- hand-written fp64 FFTs for the zero-padded D = 2 Mtilde grid,
// with the k-space scaling fused into the x-pass.
//
// Why not cuFFT: measured on B200 at D = 624 (tools/fft_probe.cu), a 3D
// D2Z runs at ~0.5 TB/s effective and the strided 1D x-pass the pruned
// transform needs takes 7.2 ms per component (it transposes through a
// full-size workspace).  Writing the passes ourselves lets every pass touch
// HBM once and skip the known zeros:
//
//   R  [i][j][n]   Mt^3 real   (spread output, compact)
//   zfwd: rows (i,j), two real rows per complex FFT, Mt inputs    -> B [i][j][kz]  Mt x Mt x Dh
//   yfwd: columns (i,kz), Mt inputs                               -> C [i][ky][kz] Mt x D  x Dh
//   xk  : columns (ky,kz): Mt inputs, FFT_x, multiply by A_eff(k) G(k) / D^3 (all a
//         components at once), inverse FFT_x, keep the Mt outputs -> C (in place, 3 comps)
//   yinv: columns (i,kz), keep j < Mt                             -> B
//   zinv: Hermitian rows, two real rows per complex FFT, keep n < Mt -> W [i][j][n] Mt^3 real
//
// The planes i >= Mt of the x-pass input and j >= Mt of the y-pass input are
// zeros that are never stored; outputs outside the window are never written.
//
// Column engines (a CTA holds NCOL columns of length D in shared memory,
// column-major with one 16-byte pad every 8 elements against bank conflicts):
//  ENG 0: Stockham autosort, one __syncthreads-separated stage per radix
//         (register butterflies for 2/3/4/5/7/8/11/13, one generic DFT stage
//         through a second buffer for any other factor, e.g. 97 in D = 194);
//  ENG>0: two-level register engine (fft_reg.cuh) for D = D1 D2 with
//         register-friendly D1, D2 (624 = 24 x 26, 1200 = 30 x 40,
//         704 = 22 x 32, 242 = 11 x 22): two shared-memory round trips per
//         element instead of one per radix stage.
// Twiddles come from host tables computed in long double, staged in shared
// memory per CTA.
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "fft_reg.cuh"
#include "fse_internal.cuh"
#include "k_fft.cuh"

namespace fsecu {

namespace {

using freg::cadd;
using freg::cis;
using freg::cmul;
using freg::csub;
using freg::Dft;
using freg::pad;

// register staging per thread: at most ~16 complex values per stage
template <int P>
constexpr int maxit() {
    return (16 + P - 1) / P;
}

// one in-place Stockham stage over NCOL columns of length D (every item is read
// before any is written, so the items must fit one batch of maxit<P>() per
// thread: the planner checks)
template <int P>
__device__ __forceinline__ void stage_reg(double2* buf, int D, int ncol, int Ns, const FDiv& fnb,
                                          const FDiv& fNs, const double2* __restrict__ tw, int sgn) {
    constexpr int MI = maxit<P>();
    const int nb = static_cast<int>(fnb.d);
    const int items = nb * ncol;
    double2 v[MI][P];
#pragma unroll
    for (int m = 0; m < MI; ++m) {
        const int it = threadIdx.x + m * blockDim.x;
        if (it < items) {
            const int c = static_cast<int>(fdiv(it, fnb)), b = it - c * nb;
            const int base = c * D + b;
#pragma unroll
            for (int r = 0; r < P; ++r) v[m][r] = buf[pad(base + r * nb)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MI; ++m) {
        const int it = threadIdx.x + m * blockDim.x;
        if (it < items) {
            const int c = static_cast<int>(fdiv(it, fnb)), b = it - c * nb;
            const int bq = static_cast<int>(fdiv(b, fNs));
            const int k = b - bq * Ns;
            if (k != 0) {
                const double2* t = tw + k * (P - 1);
#pragma unroll
                for (int r = 1; r < P; ++r) {
                    double2 w = t[r - 1];
                    if (sgn > 0) w.y = -w.y;
                    v[m][r] = cmul(v[m][r], w);
                }
            }
            Dft<P>::run(v[m], sgn);
            const int o = c * D + bq * Ns * P + k;
#pragma unroll
            for (int r = 0; r < P; ++r) buf[pad(o + r * Ns)] = v[m][r];
        }
    }
    __syncthreads();
}

// the same stage out of place (plans with a second column buffer), one item per
// thread and trip, for stages with more items than an in-place batch holds
// (D = 1730 = 173 x 2 x 5: 3 x 865 radix-2 and 3 x 346 radix-5 butterflies in the
// x pass).  Instantiated for radix 2 and 5 only (each instance costs the in-place
// stages registers); other overflowing plans are refused by the planner.
template <int P>
__device__ __forceinline__ void stage_reg_oop(const double2* in, double2* out, int D, int ncol, int Ns,
                                           int nb, const double2* __restrict__ tw, int sgn) {
    const int items = nb * ncol;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int c = it / nb, b = it - c * nb;
        const int bq = b / Ns, k = b - bq * Ns;
        double2 v[P];
#pragma unroll
        for (int r = 0; r < P; ++r) v[r] = in[pad(c * D + b + r * nb)];
        if (k != 0) {
            const double2* t = tw + k * (P - 1);
#pragma unroll
            for (int r = 1; r < P; ++r) {
                double2 w = t[r - 1];
                if (sgn > 0) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        Dft<P>::run(v, sgn);
        const int o = c * D + bq * Ns * P + k;
#pragma unroll
        for (int r = 0; r < P; ++r) out[pad(o + r * Ns)] = v[r];
    }
    __syncthreads();
}

// generic radix (any P): out-of-place, each thread computes outputs directly
__device__ __forceinline__ void stage_gen(const double2* in, double2* out, int D, int ncol, int P,
                                          int Ns, const FftPlan& pl, int s,
                                          const double2* __restrict__ W, int sgn) {
    const int tot = D * ncol, NsP = Ns * P, nb = static_cast<int>(pl.dnb[s].d);
    for (int o = threadIdx.x; o < tot; o += blockDim.x) {
        const int c = static_cast<int>(fdiv(o, pl.dD)), e = o - c * D;
        const int eN = static_cast<int>(fdiv(e, pl.dNs[s]));
        const int k = e - eN * Ns;
        const int blk = static_cast<int>(fdiv(e, pl.dNsP[s]));
        const int q = eN - blk * P;
        const int b = blk * Ns + k, m = k + q * Ns;
        double2 acc = make_double2(0.0, 0.0);
        int t = 0;
        for (int r = 0; r < P; ++r) {
            double2 w = W[t];
            if (sgn > 0) w.y = -w.y;
            const double2 x = in[pad(c * D + b + r * nb)];
            acc.x = fma(x.x, w.x, fma(-x.y, w.y, acc.x));
            acc.y = fma(x.x, w.y, fma(x.y, w.x, acc.y));
            t += m;
            if (t >= NsP) t -= NsP;
        }
        out[pad(o)] = acc;
    }
    __syncthreads();
}

// generic odd radix P as the FIRST stage (Ns = 1, no inter-stage twiddles): a
// thread per output pair (q, P - q) of one input group b, using
//   v_r W^{rq} + v_{P-r} W^{-rq} = cos(.) (v_r + v_{P-r}) + i sin(.) (v_r - v_{P-r})
// so X_q = A + iB, X_{P-q} = A - iB with A = v_0 + sum_r cos (v_r + v_{P-r}),
// B = sum_r sin (v_r - v_{P-r}), r = 1 .. (P-1)/2: half the loads and FMAs of
// stage_gen per output.  The lanes of a group load the same inputs (broadcasts).
__device__ __forceinline__ void stage_gen_pairs(const double2* in, double2* out, int D, int ncol,
                                                int P, const FftPlan& pl,
                                                const double2* __restrict__ W, int sgn) {
    const int H = (P - 1) / 2, nb = D / P;
    const int per_b = H + 1;
    const int tot = ncol * nb * per_b;
    for (int it = threadIdx.x; it < tot; it += blockDim.x) {
        const int cb = it / per_b, q = it - cb * per_b;
        const int c = cb / nb, b = cb - c * nb;
        const double2* src = in + 0;
        const int base = c * D + b;
        const double2 v0 = src[pad(base)];
        double2 A = v0, B = make_double2(0.0, 0.0);
        int t = 0;
        for (int r = 1; r <= H; ++r) {
            t += q;
            if (t >= P) t -= P;
            const double2 w = W[t];  // W_P^{rq}: (cos, sin) of the forward sign
            const double cs = w.x, sn = sgn > 0 ? -w.y : w.y;
            const double2 x1 = src[pad(base + r * nb)], x2 = src[pad(base + (P - r) * nb)];
            A.x = fma(cs, x1.x + x2.x, A.x);
            A.y = fma(cs, x1.y + x2.y, A.y);
            B.x = fma(sn, x1.x - x2.x, B.x);
            B.y = fma(sn, x1.y - x2.y, B.y);
        }
        // X_q = A + i B ; X_{P-q} = A - i B   (i B = (-B.y, B.x))
        const int o = c * D + b * P;
        out[pad(o + q)] = make_double2(A.x - B.y, A.y + B.x);
        if (q > 0) out[pad(o + P - q)] = make_double2(A.x + B.y, A.y - B.x);
    }
    __syncthreads();
}

template <int P>
__device__ __forceinline__ void run_radix(double2*& cur, double2*& other, int& s,
                                          const FftPlan& pl, int ncol,
                                          const double2* __restrict__ tw, int sgn) {
    while (s < pl.nst && pl.p[s] == P) {
        // more items than one in-place batch holds (D = 1730: 3 x 865 radix-2
        // butterflies): out of place into the generic plan's second buffer
        bool oop = false;
        if constexpr (P == 2 || P == 5) {
            oop = pl.two_bufs &&
                  static_cast<int>(pl.dnb[s].d) * ncol > maxit<P>() * static_cast<int>(blockDim.x);
            if (oop) {
                stage_reg_oop<P>(cur, other, pl.D, ncol, pl.Ns[s], static_cast<int>(pl.dnb[s].d),
                                 tw + pl.tw[s], sgn);
                double2* t = cur;
                cur = other;
                other = t;
            }
        }
        if (!oop)
            stage_reg<P>(cur, pl.D, ncol, pl.Ns[s], pl.dnb[s], pl.dNs[s], tw + pl.tw[s], sgn);
        ++s;
    }
}

// Stockham engine: the planner orders stages generic, 8s, 4, 2, 3s, 5s, 7s,
// 11s, 13s, so every radix has its own straight-line code region.
__device__ __forceinline__ double2* fft_stockham(double2* a, double2* b, int ncol,
                                                 const FftPlan& pl, const double2* __restrict__ tw,
                                                 int sgn) {
    double2* cur = a;
    double2* other = b;
    int s = 0;
    if (pl.nst > 0 && pl.p[0] > 13) {
        if (pl.Ns[0] == 1 && (pl.p[0] & 1))
            stage_gen_pairs(cur, b, pl.D, ncol, pl.p[0], pl, tw + pl.tw[0], sgn);
        else
            stage_gen(cur, b, pl.D, ncol, pl.p[0], pl.Ns[0], pl, 0, tw + pl.tw[0], sgn);
        cur = b;
        other = a;
        s = 1;
    }
    run_radix<8>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<4>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<2>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<3>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<5>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<7>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<11>(cur, other, s, pl, ncol, tw, sgn);
    run_radix<13>(cur, other, s, pl, ncol, tw, sgn);
    return cur;
}

// engine table: ENG -> (D1, D2).  BLUE engines evaluate a length-N transform
// (N = pl.D, with a prime factor the register DFTs lack, e.g. 298 = 2 x 149)
// by Bluestein's chirp-z identity nk = (n^2 + k^2 - (k - n)^2) / 2 as a
// circular convolution of length Mb = D1 D2 >= 2N - 1 on the register engine.
template <int ENG>
struct Eng {
    static constexpr int D1 = 1, D2 = 1, D3 = 1;
    static constexpr bool BLUE = false;
    static constexpr bool THREE = false;
};
template <>
struct Eng<1> {
    static constexpr int D1 = 24, D2 = 26;
    static constexpr bool BLUE = false;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};
template <>
struct Eng<2> {
    static constexpr int D1 = 30, D2 = 40;
    static constexpr bool BLUE = false;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};
template <>
struct Eng<3> {
    static constexpr int D1 = 22, D2 = 32;
    static constexpr bool BLUE = false;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};
template <>
struct Eng<4> {
    static constexpr int D1 = 11, D2 = 22;
    static constexpr bool BLUE = false;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};
template <>
struct Eng<5> {  // Bluestein, Mb = 400: N <= 200 (cfg1: 194 = 2 x 97)
    static constexpr int D1 = 20, D2 = 20;
    static constexpr bool BLUE = true;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};
template <>
struct Eng<6> {  // Bluestein, Mb = 624: N <= 312 (cfg3: 298 = 2 x 149)
    static constexpr int D1 = 24, D2 = 26;
    static constexpr bool BLUE = true;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};
template <>
struct Eng<7> {  // Bluestein, Mb = 1024: N <= 512
    static constexpr int D1 = 32, D2 = 32;
    static constexpr bool BLUE = true;
    static constexpr bool THREE = false;
    static constexpr int D3 = 1;
};

template <>
struct Eng<8> {  // three-level 1200 = 10 x 12 x 10 (cfg5)
    static constexpr int D1 = 10, D2 = 12, D3 = 10;
    static constexpr bool BLUE = false;
    static constexpr bool THREE = true;
};

template <int ENG>
__device__ __forceinline__ double2* fft_cols(double2* a, double2* b, int ncol, const FftPlan& pl,
                                             const double2* __restrict__ tw, int sgn) {
    if constexpr (ENG == 0) {
        return fft_stockham(a, b, ncol, pl, tw, sgn);
    } else if constexpr (Eng<ENG>::THREE) {
        constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2, D3 = Eng<ENG>::D3;
        freg::fft_cols_3l<D1, D2, D3>(a, ncol, sgn, pl.wd, tw, tw + D2 * D3);
        return a;
    } else if constexpr (!Eng<ENG>::BLUE) {
        constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2;
        freg::fft_cols_2l<D1, D2>(a, ncol, sgn, tw, tw + D1 * D2);
        return a;
    } else {
        // Bluestein: X_k = w_k sum_n (x_n w_n) conj(w_{k-n}), w_n = e^{-i pi n^2 / N}
        // (conjugated for the inverse); the convolution with the precomputed
        // transform Bh of the chirp (1/Mb folded in) runs on the Mb-point engine.
        constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2, Mb = D1 * D2;
        const int N = pl.D;
        const double2* tab = tw + Mb;
        const double2* chirp = tab + freg::tw_total();
        const double2* bh = chirp + N + (sgn < 0 ? 0 : Mb);
        for (int e = threadIdx.x; e < ncol * Mb; e += blockDim.x) {
            const int c = e / Mb, n = e - c * Mb;
            const int idx = freg::ridx<D1, D2>(c, n);
            double2 v = make_double2(0.0, 0.0);
            if (n < N) {
                double2 w = chirp[n];
                if (sgn > 0) w.y = -w.y;
                v = freg::cmul(a[idx], w);
            }
            a[idx] = v;
        }
        __syncthreads();
        freg::fft_cols_2l<D1, D2>(a, ncol, -1, tw, tab);
        for (int e = threadIdx.x; e < ncol * Mb; e += blockDim.x) {
            const int c = e / Mb, n = e - c * Mb;
            const int idx = freg::ridx<D1, D2>(c, n);
            a[idx] = freg::cmul(a[idx], bh[n]);
        }
        __syncthreads();
        freg::fft_cols_2l<D1, D2>(a, ncol, +1, tw, tab);
        for (int e = threadIdx.x; e < ncol * N; e += blockDim.x) {
            const int c = e / N, k = e - c * N;
            const int idx = freg::ridx<D1, D2>(c, k);
            double2 w = chirp[k];
            if (sgn > 0) w.y = -w.y;
            a[idx] = freg::cmul(a[idx], w);
        }
        __syncthreads();
        return a;
    }
}

// column-buffer index: Stockham engine pads one element in 8; the register
// engines use freg::ridx (odd column stride, one pad per D2 elements)
template <int ENG>
__device__ __forceinline__ int cidx(int c, int n, int D) {
    if constexpr (ENG == 0) {
        return pad(c * D + n);
    } else if constexpr (Eng<ENG>::THREE) {
        return freg::idx3<Eng<ENG>::D1, Eng<ENG>::D2, Eng<ENG>::D3>(c, n);
    } else {
        return freg::ridx<Eng<ENG>::D1, Eng<ENG>::D2>(c, n);
    }
}

// Row (c, x, ky) of the spectrum C in the slab-blocked layout
// [blk][c][xl][kyl][kz]: the x-slab owner's send buffer is blocked
// by ky (blk = ky / nkys), the ky-block owner's receive buffer by x (blk =
// x / nxs).  One GPU: one block, i.e. [c][x][ky][kz].  Returns the offset of
// element kz = 0 in double2 units.
__device__ __forceinline__ int64_t spec_row(int blk, int c, int xl, int kyl, int A, int nxs,
                                            int nkys, int Dh) {
    return ((((static_cast<int64_t>(blk) * A + c) * nxs + xl) * nkys + kyl) * Dh);
}

extern __shared__ __align__(16) unsigned char fse_smem[];

// Asynchronous global -> shared copies (LDGSTS): every load of a pass is in
// flight at once instead of one register round trip per element, which is
// what bounds these strided column gathers.  src_bytes = 0 zero-fills.
// L2 prefetch (no register, no completion wait): data a kernel reads later
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void cp16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src, int src_bytes = 8) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// the plan's twiddle table lives after the column buffer(s) in shared memory
__device__ __forceinline__ const double2* stage_twiddles(double2* a, const FftPlan& pl,
                                                         const double2* __restrict__ tw_g) {
    double2* t = a + pl.buf_elems * (pl.two_bufs ? 2 : 1);
    for (int e = threadIdx.x; e < pl.tw_elems; e += blockDim.x) t[e] = __ldg(tw_g + e);
    __syncthreads();
    return t;
}

// the same table staged with cp.async and NOT waited for: the caller's first
// global loads are issued before the wait (freg::pass1_mid + wait_staged)
__device__ __forceinline__ const double2* stage_twiddles_async(double2* a, const FftPlan& pl,
                                                               const double2* __restrict__ tw_g) {
    double2* t = a + pl.buf_elems * (pl.two_bufs ? 2 : 1);
    for (int e = threadIdx.x; e < pl.tw_elems; e += blockDim.x) cp16(t + e, tw_g + e);
    return t;
}
struct WaitStaged {
    __device__ __forceinline__ void operator()() const {
        cp_wait_all();
        __syncthreads();
    }
};

// CTA size per engine.  1200 = 30 x 40 (engine 2): a 40-point register DFT
// needs more than the 128 registers per thread that 256-thread CTAs at two
// per SM allow (it spilled ~1 KB per thread), so its CTAs have 128 threads
// (three columns) and the full 255 registers.
template <int ENG>
constexpr int eng_threads() { return ENG == 2 ? 128 : 256; }
inline int eng_threads_host(int eng) { return eng == 2 ? 128 : 256; }
// resident CTAs per SM the kernels are register-limited for (three-level: 3)
template <int ENG>
constexpr int eng_minb() { return Eng<ENG>::THREE ? 2 : 2; }

// CTA size of the z and y passes (one column transform each, latency-bound)
// at D = 624 (engine 1), per direction: forward FSE_YZF_T, inverse FSE_YZI_T
// threads.  128-thread CTAs (4 columns, ~55 KB) fit four per SM instead of two
// 9-column ones, so the CTAs' load / compute / barrier phases overlap better
// at the same warp count (measured: inverse y + z 2.21 -> 2.11 ms; the forward
// passes lose, 2.12 -> 2.17 ms, and keep 256)
#ifndef FSE_YZF_T
#define FSE_YZF_T 256
#endif
#ifndef FSE_YZI_T
#define FSE_YZI_T 128
#endif
template <int ENG, bool INV>
constexpr int yz_threads() { return ENG == 1 ? (INV ? FSE_YZI_T : FSE_YZF_T) : eng_threads<ENG>(); }
template <int ENG, bool INV>
constexpr int yz_minb() { return ENG == 1 ? 65536 / (yz_threads<ENG, INV>() * 128) : eng_minb<ENG>(); }
inline int yz_threads_host(int eng, bool inv) {
    return eng == 1 ? (inv ? FSE_YZI_T : FSE_YZF_T) : eng_threads_host(eng);
}

// ------------------------------------------------------------------ test kernel
template <int ENG>
__global__ void __launch_bounds__(eng_threads<ENG>(), eng_minb<ENG>()) k_fft_test(FftPlan pl, const double2* __restrict__ tw_g,
                                                     double2* data, int ncol_total, int ncol,
                                                     int sgn) {
    double2* a = reinterpret_cast<double2*>(fse_smem);
    double2* b = a + pl.buf_elems;
    const double2* tw = stage_twiddles(a, pl, tw_g);
    const int c0 = blockIdx.x * ncol;
    const int nc = min(ncol, ncol_total - c0);
    for (int e = threadIdx.x; e < nc * pl.D; e += blockDim.x)
        a[cidx<ENG>(e / pl.D, e % pl.D, pl.D)] = data[static_cast<int64_t>(c0) * pl.D + e];
    __syncthreads();
    double2* r = fft_cols<ENG>(a, b, nc, pl, tw, sgn);
    for (int e = threadIdx.x; e < nc * pl.D; e += blockDim.x)
        data[static_cast<int64_t>(c0) * pl.D + e] = r[cidx<ENG>(e / pl.D, e % pl.D, pl.D)];
}

// ------------------------------------------------------------------ z forward
// column q of the CTA = row pair (comp, i, jp): z[n] = R[i][2jp][n] + i R[i][2jp+1][n]
template <int ENG>
__global__ void __launch_bounds__(yz_threads<ENG, false>(), yz_minb<ENG, false>()) k_zfwd(FftPlan pl, const double2* __restrict__ tw_g,
                                                 int Mt, int nx, int ncomp, int ncol,
                                                 const double* __restrict__ R,
                                                 double2* __restrict__ B) {
    double2* a = reinterpret_cast<double2*>(fse_smem);
    double2* sb = a + pl.buf_elems;
    const double2* tw = stage_twiddles_async(a, pl, tw_g);
    const int D = pl.D, Dh = D / 2 + 1, Jp = (Mt + 1) / 2;
    const int64_t npairs = static_cast<int64_t>(ncomp) * nx * Jp;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * ncol;
    const int nc = static_cast<int>(npairs - q0 < ncol ? npairs - q0 : ncol);
    const int64_t vol = static_cast<int64_t>(nx) * Mt * Mt;  // one component of the slab
    const FDiv fDh = make_fdiv(Dh);
    __shared__ int64_t row0[64];  // first R/W row of the pair, in doubles
    __shared__ int64_t brow[64];  // first B row of the pair, in rows of Dh
    __shared__ int has1[64];
    if (threadIdx.x < nc) {
        const int64_t q = q0 + threadIdx.x;
        const int64_t ci = q / Jp;  // comp * nx + i (slab-local plane i)
        const int jp = static_cast<int>(q - ci * Jp);
        const int64_t comp = ci / nx, i = ci - comp * nx;
        row0[threadIdx.x] = comp * vol + (i * Mt + 2 * jp) * Mt;
        brow[threadIdx.x] = ci * Mt + 2 * jp;
        has1[threadIdx.x] = (2 * jp + 1 < Mt);
    }
    __syncthreads();
    for (int c = 0; c < nc; ++c) {
        const double* row = R + row0[c];
        const bool h1 = has1[c];
        for (int n = threadIdx.x; n < D; n += blockDim.x) {
            double* z = reinterpret_cast<double*>(a + cidx<ENG>(c, n, D));
            if (n < Mt) {
                cp8(z, row + n);
                cp8(z + 1, row + (h1 ? Mt + n : n), h1 ? 8 : 0);
            } else {
                *reinterpret_cast<double2*>(z) = make_double2(0.0, 0.0);
            }
        }
    }
    cp_wait_all();
    __syncthreads();
    double2* r = fft_cols<ENG>(a, sb, nc, pl, tw, -1);
    // split: X0[k] = (Z[k] + conj Z[-k]) / 2, X1[k] = (Z[k] - conj Z[-k]) / (2i)
    for (int e = threadIdx.x; e < nc * Dh; e += blockDim.x) {
        const int c = static_cast<int>(fdiv(e, fDh)), k = e - c * Dh;
        const double2 zk = r[cidx<ENG>(c, k, D)];
        const double2 zm = r[cidx<ENG>(c, (k == 0 ? 0 : D - k), D)];
        const double2 x0 = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        const double2 x1 = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        double2* dst = B + brow[c] * Dh + k;
        dst[0] = x0;
        if (has1[c]) dst[Dh] = x1;
    }
}

// ------------------------------------------------------------------ y passes
// forward: columns (comp, i, kz-tile of ncol); input B[comp][i][j][kz], j < Mt
// inverse: input C[comp][i][ky][kz] (all ky), output B (j < Mt)
template <int ENG, bool INV>
__global__ void __launch_bounds__(yz_threads<ENG, INV>(), yz_minb<ENG, INV>()) k_ypass(FftPlan pl, const double2* __restrict__ tw_g,
                                                  int Mt, int nx, int A, int nxs, int nkys,
                                                  int ncol, double2* __restrict__ B,
                                                  double2* __restrict__ Cb, BlockDest dst) {
    double2* a = reinterpret_cast<double2*>(fse_smem);
    double2* sb = a + pl.buf_elems;
    const double2* tw = stage_twiddles_async(a, pl, tw_g);
    const int D = pl.D, Dh = D / 2 + 1;
    const int ntz = (Dh + ncol - 1) / ncol;
    const int ci = blockIdx.x / ntz;  // comp * nx + i (slab-local plane i)
    const int tz = blockIdx.x - ci * ntz;
    const int comp = ci / nx, xl = ci - comp * nx;
    const int kz0 = tz * ncol;
    const int nc = min(ncol, Dh - kz0);
    const FDiv fnc = make_fdiv(nc);
    const FDiv fky = make_fdiv(nkys);
    double2* Bp = B + static_cast<int64_t>(ci) * Mt * Dh + kz0;   // [j][kz]
    // C row ky of (comp, xl): spec_row(ky / nkys, comp, xl, ky % nkys) (send layout)
    auto crow = [&](int ky) -> int64_t {
        const int blk = static_cast<int>(fdiv(ky, fky));
        return spec_row(blk, comp, xl, ky - blk * nkys, A, nxs, nkys, Dh) + kz0;
    };
    const int nin = INV ? D : Mt;
    for (int e = threadIdx.x; e < nc * nin; e += blockDim.x) {
        const int j = static_cast<int>(fdiv(e, fnc)), c = e - j * nc;  // lanes walk kz
        const double2* src = INV ? Cb + crow(j) + c : Bp + static_cast<int64_t>(j) * Dh + c;
        cp16(a + cidx<ENG>(c, j, D), src);
    }
    if (!INV)
        for (int e = threadIdx.x; e < nc * (D - Mt); e += blockDim.x) {
            const int jj = static_cast<int>(fdiv(e, fnc)), c = e - jj * nc;
            a[cidx<ENG>(c, Mt + jj, D)] = make_double2(0.0, 0.0);
        }
    cp_wait_all();
    __syncthreads();
    double2* r = fft_cols<ENG>(a, sb, nc, pl, tw, INV ? +1 : -1);
    const int nout = INV ? Mt : D;
    const int rb = (comp * nxs + xl) * nkys;  // row of (comp, xl, kyl = 0) within a block
    for (int e = threadIdx.x; e < nc * nout; e += blockDim.x) {
        const int j = static_cast<int>(fdiv(e, fnc)), c = e - j * nc;
        double2* out;
        if (INV) {
            out = Bp + static_cast<int64_t>(j) * Dh + c;
        } else {  // block j / nkys goes to its ky owner
            const int blk = static_cast<int>(fdiv(j, fky));
            out = block_ptr(dst, blk) + static_cast<int64_t>(rb + j - blk * nkys) * Dh + kz0 + c;
        }
        *out = r[cidx<ENG>(c, j, D)];
    }
}

// ------------------------------------------------------------------ x pass + scale
// KIND_SCALAR: fse::freespace_solve (greens.cpp:115-139): one component,
// multiplied by the (real, even) Green's table only.
constexpr int KIND_SCALAR = 3;
template <int KIND>
constexpr int arity_k() { return KIND == FSE_STRESSLET ? 9 : (KIND == KIND_SCALAR ? 1 : 3); }
template <int KIND>
constexpr int nout_k() { return KIND == KIND_SCALAR ? 1 : 3; }

// per-axis factors of the multiplier's exp(-(1 - eta) k^2 / (4 xi^2)):
// ex[q] = exp(-(1 - eta) kax(q)^2 / (4 xi^2)), q < D (once per call)
__global__ void k_ex_axis(int D, double dk, double eta, double inv4xi2, double* __restrict__ ex) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < D) {
        const double kq = dk * (q < D / 2 ? q : q - D);
        ex[q] = exp(-(1.0 - eta) * (kq * kq) * inv4xi2);
    }
}

template <int KIND>
__device__ __forceinline__ void apply(const double k[3], double k2, double gval, double rem,
                                      double inv4xi2, const double2* g, double2* out) {
    if (KIND == FSE_STOKESLET) {
        const double b = -gval * (1.0 + k2 * inv4xi2) * rem;
        const double kgr = k[0] * g[0].x + k[1] * g[1].x + k[2] * g[2].x;
        const double kgi = k[0] * g[0].y + k[1] * g[1].y + k[2] * g[2].y;
#pragma unroll
        for (int p = 0; p < 3; ++p)
            out[p] = make_double2(b * (k2 * g[p].x - k[p] * kgr), b * (k2 * g[p].y - k[p] * kgi));
    } else if (KIND == FSE_STRESSLET) {
        const double b = gval * (1.0 + k2 * inv4xi2) * rem;
        double ar[3] = {0, 0, 0}, ai[3] = {0, 0, 0}, br[3] = {0, 0, 0}, bi[3] = {0, 0, 0};
        double trr = 0, tri = 0, kgkr = 0, kgki = 0;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            trr += g[3 * p + p].x;
            tri += g[3 * p + p].y;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                ar[p] += g[3 * p + q].x * k[q];
                ai[p] += g[3 * p + q].y * k[q];
                br[q] += k[p] * g[3 * p + q].x;
                bi[q] += k[p] * g[3 * p + q].y;
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
            out[p] = make_double2(b * vi, -b * vr);
        }
    } else if (KIND == KIND_SCALAR) {
        out[0] = make_double2(gval * g[0].x, gval * g[0].y);
    } else {
        const double cm = -gval * rem;
        const double vr[3] = {g[1].x * k[2] - g[2].x * k[1], g[2].x * k[0] - g[0].x * k[2],
                              g[0].x * k[1] - g[1].x * k[0]};
        const double vi[3] = {g[1].y * k[2] - g[2].y * k[1], g[2].y * k[0] - g[0].y * k[2],
                              g[0].y * k[1] - g[1].y * k[0]};
#pragma unroll
        for (int p = 0; p < 3; ++p) out[p] = make_double2(-cm * vi[p], cm * vr[p]);
    }
}

__device__ __forceinline__ double kax(int q, int D, double dk) {
    return dk * (q < D / 2 ? q : q - D);
}

// columns (ky, kz-tile); smem holds a*nc columns: column (comp*nc + c)
// x-pass CTA size: the stresslet's nine input columns of one kz need
// 9 max(D1, D2) threads, more than the engine's default CTA for 1200 = 30 x 40,
// 704 = 22 x 32 and the 1024-point Bluestein engine: those launch 384-thread
// CTAs (one per SM).
template <int ENG, int KIND>
constexpr int xs_threads() {
    return (KIND == FSE_STRESSLET && ENG > 0 &&
            9 * (Eng<ENG>::D1 > Eng<ENG>::D2 ? Eng<ENG>::D1 : Eng<ENG>::D2) > eng_threads<ENG>())
               ? 384
               : eng_threads<ENG>();
}
template <int ENG, int KIND>
constexpr int xs_minb() { return xs_threads<ENG, KIND>() > 256 ? 1 : 2; }

template <int ENG, int KIND>
__global__ void __launch_bounds__(xs_threads<ENG, KIND>(), xs_minb<ENG, KIND>()) k_xscale(FftPlan pl, const double2* __restrict__ tw_g,
                                                   GridParams g, int ncol,
                                                   const double* __restrict__ G,
                                                   double2* __restrict__ Cb, BlockDest dst,
                                                   const double* __restrict__ ex_g) {
    constexpr int A = arity_k<KIND>(), NO = nout_k<KIND>();
    double2* a = reinterpret_cast<double2*>(fse_smem);
    double2* sb = a + pl.buf_elems;
    const double2* tw = stage_twiddles_async(a, pl, tw_g);
    const int D = pl.D, Dh = D / 2 + 1, Mt = g.Mt;
    const int ntz = (Dh + ncol - 1) / ncol;
    const int kyl = blockIdx.x / ntz;  // row of this rank's ky block
    const int ky = g.ky_lo + kyl;
    const int tz = blockIdx.x - kyl * ntz;
    const int kz0 = tz * ncol;
    const int nc = min(ncol, Dh - kz0);
    const FDiv fnc = make_fdiv(nc);
    const FDiv fnxs = make_fdiv(g.nxs);
    // C row (comp, x) of this ky in the receive layout (blocked by x / nxs)
    auto crow = [&](int comp, int i) -> int64_t {
        const int blk = static_cast<int>(fdiv(i, fnxs));
        return spec_row(blk, comp, i - blk * g.nxs, kyl, A, g.nxs, g.nkys, Dh) + kz0;
    };
    // Green's column slice G[kx][ky][kz0 + c] staged with the data
    double* Gs = reinterpret_cast<double*>(const_cast<double2*>(tw) + pl.tw_elems);
    for (int e = threadIdx.x; e < nc * D; e += blockDim.x) {
        const int kx = static_cast<int>(fdiv(e, fnc)), c = e - kx * nc;
        cp8(Gs + e, G + (static_cast<int64_t>(kx) * D + ky) * Dh + kz0 + c);
    }
    for (int comp = 0; comp < A; ++comp) {
        for (int e = threadIdx.x; e < nc * Mt; e += blockDim.x) {
            const int i = static_cast<int>(fdiv(e, fnc)), c = e - i * nc;  // lanes walk kz
            cp16(a + cidx<ENG>(comp * nc + c, i, D), Cb + crow(comp, i) + c);
        }
        for (int e = threadIdx.x; e < nc * (D - Mt); e += blockDim.x) {
            const int ii = static_cast<int>(fdiv(e, fnc)), c = e - ii * nc;
            a[cidx<ENG>(comp * nc + c, Mt + ii, D)] = make_double2(0.0, 0.0);
        }
    }
    cp_wait_all();
    __syncthreads();
    double2* r = fft_cols<ENG>(a, sb, A * nc, pl, tw, -1);
    // pointwise multiplier (ewald.cpp:216-293) with the Nyquist-exact
    // Hermitian average (see k_kscale.cu), 1/D^3 folded in
    const int half = D / 2;
    for (int e = threadIdx.x; e < nc * D; e += blockDim.x) {
        const int kx = static_cast<int>(fdiv(e, fnc)), c = e - kx * nc;
        const int kz = kz0 + c;
        double k[3] = {kax(kx, D, g.dk), kax(ky, D, g.dk), kax(kz, D, g.dk)};
        const double k2 = __dadd_rn(__dadd_rn(__dmul_rn(k[0], k[0]), __dmul_rn(k[1], k[1])),
                                    __dmul_rn(k[2], k[2]));
        // exp(-(1 - eta) k^2 / (4 xi^2)) as the product of its per-axis factors
        const double rem = __ldg(ex_g + kx) * __ldg(ex_g + ky) * __ldg(ex_g + kz);
        const double gval = Gs[e];
        double2 gh[A];
#pragma unroll
        for (int q = 0; q < A; ++q) gh[q] = r[cidx<ENG>(q * nc + c, kx, D)];
        double2 out[3];
        apply<KIND>(k, k2, gval, rem, g.inv4xi2, gh, out);
        if (KIND != KIND_SCALAR && (kx == half || ky == half || kz == half)) {
            if (kx == half) k[0] = -k[0];
            if (ky == half) k[1] = -k[1];
            if (kz == half) k[2] = -k[2];
            double2 o2[3];
            apply<KIND>(k, k2, gval, rem, g.inv4xi2, gh, o2);
#pragma unroll
            for (int p = 0; p < 3; ++p)
                out[p] = make_double2(0.5 * (out[p].x + o2[p].x), 0.5 * (out[p].y + o2[p].y));
        }
#pragma unroll
        for (int p = 0; p < NO; ++p)
            r[cidx<ENG>(p * nc + c, kx, D)] = make_double2(out[p].x * g.invD3, out[p].y * g.invD3);
    }
    __syncthreads();
    double2* other = (r == a) ? sb : a;
    double2* r2 = fft_cols<ENG>(r, other, NO * nc, pl, tw, +1);
    // x block i / nxs goes back to its slab owner
    for (int comp = 0; comp < NO; ++comp) {
        for (int e = threadIdx.x; e < nc * Mt; e += blockDim.x) {
            const int i = static_cast<int>(fdiv(e, fnc)), c = e - i * nc;
            const int blk = static_cast<int>(fdiv(i, fnxs));
            const int row = ((comp * g.nxs) + i - blk * g.nxs) * g.nkys + kyl;
            block_ptr(dst, blk)[static_cast<int64_t>(row) * Dh + kz0 + c] =
                r2[cidx<ENG>(comp * nc + c, i, D)];
        }
    }
}

// ------------------------------------------------------------------ z inverse
// row pair (comp, i, jp): Z = X0 + i X1 over the Hermitian extension; keep n < Mt
template <int ENG>
__global__ void __launch_bounds__(yz_threads<ENG, true>(), yz_minb<ENG, true>()) k_zinv(FftPlan pl, const double2* __restrict__ tw_g,
                                                 int Mt, int nx, int ncomp, int ncol,
                                                 const double2* __restrict__ B,
                                                 double* __restrict__ W) {
    double2* a = reinterpret_cast<double2*>(fse_smem);
    double2* sb = a + pl.buf_elems;
    const double2* tw = stage_twiddles_async(a, pl, tw_g);
    const int D = pl.D, Dh = D / 2 + 1, Jp = (Mt + 1) / 2;
    const int64_t npairs = static_cast<int64_t>(ncomp) * nx * Jp;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * ncol;
    const int nc = static_cast<int>(npairs - q0 < ncol ? npairs - q0 : ncol);
    const int64_t vol = static_cast<int64_t>(nx) * Mt * Mt;
    const FDiv fDh = make_fdiv(Dh);
    __shared__ int64_t row0[64];
    __shared__ int64_t brow[64];
    __shared__ int has1[64];
    if (threadIdx.x < nc) {
        const int64_t q = q0 + threadIdx.x;
        const int64_t ci = q / Jp;
        const int jp = static_cast<int>(q - ci * Jp);
        const int64_t comp = ci / nx, i = ci - comp * nx;
        row0[threadIdx.x] = comp * vol + (i * Mt + 2 * jp) * Mt;
        brow[threadIdx.x] = ci * Mt + 2 * jp;
        has1[threadIdx.x] = (2 * jp + 1 < Mt);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nc * Dh; e += blockDim.x) {
        const int c = static_cast<int>(fdiv(e, fDh)), k = e - c * Dh;
        const double2* src = B + brow[c] * Dh + k;
        double2 x0 = src[0];
        double2 x1 = has1[c] ? src[Dh] : make_double2(0.0, 0.0);
        if (k == 0 || k == D / 2) {  // C2R: self-conjugate bins are real
            x0.y = 0.0;
            x1.y = 0.0;
        }
        // Z[k] = X0 + i X1 ; Z[D-k] = conj(X0) + i conj(X1)
        a[cidx<ENG>(c, k, D)] = make_double2(x0.x - x1.y, x0.y + x1.x);
        if (k != 0 && k != D / 2) a[cidx<ENG>(c, D - k, D)] = make_double2(x0.x + x1.y, -x0.y + x1.x);
    }
    cp_wait_all();  // the twiddles (staged asynchronously)
    __syncthreads();
    double2* r = fft_cols<ENG>(a, sb, nc, pl, tw, +1);
    for (int c = 0; c < nc; ++c) {
        double* row = W + row0[c];
        const bool h1 = has1[c];
        for (int n = threadIdx.x; n < Mt; n += blockDim.x) {
            const double2 z = r[cidx<ENG>(c, n, D)];
            row[n] = z.x;
            if (h1) row[Mt + n] = z.y;
        }
    }
}

// ================================================================ v2 kernels
// Register engines (ENG > 0) with direct global I/O (freg::pass1 / pass2):
// the first pass of each transform loads its columns straight from global
// memory into registers (the zero-padded half is never loaded: NZ1) and the
// last pass stores straight to global memory (only the kept window: NOUT2),
// so a plain transform makes one shared-memory round trip (the transpose)
// instead of three (staging, transpose, unstaging).

// z forward: column c = row pair (comp, i, jp), rows contiguous -> n2-fastest
template <int ENG>
__global__ void __launch_bounds__(yz_threads<ENG, false>(), yz_minb<ENG, false>()) k_zfwd2(FftPlan pl, const double2* __restrict__ tw_g,
                                                  int Mt, int nx, int ncomp, int ncol,
                                                  const double* __restrict__ R,
                                                  double2* __restrict__ B) {
    constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2, D = D1 * D2;
    double2* a = reinterpret_cast<double2*>(fse_smem);
    const double2* tw = stage_twiddles_async(a, pl, tw_g);
    const double2* tab = tw + D;
    const int Dh = D / 2 + 1, Jp = (Mt + 1) / 2;
    const int64_t npairs = static_cast<int64_t>(ncomp) * nx * Jp;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * ncol;
    const int nc = static_cast<int>(npairs - q0 < ncol ? npairs - q0 : ncol);
    const int64_t vol = static_cast<int64_t>(nx) * Mt * Mt;
    const FDiv fDh = make_fdiv(Dh);
    __shared__ int64_t row0[64];
    __shared__ int64_t brow[64];
    __shared__ int has1[64];
    if (threadIdx.x < nc) {
        const int64_t q = q0 + threadIdx.x;
        const int64_t ci = q / Jp;
        const int jp = static_cast<int>(q - ci * Jp);
        const int64_t comp = ci / nx, i = ci - comp * nx;
        row0[threadIdx.x] = comp * vol + (i * Mt + 2 * jp) * Mt;
        brow[threadIdx.x] = ci * Mt + 2 * jp;
        has1[threadIdx.x] = (2 * jp + 1 < Mt);
    }
    __syncthreads();
    freg::pass1_mid<D1, D2, false, (D1 + 1) / 2>(a, nc, -1, tw, tab, [&](int c, int n) {
        double2 z = make_double2(0.0, 0.0);
        if (n < Mt) {
            const double* row = R + row0[c];
            z.x = __ldg(row + n);
            if (has1[c]) z.y = __ldg(row + Mt + n);
        }
        return z;
    }, WaitStaged{});
    __syncthreads();
    freg::pass2_smem<D1, D2, false>(a, nc, -1, tab);
    __syncthreads();
    // split: X0[k] = (Z[k] + conj Z[-k]) / 2, X1[k] = (Z[k] - conj Z[-k]) / (2i)
    for (int e = threadIdx.x; e < nc * Dh; e += blockDim.x) {
        const int c = static_cast<int>(fdiv(e, fDh)), k = e - c * Dh;
        const double2 zk = a[freg::ridx<D1, D2>(c, k)];
        const double2 zm = a[freg::ridx<D1, D2>(c, k == 0 ? 0 : D - k)];
        const double2 x0 = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        const double2 x1 = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        double2* dst = B + brow[c] * Dh + k;
        dst[0] = x0;
        if (has1[c]) dst[Dh] = x1;
    }
}

// y passes: column c = (comp, slab plane xl, kz0 + c), columns adjacent in kz -> c-fastest
template <int ENG, bool INV>
__global__ void __launch_bounds__(yz_threads<ENG, INV>(), yz_minb<ENG, INV>()) k_ypass2(FftPlan pl, const double2* __restrict__ tw_g,
                                                   int Mt, int nx, int A, int nxs, int nkys,
                                                   int ncol, double2* __restrict__ B,
                                                   double2* __restrict__ Cb, BlockDest dst) {
    constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2, D = D1 * D2;
    double2* a = reinterpret_cast<double2*>(fse_smem);
    const double2* tw = stage_twiddles_async(a, pl, tw_g);
    const double2* tab = tw + D;
    const int Dh = D / 2 + 1;
    const int ntz = (Dh + ncol - 1) / ncol;
    const int ci = blockIdx.x / ntz;
    const int tz = blockIdx.x - ci * ntz;
    const int comp = ci / nx, xl = ci - comp * nx;
    const int kz0 = tz * ncol;
    const int nc = min(ncol, Dh - kz0);
    const FDiv fky = make_fdiv(nkys);
    double2* Bp = B + static_cast<int64_t>(ci) * Mt * Dh + kz0;
    // spec_row(blk, comp, xl, ky - blk nkys) in 32-bit arithmetic
    const int rbase = (comp * nxs + xl) * nkys, bstep = (A * nxs - 1) * nkys;
    double2* Ck = Cb + kz0;
    auto crow = [&](int ky) -> int64_t {
        const int blk = static_cast<int>(fdiv(ky, fky));
        return static_cast<int64_t>(rbase + blk * bstep + ky) * Dh;
    };
    if (!INV) {
        freg::pass1_mid<D1, D2, true, (D1 + 1) / 2>(a, nc, -1, tw, tab, [&](int c, int n) {
            return n < Mt ? Bp[static_cast<int64_t>(n) * Dh + c] : make_double2(0.0, 0.0);
        }, WaitStaged{});
        __syncthreads();
        // block k / nkys goes to its ky owner
        const int rb = (comp * nxs + xl) * nkys;
        freg::pass2<D1, D2, true, D2>(a, nc, -1, tab, [&](int c, int k, double2 v) {
            const int blk = static_cast<int>(fdiv(k, fky));
            block_ptr(dst, blk)[static_cast<int64_t>(rb + k - blk * nkys) * Dh + kz0 + c] = v;
        });
    } else {
        freg::pass1_mid<D1, D2, true, D1>(a, nc, +1, tw, tab,
                                      [&](int c, int n) { return Ck[crow(n) + c]; }, WaitStaged{});
        __syncthreads();
        freg::pass2<D1, D2, true, D2 / 2>(a, nc, +1, tab, [&](int c, int k, double2 v) {
            Bp[static_cast<int64_t>(k) * Dh + c] = v;  // k < Mt by NOUT2
        });
    }
}

// x pass + multiplier: columns (comp, kz0 + c), c-fastest
// multiplier elements per thread of the v2 x pass: nc <= T / (A max(D1, D2))
// columns per CTA (one pass item per thread), so nc D / T <= min(D1, D2) / A
template <int ENG, int KIND>
constexpr int xs_ng() {
    constexpr int mn = Eng<ENG>::D1 < Eng<ENG>::D2 ? Eng<ENG>::D1 : Eng<ENG>::D2;
    return (mn + arity_k<KIND>() - 1) / arity_k<KIND>();
}

template <int ENG, int KIND>
__global__ void __launch_bounds__(xs_threads<ENG, KIND>(), xs_minb<ENG, KIND>()) k_xscale2(FftPlan pl, const double2* __restrict__ tw_g,
                                                    GridParams g, int ncol,
                                                    const double* __restrict__ G,
                                                    double2* __restrict__ Cb, BlockDest dst,
                                                    const double* __restrict__ ex_g) {
    constexpr int A = arity_k<KIND>(), NO = nout_k<KIND>();
    constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2, D = D1 * D2;
    double2* a = reinterpret_cast<double2*>(fse_smem);
    // twiddles and the exp factor table are staged asynchronously (cp.async),
    // in flight together with pass 1's input loads
    double2* twm = a + pl.buf_elems * (pl.two_bufs ? 2 : 1);
    for (int e = threadIdx.x; e < pl.tw_elems; e += blockDim.x) cp16(twm + e, tw_g + e);
    const double2* tw = twm;
    const double2* tab = tw + D;
    const int Dh = D / 2 + 1, Mt = g.Mt;
    const int ntz = (Dh + ncol - 1) / ncol;
    const int kyl = blockIdx.x / ntz;
    const int ky = g.ky_lo + kyl;
    const int tz = blockIdx.x - kyl * ntz;
    const int kz0 = tz * ncol;
    const int nc = min(ncol, Dh - kz0);
    const FDiv fnc = make_fdiv(nc);
    // spectrum row of (comp, x = i, this ky) in units of Dh: spec_row with
    // blk = i / nxs, xl = i - blk nxs, in 32-bit arithmetic
    const FDiv fnxs = make_fdiv(g.nxs);
    const int bstep = (A - 1) * g.nxs;
    double2* Ck = Cb + kz0;
    auto at = [&](int comp, int i, int c) -> double2* {
        const int blk = static_cast<int>(fdiv(i, fnxs));
        const int row = (i + blk * bstep + comp * g.nxs) * g.nkys + kyl;
        return Ck + static_cast<int64_t>(row) * Dh + c;
    };
    // per-axis factors of exp(-(1 - eta) k^2 / (4 xi^2)) (k_ex_axis, once per
    // call): rem = ex[kx] * ex[ky] * ex[kz]
    double* ex = reinterpret_cast<double*>(const_cast<double2*>(tab) + pl.tw_elems - D);
    for (int q = threadIdx.x; q < D; q += blockDim.x) cp8(ex + q, ex_g + q);
    // forward x-FFT of the A components (pass 1 straight from global memory)
    freg::pass1_mid<D1, D2, true, (D1 + 1) / 2>(
        a, A * nc, -1, tw, tab,
        [&](int col, int n) {
            const int comp = static_cast<int>(fdiv(col, fnc)), c = col - comp * nc;
            return n < Mt ? *at(comp, n, c) : make_double2(0.0, 0.0);
        },
        [] {
            cp_wait_all();
            __syncthreads();
        });
    __syncthreads();
    freg::pass2_smem<D1, D2, true>(a, A * nc, -1, tab);
    // the multiplier's Green's values, all in flight at once (one latency per
    // CTA instead of one per element), issued before the barrier
    constexpr int NG = xs_ng<ENG, KIND>();
    double gv[NG];
    {
        const double* Gk = G + static_cast<int64_t>(ky) * Dh + kz0;
#pragma unroll
        for (int m = 0; m < NG; ++m) {
            const int e = threadIdx.x + m * static_cast<int>(blockDim.x);
            gv[m] = 0.0;
            if (e < nc * D) {
                const int kx = static_cast<int>(fdiv(e, fnc)), c = e - kx * nc;
                gv[m] = __ldg(Gk + static_cast<int64_t>(kx) * D * Dh + c);
            }
        }
    }
    __syncthreads();
    // pointwise multiplier (ewald.cpp:216-293) with the Nyquist-exact
    // Hermitian average (see k_kscale.cu), 1/D^3 folded in
    const int half = D / 2;
    const double ex_y = ex[ky];
#pragma unroll
    for (int m = 0; m < NG; ++m) {
        const int e = threadIdx.x + m * static_cast<int>(blockDim.x);
        if (e >= nc * D) break;
        const int kx = static_cast<int>(fdiv(e, fnc)), c = e - kx * nc;
        const int kz = kz0 + c;
        double k[3] = {kax(kx, D, g.dk), kax(ky, D, g.dk), kax(kz, D, g.dk)};
        const double k2 = __dadd_rn(__dadd_rn(__dmul_rn(k[0], k[0]), __dmul_rn(k[1], k[1])),
                                    __dmul_rn(k[2], k[2]));
        const double rem = ex[kx] * ex_y * ex[kz];
        const double gval = gv[m];
        double2 gh[A];
#pragma unroll
        for (int q = 0; q < A; ++q) gh[q] = a[freg::ridx<D1, D2>(q * nc + c, kx)];
        double2 out[3];
        apply<KIND>(k, k2, gval, rem, g.inv4xi2, gh, out);
        if (KIND != KIND_SCALAR && (kx == half || ky == half || kz == half)) {
            if (kx == half) k[0] = -k[0];
            if (ky == half) k[1] = -k[1];
            if (kz == half) k[2] = -k[2];
            double2 o2[3];
            apply<KIND>(k, k2, gval, rem, g.inv4xi2, gh, o2);
#pragma unroll
            for (int p = 0; p < 3; ++p)
                out[p] = make_double2(0.5 * (out[p].x + o2[p].x), 0.5 * (out[p].y + o2[p].y));
        }
#pragma unroll
        for (int p = 0; p < NO; ++p)
            a[freg::ridx<D1, D2>(p * nc + c, kx)] =
                make_double2(out[p].x * g.invD3, out[p].y * g.invD3);
    }
    __syncthreads();
    // inverse x-FFT of the 3 results (pass 1 in place from shared memory:
    // every item reads and writes only its own (column, n2) elements)
    freg::pass1_inplace<D1, D2, true>(a, NO * nc, +1, tw, tab);
    __syncthreads();
    freg::pass2<D1, D2, true, D2 / 2>(a, NO * nc, +1, tab, [&](int col, int k, double2 v) {
        const int comp = static_cast<int>(fdiv(col, fnc)), c = col - comp * nc;
        // k < Mt by NOUT2; x block k / nxs goes back to its slab owner
        const int blk = static_cast<int>(fdiv(k, fnxs));
        const int row = (comp * g.nxs + k - blk * g.nxs) * g.nkys + kyl;
        block_ptr(dst, blk)[static_cast<int64_t>(row) * Dh + kz0 + c] = v;
    });
}

// z inverse: row pairs, Hermitian extension loaded straight from B, n2-fastest
template <int ENG>
__global__ void __launch_bounds__(yz_threads<ENG, true>(), yz_minb<ENG, true>()) k_zinv2(FftPlan pl, const double2* __restrict__ tw_g,
                                                  int Mt, int nx, int ncomp, int ncol,
                                                  const double2* __restrict__ B,
                                                  double* __restrict__ W) {
    constexpr int D1 = Eng<ENG>::D1, D2 = Eng<ENG>::D2, D = D1 * D2;
    double2* a = reinterpret_cast<double2*>(fse_smem);
    // (624 = 24 x 26: the overlapped staging spills; staged up front there)
    const double2* tw = ENG == 1 ? stage_twiddles(a, pl, tw_g) : stage_twiddles_async(a, pl, tw_g);
    const double2* tab = tw + D;
    const int Dh = D / 2 + 1, Jp = (Mt + 1) / 2;
    const int64_t npairs = static_cast<int64_t>(ncomp) * nx * Jp;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * ncol;
    const int nc = static_cast<int>(npairs - q0 < ncol ? npairs - q0 : ncol);
    const int64_t vol = static_cast<int64_t>(nx) * Mt * Mt;
    __shared__ int64_t row0[64];
    __shared__ int64_t brow[64];
    __shared__ int has1[64];
    if (threadIdx.x < nc) {
        const int64_t q = q0 + threadIdx.x;
        const int64_t ci = q / Jp;
        const int jp = static_cast<int>(q - ci * Jp);
        const int64_t comp = ci / nx, i = ci - comp * nx;
        row0[threadIdx.x] = comp * vol + (i * Mt + 2 * jp) * Mt;
        brow[threadIdx.x] = ci * Mt + 2 * jp;
        has1[threadIdx.x] = (2 * jp + 1 < Mt);
    }
    __syncthreads();
    freg::pass1_mid<D1, D2, false, D1>(a, nc, +1, tw, tab, [&](int c, int n) {
        // Z[n] = X0 + i X1 (n <= D/2); conj(X0[D-n]) + i conj(X1[D-n]) above
        const bool lo = n <= D / 2;
        const int k = lo ? n : D - n;
        const double2* src = B + brow[c] * Dh + k;
        double2 x0 = src[0];
        double2 x1 = has1[c] ? src[Dh] : make_double2(0.0, 0.0);
        if (k == 0 || k == D / 2) {  // C2R: self-conjugate bins are real
            x0.y = 0.0;
            x1.y = 0.0;
        }
        return lo ? make_double2(x0.x - x1.y, x0.y + x1.x)
                  : make_double2(x0.x + x1.y, -x0.y + x1.x);
    }, [] {
        if (ENG != 1) WaitStaged{}();
    });
    __syncthreads();
    freg::pass2<D1, D2, false, D2 / 2>(a, nc, +1, tab, [&](int c, int n, double2 v) {
        double* row = W + row0[c];  // n < Mt by NOUT2
        row[n] = v.x;
        if (has1[c]) row[Mt + n] = v.y;
    });
}

int maxit_host(int p) { return (16 + p - 1) / p; }
bool is_reg_radix(int p) {
    return p == 2 || p == 3 || p == 4 || p == 5 || p == 7 || p == 8 || p == 11 || p == 13;
}

bool g_consts_ready[64] = {};

void upload_consts() {
    int dev = 0;
    FSE_CU(cudaGetDevice(&dev));
    if (dev < 64 && g_consts_ready[dev]) return;
    double cs[4][14] = {}, sn[4][14] = {};
    const int ps[4] = {5, 7, 11, 13};
    for (int k = 0; k < 4; ++k)
        for (int t = 0; t < ps[k]; ++t) {
            const long double ang = 2.0L * 3.141592653589793238462643383279502884L * t / ps[k];
            cs[k][t] = static_cast<double>(cosl(ang));
            sn[k][t] = static_cast<double>(sinl(ang));
        }
    FSE_CU(cudaMemcpyToSymbol(freg::c_rcos, cs, sizeof cs));
    FSE_CU(cudaMemcpyToSymbol(freg::c_rsin, sn, sizeof sn));
    if (dev < 64) g_consts_ready[dev] = true;
}

// D -> two-level engine id and factors
int engine_for(int D, int* D1, int* D2) {
    struct E {
        int D, e, d1, d2;
    };
    const E table[] = {{624, 1, 24, 26}, {1200, 2, 30, 40}, {704, 3, 22, 32}, {242, 4, 11, 22}};
    if (std::getenv("FSE_FFT_STOCKHAM")) return 0;
    // three-level engine, opt-in: measured slower than the two-level ones on B200
    // (cfg5: forward z+y 25.0 vs 18.5 ms, x pass 74.8 vs 71.1 ms, inverse 27.0 vs
    // 17.7 ms; the same split for 624 = 8 x 6 x 13: x pass 9.4 vs 5.6 ms) -- more
    // resident warps, but three shared-memory passes and the staged (v1) kernels
    if (D == 1200 && std::getenv("FSE_FFT_1200_3L")) {  // three-level 10 x 12 x 10
        *D1 = 10;
        *D2 = 12;
        return 8;
    }

    for (const E& t : table)
        if (t.D == D) {
            *D1 = t.d1;
            *D2 = t.d2;
            return t.e;
        }
    // a prime factor beyond the register DFTs (2..13): Bluestein on the
    // smallest register engine with Mb >= 2D - 1 (FSE_FFT_NOBLUE: Stockham's
    // generic O(p^2) stage instead)
    int rem = D;
    for (int p : {2, 3, 5, 7, 11, 13})
        while (rem % p == 0) rem /= p;
    // ... unless that factor is small: Stockham's generic O(p^2) first stage then beats
    // the four engine transforms of a Bluestein column (measured on B200, whole step:
    // D = 348 = 12 x 29 16.3 vs 24.9 ms; but D = 194 = 2 x 97 2.37 vs 1.67 and
    // D = 298 = 2 x 149 22.1 vs 16.0 ms, so the switch sits between 29 and 97)
    if (rem > 48 && !std::getenv("FSE_FFT_NOBLUE")) {
        const E blue[] = {{400, 5, 20, 20}, {624, 6, 24, 26}, {1024, 7, 32, 32}};
        for (const E& t : blue)
            if (t.D >= 2 * D - 1) {
                *D1 = t.d1;
                *D2 = t.d2;
                return t.e;
            }
    }
    return 0;
}

double2 cexp_neg(long double num, long double den) {
    const long double two_pi = 2.0L * 3.141592653589793238462643383279502884L;
    const long double ang = -two_pi * num / den;
    return make_double2(static_cast<double>(cosl(ang)), static_cast<double>(sinl(ang)));
}

constexpr int kThreads = 256;

// which passes use the direct-I/O register kernels (bit 0 z fwd, 1 y fwd,
// 2 x-pass, 3 y inv, 4 z inv).  Measured at D = 624 (24 x 26): z fwd, x-pass
// and z inv gain, y inv loses (register spills at the 2-CTA/SM cap), y fwd
// is even; at D = 1200 (30 x 40, 40-element pass-2 registers) every v2
// pass loses.  FSE_FFT_V2 overrides (profiling aid).
int v2_mask_env() {
    static const int m = [] {
        const char* e = std::getenv("FSE_FFT_V2");
        return e ? std::atoi(e) : -1;
    }();
    return m;
}
template <int ENG>
int v2_mask_for() {
    if (Eng<ENG>::BLUE || Eng<ENG>::THREE) return 0;
    const int e = v2_mask_env();
    if (e >= 0) return e;
    // measured per engine on B200: 624 (cfg2) and 704 (cfg4t) all but the inverse y
    // pass; 1200 (cfg5) all (the x pass since its Green's loads are batched: 66.7 ->
    // 64.9 ms); 242 (cfg1t) all (inverse 0.161 -> 0.123 ms)
    return (ENG == 2 || ENG == 4) ? (1 | 2 | 4 | 8 | 16) : (1 | 2 | 4 | 16);
}
constexpr size_t kSmemCap = 112 * 1024;  // two CTAs per SM

}  // namespace

// ------------------------------------------------------------------ host side
HostFftPlan make_fft_plan(int D) {
    HostFftPlan h;
    std::memset(&h.dev, 0, sizeof h.dev);
    h.dev.D = D;
    h.eng = engine_for(D, &h.D1, &h.D2);
    if (h.eng == 8) {
        // staged: W_{D2 D3}^t (t < D2 D3) and the small register tables; then
        // W_D^t (t < D) read from global memory (dev.wd, set per launch)
        h.D3 = D / (h.D1 * h.D2);
        const int M23 = h.D2 * h.D3;
        for (int t = 0; t < M23; ++t) h.tw.push_back(cexp_neg(t, M23));
        for (int i = 0; i < freg::kNumRegSizes; ++i) {
            const int n = freg::kRegSizes[i];
            for (int t = 0; t < n; ++t) h.tw.push_back(cexp_neg(t, n));
        }
        h.tw_staged = static_cast<int>(h.tw.size());
        for (int t = 0; t < D; ++t) h.tw.push_back(cexp_neg(t, D));
        h.dev.nst = 0;
        h.dev.dD = make_fdiv(D);
        return h;
    }
    if (h.eng > 0) {
        const int Mb = h.D1 * h.D2;  // = D for the plain register engines
        // table: W_Mb^t (t < Mb), then the small register-FFT tables
        for (int t = 0; t < Mb; ++t) h.tw.push_back(cexp_neg(t, Mb));
        for (int i = 0; i < freg::kNumRegSizes; ++i) {
            const int n = freg::kRegSizes[i];
            for (int t = 0; t < n; ++t) h.tw.push_back(cexp_neg(t, n));
        }
        if (Mb != D) {
            // Bluestein: chirp w_n = e^{-i pi n^2 / D} (n^2 reduced mod 2D, long
            // double), then Bh = FFT_Mb(b) / Mb for b_m = conj(w_|m|) on the
            // circular support |m| < D, for the forward and the inverse sign
            h.blue = true;
            const long double pi = 3.141592653589793238462643383279502884L;
            auto w = [&](long long n, int sgn) {
                const long double ang = sgn * pi * static_cast<long double>((n * n) % (2LL * D)) / D;
                return std::complex<long double>(cosl(ang), sinl(ang));
            };
            for (int n = 0; n < D; ++n) {
                const std::complex<long double> c = w(n, -1);
                h.tw.push_back(make_double2(static_cast<double>(c.real()),
                                            static_cast<double>(c.imag())));
            }
            for (int sgn : {-1, +1}) {
                std::vector<std::complex<long double>> b(Mb, 0.0L), B(Mb);
                for (int m = 0; m < D; ++m) {
                    b[m] = std::conj(w(m, sgn));
                    if (m > 0) b[Mb - m] = b[m];
                }
                for (int k = 0; k < Mb; ++k) {  // direct DFT in long double (host, once)
                    std::complex<long double> acc = 0.0L;
                    for (int m = 0; m < Mb; ++m) {
                        const long double ang =
                            -2.0L * pi * static_cast<long double>((static_cast<long long>(k) * m) % Mb) / Mb;
                        acc += b[m] * std::complex<long double>(cosl(ang), sinl(ang));
                    }
                    B[k] = acc / static_cast<long double>(Mb);
                }
                for (int k = 0; k < Mb; ++k)
                    h.tw.push_back(make_double2(static_cast<double>(B[k].real()),
                                                static_cast<double>(B[k].imag())));
            }
        }
        h.dev.nst = 0;
        h.dev.dD = make_fdiv(D);
        return h;
    }
    std::vector<int> rad;
    int rem = D;
    while (rem % 8 == 0) { rad.push_back(8); rem /= 8; }
    while (rem % 4 == 0) { rad.push_back(4); rem /= 4; }
    while (rem % 2 == 0) { rad.push_back(2); rem /= 2; }
    for (int p : {3, 5, 7, 11, 13})
        while (rem % p == 0) { rad.push_back(p); rem /= p; }
    if (rem > 1) rad.insert(rad.begin(), rem);  // one generic stage for the rest
    if (static_cast<int>(rad.size()) > kFftMaxStages) throw Error(FSE_EINVAL, "FFT: too many stages");
    int Ns = 1;
    h.generic = false;
    for (size_t s = 0; s < rad.size(); ++s) {
        const int p = rad[s];
        h.dev.p[s] = p;
        h.dev.Ns[s] = Ns;
        h.dev.tw[s] = static_cast<int>(h.tw.size());
        if (is_reg_radix(p)) {
            for (int k = 0; k < Ns; ++k)
                for (int r = 1; r < p; ++r)
                    h.tw.push_back(cexp_neg((static_cast<long long>(r) * k) %
                                                (static_cast<long long>(Ns) * p),
                                            static_cast<long double>(Ns) * p));
        } else {
            h.generic = true;
            for (int t = 0; t < Ns * p; ++t) h.tw.push_back(cexp_neg(t, static_cast<long double>(Ns) * p));
        }
        if (h.tw.empty()) h.tw.push_back(make_double2(1.0, 0.0));
        Ns *= p;
    }
    h.dev.nst = static_cast<int>(rad.size());
    h.radices = rad;
    h.dev.dD = make_fdiv(D);
    for (int s = 0; s < h.dev.nst; ++s) {
        h.dev.dnb[s] = make_fdiv(D / h.dev.p[s]);
        h.dev.dNs[s] = make_fdiv(h.dev.Ns[s]);
        h.dev.dP[s] = make_fdiv(h.dev.p[s]);
        h.dev.dNsP[s] = make_fdiv(h.dev.Ns[s] * h.dev.p[s]);
    }
    return h;
}

namespace {

size_t col_elems(const HostFftPlan& h, int cols) {
    if (h.eng == 8)  // freg::idx3 layout
        return static_cast<size_t>(cols) * freg::col_stride3(h.dev.D, h.D3) + 8;
    if (h.eng > 0)  // freg::ridx layout (Bluestein: columns of the Mb-point engine)
        return static_cast<size_t>(cols) * freg::col_stride(h.D1, h.D2) + 8;
    return static_cast<size_t>(cols) * h.dev.D + (static_cast<size_t>(cols) * h.dev.D) / 8 + 8;
}

size_t staged_tw(const HostFftPlan& h) {
    return h.tw_staged >= 0 ? static_cast<size_t>(h.tw_staged) : h.tw.size();
}

size_t smem_bytes(const HostFftPlan& h, int cols) {
    return (col_elems(h, cols) * (h.generic ? 2 : 1) + staged_tw(h)) * sizeof(double2);
}

// largest number of units (each `cols_per_unit` columns) that fits the
// shared-memory cap and the engine's per-thread work limits
int units_per_cta(const HostFftPlan& h, int cols_per_unit, size_t cap, int threads) {
    const int D = h.dev.D;
    int best = 0;
    for (int u = 1; u <= 64; ++u) {
        const int cols = u * cols_per_unit;
        if (smem_bytes(h, cols) > cap) break;
        bool ok = true;
        if (h.eng == 8) {
            ok = true;  // the three-level passes loop over their items
        } else if (h.eng > 0) {
            const int T = threads > 0 ? threads : eng_threads_host(h.eng);
            ok = cols * h.D1 <= T && cols * h.D2 <= T;
        } else {
            // in-place stages hold all their items in one register batch; the radix-2
            // and radix-5 stages of a plan with a second buffer (generic first stage)
            // may run out of place in several batches instead
            for (int p : h.radices)
                if (!(h.generic && (p == 2 || p == 5)) && is_reg_radix(p) &&
                    static_cast<long long>(cols) * (D / p) > static_cast<long long>(kThreads) * maxit_host(p))
                    ok = false;
        }
        if (!ok) break;
        best = u;
    }
    return best;
}

// two CTAs per SM when possible, otherwise one CTA with up to 220 KB, and as the
// last resort the sm_100 per-CTA maximum of 227 KB (D = 1730 = 2 x 5 x 173, cfg5's
// tolerance-consistent grid: the x pass of three generic-Stockham columns needs 223 KB)
int units_fit(const HostFftPlan& h, int cols_per_unit, size_t extra_per_unit, int threads = 0) {
    // three-level engine: three CTAs per SM when they fit
    const size_t cap3 = (h.eng == 8) ? static_cast<size_t>(74 * 1024) : kSmemCap;
    for (size_t cap : {cap3, kSmemCap, static_cast<size_t>(220 * 1024),
                       static_cast<size_t>(227 * 1024)}) {
        int u = units_per_cta(h, cols_per_unit, cap, threads);
        while (u > 0 && smem_bytes(h, u * cols_per_unit) + extra_per_unit * u > cap) --u;
        if (u > 0) return u;
    }
    throw Error(FSE_EINVAL, "FFT: grid size does not fit the shared-memory engine");
}

void set_buf(FftPlan& p, const HostFftPlan& h, int cols, const double2* d_tw) {
    p.buf_elems = static_cast<int>(col_elems(h, cols));
    p.wd = d_tw + staged_tw(h);  // three-level engine: the global W_D table
    p.two_bufs = h.generic ? 1 : 0;
    p.tw_elems = static_cast<int>(staged_tw(h));
}

template <class K>
void allow_smem(K kern, size_t bytes) {
    FSE_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
}

// dispatch a callable on the engine id as a compile-time constant
template <class F>
void with_engine(int eng, F&& f) {
    switch (eng) {
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 3: f(std::integral_constant<int, 3>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 5: f(std::integral_constant<int, 5>{}); break;
        case 6: f(std::integral_constant<int, 6>{}); break;
        case 7: f(std::integral_constant<int, 7>{}); break;
        case 8: f(std::integral_constant<int, 8>{}); break;
        default: f(std::integral_constant<int, 0>{}); break;
    }
}

}  // namespace

void fft_test_columns(const Launch& L, const HostFftPlan& h, const double2* d_tw, double2* data,
                      int ncols, int inverse) {
    upload_consts();
    const int u = units_fit(h, 1, 0);
    FftPlan p = h.dev;
    set_buf(p, h, u, d_tw);
    const size_t sm = smem_bytes(h, u);
    with_engine(h.eng, [&](auto E) {
        constexpr int EV = decltype(E)::value;
        allow_smem(k_fft_test<EV>, sm);
        k_fft_test<EV><<<(ncols + u - 1) / u, eng_threads<EV>(), sm, L.s>>>(p, d_tw, data, ncols, u,
                                                                   inverse ? +1 : -1);
    });
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

// local block table: block b of the exchange buffer C (block = ncomp nxs nkys Dh)
BlockDest local_blocks(const GridParams& g, int ncomp, double2* C) {
    BlockDest d{};
    d.base = C;
    d.stride = static_cast<int64_t>(ncomp) * g.nxs * g.nkys * g.Dh;
    d.tab = nullptr;
    return d;
}

void launch_fft_forward_zy(const Launch& L, const HostFftPlan& h, const double2* d_tw,
                           const GridParams& g, int ncomp, const double* R, double2* B,
                           double2* C, const BlockDest* peers) {
    upload_consts();
    const BlockDest dst = peers ? *peers : local_blocks(g, ncomp, C);
    const int Mt = g.Mt, nx = g.nx;
    const int D = h.dev.D, Dh = D / 2 + 1, Jp = (Mt + 1) / 2;
    if (nx <= 0 || ncomp <= 0) return;  // empty slab
    with_engine(h.eng, [&](auto E) {
        constexpr int EV = decltype(E)::value;
        {
            const int u = units_fit(h, 1, 0, yz_threads_host(h.eng, false));
            FftPlan p = h.dev;
            set_buf(p, h, u, d_tw);
            const size_t sm = smem_bytes(h, u);
            const int64_t npairs = static_cast<int64_t>(ncomp) * nx * Jp;
            const unsigned nb = static_cast<unsigned>((npairs + u - 1) / u);
            if constexpr (EV > 0 && !Eng<EV>::BLUE && !Eng<EV>::THREE) {
                if (v2_mask_for<EV>() & 1) {
                    allow_smem(k_zfwd2<EV>, sm);
                    k_zfwd2<EV><<<nb, yz_threads<EV, false>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, u, R, B);
                } else {
                    allow_smem(k_zfwd<EV>, sm);
                    k_zfwd<EV><<<nb, yz_threads<EV, false>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, u, R, B);
                }
            } else {
                allow_smem(k_zfwd<EV>, sm);
                k_zfwd<EV><<<nb, yz_threads<EV, false>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, u, R, B);
            }
            FSE_LAUNCH_CHECK();
            ++*L.launches;
        }
        {
            const int u = std::min(units_fit(h, 1, 0, yz_threads_host(h.eng, false)), Dh);
            FftPlan p = h.dev;
            set_buf(p, h, u, d_tw);
            const size_t sm = smem_bytes(h, u);
            const int ntz = (Dh + u - 1) / u;
            const unsigned nb = static_cast<unsigned>(static_cast<int64_t>(ncomp) * nx * ntz);
            if constexpr (EV > 0 && !Eng<EV>::BLUE && !Eng<EV>::THREE) {
                if (v2_mask_for<EV>() & 2) {
                    allow_smem(k_ypass2<EV, false>, sm);
                    k_ypass2<EV, false><<<nb, yz_threads<EV, false>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, g.nxs,
                                                                   g.nkys, u, B, C, dst);
                } else {
                    allow_smem(k_ypass<EV, false>, sm);
                    k_ypass<EV, false><<<nb, yz_threads<EV, false>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, g.nxs,
                                                                  g.nkys, u, B, C, dst);
                }
            } else {
                allow_smem(k_ypass<EV, false>, sm);
                k_ypass<EV, false><<<nb, yz_threads<EV, false>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, g.nxs,
                                                              g.nkys, u, B, C, dst);
            }
            FSE_LAUNCH_CHECK();
            ++*L.launches;
        }
    });
}

// throws invalid_argument when the x pass of this grid does not fit the FFT
// engines (called before the spectra are allocated)
void fft_xscale_check(const HostFftPlan& h, int kind) {
    const int A = kind == KIND_SCALAR ? 1 : arity_of(kind);
    int xmask = 0;
    with_engine(h.eng, [&](auto E) { xmask = v2_mask_for<decltype(E)::value>(); });
    const size_t gcol = (h.eng > 0 && (xmask & 4)) ? 0 : sizeof(double) * static_cast<size_t>(h.dev.D);
    const int mx = std::max(h.D1, h.D2);
    const int xthr = (A == 9 && h.eng > 0 && 9 * mx > eng_threads_host(h.eng))
                         ? 384
                         : eng_threads_host(h.eng);
    (void)units_fit(h, A, gcol, xthr);
}

void launch_fft_xscale(const Launch& L, const HostFftPlan& h, const double2* d_tw,
                       const GridParams& g, int kind, const double* G, double2* C,
                       double* d_ex, const BlockDest* peers) {
    upload_consts();
    if (g.nky <= 0) return;
    k_ex_axis<<<(h.dev.D + 255) / 256, 256, 0, L.s>>>(h.dev.D, g.dk, g.eta, g.inv4xi2, d_ex);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
    const int A = kind == KIND_SCALAR ? 1 : arity_of(kind);
    // results (3 comps) go back in place (local) or to the x-slab owners
    const BlockDest dst = peers ? *peers : local_blocks(g, A, C);
    const int D = h.dev.D, Dh = D / 2 + 1;
    // v2 (register engines) reads G from global memory; v1 stages it
    int xmask = 0;
    with_engine(h.eng, [&](auto E) { xmask = v2_mask_for<decltype(E)::value>(); });
    const size_t gcol = (h.eng > 0 && (xmask & 4)) ? 0 : sizeof(double) * static_cast<size_t>(D);
    // the stresslet's 9 columns may need a larger CTA (xs_threads)
    const int mx = std::max(h.D1, h.D2);
    const int xthr = (A == 9 && h.eng > 0 && 9 * mx > eng_threads_host(h.eng))
                         ? 384
                         : eng_threads_host(h.eng);
    const int u = std::min(units_fit(h, A, gcol, xthr), Dh);
    FftPlan p = h.dev;
    set_buf(p, h, A * u, d_tw);
    // v2: exp factor table (D doubles) after the twiddles
    const size_t sm = smem_bytes(h, A * u) + gcol * u + (gcol ? 0 : sizeof(double) * D);
    const int ntz = (Dh + u - 1) / u;
    const unsigned blocks = static_cast<unsigned>(g.nky) * ntz;
    if (blocks == 0) return;
    with_engine(h.eng, [&](auto E) {
        constexpr int EV = decltype(E)::value;
        if constexpr (EV > 0 && !Eng<EV>::BLUE && !Eng<EV>::THREE) if (v2_mask_for<EV>() & 4) {
            {
                const int thr = xs_threads<EV, FSE_STOKESLET>();
                const int ng = kind == FSE_STRESSLET ? xs_ng<EV, FSE_STRESSLET>()
                             : kind == KIND_SCALAR ? xs_ng<EV, KIND_SCALAR>()
                                                   : xs_ng<EV, FSE_STOKESLET>();
                const int thr2 = kind == FSE_STRESSLET ? xs_threads<EV, FSE_STRESSLET>() : thr;
                if (u * D > ng * thr2)
                    throw Error(FSE_EINVAL, "x pass: multiplier elements exceed the per-thread batch");
            }
            if (kind == FSE_STOKESLET) {
                allow_smem(k_xscale2<EV, FSE_STOKESLET>, sm);
                k_xscale2<EV, FSE_STOKESLET><<<blocks, xs_threads<EV, FSE_STOKESLET>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
            } else if (kind == FSE_STRESSLET) {
                allow_smem(k_xscale2<EV, FSE_STRESSLET>, sm);
                k_xscale2<EV, FSE_STRESSLET><<<blocks, xs_threads<EV, FSE_STRESSLET>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
            } else if (kind == KIND_SCALAR) {
                allow_smem(k_xscale2<EV, KIND_SCALAR>, sm);
                k_xscale2<EV, KIND_SCALAR><<<blocks, xs_threads<EV, KIND_SCALAR>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
            } else {
                allow_smem(k_xscale2<EV, FSE_ROTLET>, sm);
                k_xscale2<EV, FSE_ROTLET><<<blocks, xs_threads<EV, FSE_ROTLET>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
            }
            return;
        }
        if (kind == FSE_STOKESLET) {
            allow_smem(k_xscale<EV, FSE_STOKESLET>, sm);
            k_xscale<EV, FSE_STOKESLET><<<blocks, xs_threads<EV, FSE_STOKESLET>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
        } else if (kind == FSE_STRESSLET) {
            allow_smem(k_xscale<EV, FSE_STRESSLET>, sm);
            k_xscale<EV, FSE_STRESSLET><<<blocks, xs_threads<EV, FSE_STRESSLET>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
        } else if (kind == KIND_SCALAR) {
            allow_smem(k_xscale<EV, KIND_SCALAR>, sm);
            k_xscale<EV, KIND_SCALAR><<<blocks, xs_threads<EV, KIND_SCALAR>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
        } else {
            allow_smem(k_xscale<EV, FSE_ROTLET>, sm);
            k_xscale<EV, FSE_ROTLET><<<blocks, xs_threads<EV, FSE_ROTLET>(), sm, L.s>>>(p, d_tw, g, u, G, C, dst, d_ex);
        }
    });
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_fft_inverse_yz(const Launch& L, const HostFftPlan& h, const double2* d_tw,
                           const GridParams& g, int A, double2* C, double2* B, double* W,
                           int ncomp) {
    upload_consts();
    const int Mt = g.Mt, nx = g.nx;
    const int D = h.dev.D, Dh = D / 2 + 1, Jp = (Mt + 1) / 2;
    if (nx <= 0) return;  // empty slab
    with_engine(h.eng, [&](auto E) {
        constexpr int EV = decltype(E)::value;
        {
            const int u = std::min(units_fit(h, 1, 0, yz_threads_host(h.eng, true)), Dh);
            FftPlan p = h.dev;
            set_buf(p, h, u, d_tw);
            const size_t sm = smem_bytes(h, u);
            const int ntz = (Dh + u - 1) / u;
            const unsigned nb = static_cast<unsigned>(static_cast<int64_t>(ncomp) * nx * ntz);
            if constexpr (EV > 0 && !Eng<EV>::BLUE && !Eng<EV>::THREE) {
                if (v2_mask_for<EV>() & 8) {
                    allow_smem(k_ypass2<EV, true>, sm);
                    k_ypass2<EV, true><<<nb, yz_threads<EV, true>(), sm, L.s>>>(p, d_tw, Mt, nx, A, g.nxs, g.nkys,
                                                                  u, B, C, BlockDest{});
                } else {
                    allow_smem(k_ypass<EV, true>, sm);
                    k_ypass<EV, true><<<nb, yz_threads<EV, true>(), sm, L.s>>>(p, d_tw, Mt, nx, A, g.nxs, g.nkys, u,
                                                                 B, C, BlockDest{});
                }
            } else {
                allow_smem(k_ypass<EV, true>, sm);
                k_ypass<EV, true><<<nb, yz_threads<EV, true>(), sm, L.s>>>(p, d_tw, Mt, nx, A, g.nxs, g.nkys, u,
                                                             B, C, BlockDest{});
            }
            FSE_LAUNCH_CHECK();
            ++*L.launches;
        }
        {
            const int u = units_fit(h, 1, 0, yz_threads_host(h.eng, true));
            FftPlan p = h.dev;
            set_buf(p, h, u, d_tw);
            const size_t sm = smem_bytes(h, u);
            const int64_t npairs = static_cast<int64_t>(ncomp) * nx * Jp;
            const unsigned nb = static_cast<unsigned>((npairs + u - 1) / u);
            if constexpr (EV > 0 && !Eng<EV>::BLUE && !Eng<EV>::THREE) {
                if (v2_mask_for<EV>() & 16) {
                    allow_smem(k_zinv2<EV>, sm);
                    k_zinv2<EV><<<nb, yz_threads<EV, true>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, u, B, W);
                } else {
                    allow_smem(k_zinv<EV>, sm);
                    k_zinv<EV><<<nb, yz_threads<EV, true>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, u, B, W);
                }
            } else {
                allow_smem(k_zinv<EV>, sm);
                k_zinv<EV><<<nb, yz_threads<EV, true>(), sm, L.s>>>(p, d_tw, Mt, nx, ncomp, u, B, W);
            }
            FSE_LAUNCH_CHECK();
            ++*L.launches;
        }
    });
}

}  // namespace fsecu
