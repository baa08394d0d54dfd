// fft_reg.cuh -- register-resident FFT building blocks for k_fft.cu.
//
// rfft<N>(v): in-place FFT of N complex values held in registers, decimation
// in time with a compile-time radix split N = P x M (radices 8, 4, 2, 3, 5,
// 7, 11, 13), so every index is a constant after unrolling.  Twiddles
// W_N^t come from a shared-memory table at a compile-time offset
// (tw_off<N>()), loaded as broadcasts.
//
// fft_cols_2l<D1, D2>: the column FFT of length D = D1 D2 ("four-step"):
//   pass 1: thread (col, n2) holds x[n1 D2 + n2], n1 < D1, does FFT_D1,
//           multiplies by W_D^{n2 k1} and writes [k1][n2] to shared memory;
//   pass 2: thread (col, k1) reads the D2 values, does FFT_D2 and writes
//           X[k1 + D1 k2].
// Two shared-memory round trips per element instead of one per radix stage.
#pragma once

#include "fse_internal.cuh"

namespace fsecu {
namespace freg {

__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cis(double2 a, int s) {
    return s > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// ---- small DFTs (sign s: -1 forward, +1 inverse)
template <int P>
struct Dft;
template <>
struct Dft<2> {
    __device__ __forceinline__ static void run(double2* v, int) {
        const double2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};
template <>
struct Dft<3> {
    __device__ __forceinline__ static void run(double2* v, int s) {
        const double h = 0.86602540378443864676372317075293618;
        const double2 t1 = cadd(v[1], v[2]);
        const double2 t2 = make_double2(fma(-0.5, t1.x, v[0].x), fma(-0.5, t1.y, v[0].y));
        const double2 d = csub(v[1], v[2]);
        const double2 t3 = cis(make_double2(h * d.x, h * d.y), s);
        v[0] = cadd(v[0], t1);
        v[1] = cadd(t2, t3);
        v[2] = csub(t2, t3);
    }
};
template <>
struct Dft<4> {
    __device__ __forceinline__ static void run(double2* v, int s) {
        const double2 s0 = cadd(v[0], v[2]), d0 = csub(v[0], v[2]);
        const double2 s1 = cadd(v[1], v[3]), d1 = cis(csub(v[1], v[3]), s);
        v[0] = cadd(s0, s1);
        v[2] = csub(s0, s1);
        v[1] = cadd(d0, d1);
        v[3] = csub(d0, d1);
    }
};
template <>
struct Dft<8> {
    __device__ __forceinline__ static void run(double2* v, int s) {
        double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4>::run(e, s);
        Dft<4>::run(o, s);
        const double r = 0.70710678118654752440084436210484904;
        const double2 o1 = o[1], o3 = o[3];
        o[1] = make_double2(r * (o1.x - s * o1.y), r * (o1.y + s * o1.x));
        o[2] = cis(o[2], s);
        o[3] = make_double2(r * (-o3.x - s * o3.y), r * (-o3.y + s * o3.x));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = cadd(e[q], o[q]);
            v[q + 4] = csub(e[q], o[q]);
        }
    }
};

// cos / sin (2 pi t / p) for p = 5, 7, 11, 13, filled by the host
__constant__ double c_rcos[4][14];
__constant__ double c_rsin[4][14];

template <int P, int T>
struct DftOdd {
    __device__ __forceinline__ static void run(double2* v, int sgn) {
        constexpr int H = (P - 1) / 2;
        double2 sr[H], dr[H];
#pragma unroll
        for (int r = 1; r <= H; ++r) {
            sr[r - 1] = cadd(v[r], v[P - r]);
            dr[r - 1] = csub(v[r], v[P - r]);
        }
        const double2 v0 = v[0];
        double2 y0 = v0;
#pragma unroll
        for (int r = 0; r < H; ++r) y0 = cadd(y0, sr[r]);
#pragma unroll
        for (int q = 1; q <= H; ++q) {
            double2 A = v0, B = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 1; r <= H; ++r) {
                const int t = (r * q) % P;
                const double c = c_rcos[T][t], sn = c_rsin[T][t];
                A.x = fma(sr[r - 1].x, c, A.x);
                A.y = fma(sr[r - 1].y, c, A.y);
                B.x = fma(dr[r - 1].x, sn, B.x);
                B.y = fma(dr[r - 1].y, sn, B.y);
            }
            const double2 iB = cis(B, sgn);
            v[q] = cadd(A, iB);
            v[P - q] = csub(A, iB);
        }
        v[0] = y0;
    }
};
template <>
struct Dft<5> : DftOdd<5, 0> {};
template <>
struct Dft<7> : DftOdd<7, 1> {};
template <>
struct Dft<11> : DftOdd<11, 2> {};
template <>
struct Dft<13> : DftOdd<13, 3> {};

// ---- compile-time radix choice and twiddle-table layout
__host__ __device__ constexpr bool is_base(int n) {
    return n == 2 || n == 3 || n == 4 || n == 5 || n == 7 || n == 8 || n == 11 || n == 13;
}
__host__ __device__ constexpr int first_radix(int n) {
    return (n % 8 == 0) ? 8 : (n % 4 == 0) ? 4 : (n % 2 == 0) ? 2 : (n % 3 == 0) ? 3
         : (n % 5 == 0) ? 5 : (n % 7 == 0) ? 7 : (n % 11 == 0) ? 11 : 13;
}
// composite register sizes that own a twiddle table, in table order
// (only the composite sizes the engines in k_fft.cu use; twid<> static_asserts)
constexpr int kRegSizes[] = {10, 12, 15, 20, 22, 24, 26, 30, 32, 40};
constexpr int kNumRegSizes = sizeof(kRegSizes) / sizeof(int);
__host__ __device__ constexpr int tw_off_of(int n) {
    int off = 0;
    for (int i = 0; i < kNumRegSizes; ++i) {
        if (kRegSizes[i] == n) return off;
        off += kRegSizes[i];
    }
    return -1;
}
__host__ __device__ constexpr int tw_total() {
    int off = 0;
    for (int i = 0; i < kNumRegSizes; ++i) off += kRegSizes[i];
    return off;
}

template <int N>
__device__ __forceinline__ double2 twid(int t, int sgn, const double2* tab) {
    constexpr int off = tw_off_of(N);
    static_assert(off >= 0, "register FFT size without a twiddle table");
    double2 w = tab[off + t];
    if (sgn > 0) w.y = -w.y;
    return w;
}

template <int N>
__device__ __forceinline__ void rfft(double2* v, int sgn, const double2* tab) {
    if constexpr (is_base(N)) {
        Dft<N>::run(v, sgn);
    } else {
        constexpr int P = first_radix(N), M = N / P;
        double2 sub[P][M];
#pragma unroll
        for (int r = 0; r < P; ++r)
#pragma unroll
            for (int j = 0; j < M; ++j) sub[r][j] = v[j * P + r];
#pragma unroll
        for (int r = 0; r < P; ++r) rfft<M>(sub[r], sgn, tab);
#pragma unroll
        for (int k = 0; k < M; ++k) {
            double2 y[P];
#pragma unroll
            for (int r = 0; r < P; ++r) {
                y[r] = sub[r][k];
                if ((r * k) % N != 0) y[r] = cmul(y[r], twid<N>((r * k) % N, sgn, tab));
            }
            Dft<P>::run(y, sgn);
#pragma unroll
            for (int q = 0; q < P; ++q) v[k + M * q] = y[q];
        }
    }
}

// Shared-memory column layout of the register engines: one pad element after
// every D2 elements and a column stride >= D + D1 + 1 that is 3 mod 8 (in
// 16-byte elements; 8 of them fill the 32 banks).  Lanes that walk columns
// (stride 3 mod 8) and elements (stride 1) then hit distinct bank groups in
// the passes and in the x-pass multiplier, whose lanes walk (kz column, kx)
// three columns at a time (a stride of 1 mod 8 put three lanes on one bank
// group there: 3x shared-memory wavefronts).
__host__ __device__ constexpr int col_stride(int D1, int D2) {
    return D1 * D2 + D1 + 1 + ((3 - (D1 * D2 + D1 + 1) % 8) + 8) % 8;
}
template <int D1, int D2>
__device__ __forceinline__ int ridx(int c, int n) {
    return c * col_stride(D1, D2) + n + n / D2;
}

// Column FFT of length D1*D2 on `ncol` columns stored at buf[ridx(c, n)].
// Requires ncol*D2 <= blockDim.x and ncol*D1 <= blockDim.x (one item per thread).
// twD: W_D^t, t < D; tab: small-size twiddles (tw_off_of layout).
template <int D1, int D2>
__device__ __forceinline__ void fft_cols_2l(double2* buf, int ncol, int sgn,
                                            const double2* twD, const double2* tab) {
    constexpr int D = D1 * D2;
    const int tid = threadIdx.x;
    // pass 1: item (c, n2)
    double2 v[D1];
    const bool a1 = tid < ncol * D2;
    int c1 = 0, n2 = 0;
    if (a1) {
        c1 = tid / D2;
        n2 = tid - c1 * D2;
        // ridx(c, n1 D2 + n2) = ridx(c, n2) + n1 (D2 + 1) for n2 < D2
        const double2* src = buf + ridx<D1, D2>(c1, n2);
#pragma unroll
        for (int n1 = 0; n1 < D1; ++n1) v[n1] = src[n1 * (D2 + 1)];
        rfft<D1>(v, sgn, tab);
        int t = 0;  // n2 * k1 mod D
#pragma unroll
        for (int k1 = 0; k1 < D1; ++k1) {
            if (k1 > 0) {
                double2 w = twD[t];
                if (sgn > 0) w.y = -w.y;
                v[k1] = cmul(v[k1], w);
            }
            t += n2;
            if (t >= D) t -= D;
        }
    }
    __syncthreads();
    if (a1) {
        double2* dst = buf + ridx<D1, D2>(c1, n2);
#pragma unroll
        for (int k1 = 0; k1 < D1; ++k1) dst[k1 * (D2 + 1)] = v[k1];
    }
    __syncthreads();
    // pass 2: item (c, k1)
    double2 u[D2];
    const bool a2 = tid < ncol * D1;
    int c2 = 0, k1 = 0;
    if (a2) {
        c2 = tid / D1;
        k1 = tid - c2 * D1;
        // ridx(c, k1 D2 + j) = ridx(c, 0) + k1 (D2 + 1) + j for j < D2
        const double2* src = buf + ridx<D1, D2>(c2, 0) + k1 * (D2 + 1);
#pragma unroll
        for (int j = 0; j < D2; ++j) u[j] = src[j];
        rfft<D2>(u, sgn, tab);
    }
    __syncthreads();
    if (a2) {
#pragma unroll
        for (int k2 = 0; k2 < D2; ++k2) buf[ridx<D1, D2>(c2, k1 + D1 * k2)] = u[k2];
    }
    __syncthreads();
}

// ---- two-level passes with caller-supplied global I/O (the "v2" kernels in
// k_fft.cu): pass 1 loads straight from global memory into registers and
// pass 2 stores straight from registers, so the only shared-memory round trip
// of a plain transform is the transpose between the passes.
//
// Item mapping: CF (column-fastest) -- consecutive threads walk the columns,
// for passes whose columns are adjacent in memory (y, x); otherwise
// consecutive threads walk n2 (pass 1) / k1 (pass 2), for rows (z).

template <int D1, int D2, bool CF>
__device__ __forceinline__ bool item1(int ncol, int& c, int& n2) {
    const int tid = threadIdx.x;
    if (tid >= ncol * D2) return false;
    if (CF) {
        n2 = tid / ncol;
        c = tid - n2 * ncol;
    } else {
        c = tid / D2;
        n2 = tid - c * D2;
    }
    return true;
}

template <int D1, int D2, bool CF>
__device__ __forceinline__ bool item2(int ncol, int& c, int& k1) {
    const int tid = threadIdx.x;
    if (tid >= ncol * D1) return false;
    if (CF) {
        k1 = tid / ncol;
        c = tid - k1 * ncol;
    } else {
        c = tid / D1;
        k1 = tid - c * D1;
    }
    return true;
}

// pass 1: v[n1] = load(c, n1 D2 + n2) for n1 < NZ1 (rows n1 >= NZ1 are known
// zeros: zero-padded inputs), FFT_D1, twiddle W_D^{n2 k1}, store the transpose
// into buf[ridx(c, k1 D2 + n2)].  No barriers inside.
template <int D1, int D2, bool CF, int NZ1, class LOAD>
__device__ __forceinline__ void pass1(double2* buf, int ncol, int sgn, const double2* twD,
                                      const double2* tab, LOAD load) {
    constexpr int D = D1 * D2;
    int c, n2;
    if (!item1<D1, D2, CF>(ncol, c, n2)) return;
    double2 v[D1];
#pragma unroll
    for (int n1 = 0; n1 < D1; ++n1) v[n1] = n1 < NZ1 ? load(c, n1 * D2 + n2) : make_double2(0.0, 0.0);
    rfft<D1>(v, sgn, tab);
    int t = 0;  // n2 * k1 mod D
#pragma unroll
    for (int k1 = 0; k1 < D1; ++k1) {
        if (k1 > 0) {
            double2 w = twD[t];
            if (sgn > 0) w.y = -w.y;
            v[k1] = cmul(v[k1], w);
        }
        t += n2;
        if (t >= D) t -= D;
    }
    double2* dst = buf + ridx<D1, D2>(c, n2);  // + k1 (D2 + 1): ridx(c, k1 D2 + n2)
#pragma unroll
    for (int k1 = 0; k1 < D1; ++k1) dst[k1 * (D2 + 1)] = v[k1];
}

// pass 1 as above, with mid() called by EVERY thread of the CTA between the
// loads and the first use of the twiddle tables (e.g. the wait for their
// asynchronous staging), so the loads' latency overlaps the staging's
template <int D1, int D2, bool CF, int NZ1, class LOAD, class MID>
__device__ __forceinline__ void pass1_mid(double2* buf, int ncol, int sgn, const double2* twD,
                                          const double2* tab, LOAD load, MID mid) {
    constexpr int D = D1 * D2;
    int c = 0, n2 = 0;
    const bool act = item1<D1, D2, CF>(ncol, c, n2);
    double2 v[D1];
    if (act) {
#pragma unroll
        for (int n1 = 0; n1 < D1; ++n1)
            v[n1] = n1 < NZ1 ? load(c, n1 * D2 + n2) : make_double2(0.0, 0.0);
    }
    mid();
    if (!act) return;
    rfft<D1>(v, sgn, tab);
    int t = 0;  // n2 * k1 mod D
#pragma unroll
    for (int k1 = 0; k1 < D1; ++k1) {
        if (k1 > 0) {
            double2 w = twD[t];
            if (sgn > 0) w.y = -w.y;
            v[k1] = cmul(v[k1], w);
        }
        t += n2;
        if (t >= D) t -= D;
    }
    double2* dst = buf + ridx<D1, D2>(c, n2);
#pragma unroll
    for (int k1 = 0; k1 < D1; ++k1) dst[k1 * (D2 + 1)] = v[k1];
}

// pass 1 in place on buf (loads ridx(c, n1 D2 + n2) of its own item, FFT_D1,
// twiddle, stores the transpose over them; no barriers inside)
template <int D1, int D2, bool CF>
__device__ __forceinline__ void pass1_inplace(double2* buf, int ncol, int sgn, const double2* twD,
                                              const double2* tab) {
    constexpr int D = D1 * D2;
    int c, n2;
    if (!item1<D1, D2, CF>(ncol, c, n2)) return;
    double2* col = buf + ridx<D1, D2>(c, n2);
    double2 v[D1];
#pragma unroll
    for (int n1 = 0; n1 < D1; ++n1) v[n1] = col[n1 * (D2 + 1)];
    rfft<D1>(v, sgn, tab);
    int t = 0;  // n2 * k1 mod D
#pragma unroll
    for (int k1 = 0; k1 < D1; ++k1) {
        if (k1 > 0) {
            double2 w = twD[t];
            if (sgn > 0) w.y = -w.y;
            v[k1] = cmul(v[k1], w);
        }
        t += n2;
        if (t >= D) t -= D;
    }
#pragma unroll
    for (int k1 = 0; k1 < D1; ++k1) col[k1 * (D2 + 1)] = v[k1];
}

// pass 2 (after a barrier): u[j] = buf[ridx(c, k1 D2 + j)], FFT_D2, then
// store(c, k1 + D1 k2, u[k2]) for k2 < NOUT2 (outputs k2 >= NOUT2 are not
// needed: pruned windows).  No barriers inside.
template <int D1, int D2, bool CF, int NOUT2, class STORE>
__device__ __forceinline__ void pass2(const double2* buf, int ncol, int sgn, const double2* tab,
                                      STORE store) {
    int c, k1;
    if (!item2<D1, D2, CF>(ncol, c, k1)) return;
    double2 u[D2];
    const double2* src = buf + ridx<D1, D2>(c, 0) + k1 * (D2 + 1);  // ridx(c, k1 D2 + j) - j
#pragma unroll
    for (int j = 0; j < D2; ++j) u[j] = src[j];
    rfft<D2>(u, sgn, tab);
#pragma unroll
    for (int k2 = 0; k2 < NOUT2; ++k2) store(c, k1 + D1 * k2, u[k2]);
}

// pass 2 back into buf in natural order (for a following shared-memory stage):
// loads, barrier, stores (every thread of the CTA must call it)
template <int D1, int D2, bool CF>
__device__ __forceinline__ void pass2_smem(double2* buf, int ncol, int sgn, const double2* tab) {
    int c = 0, k1 = 0;
    const bool act = item2<D1, D2, CF>(ncol, c, k1);
    double2 u[D2];
    if (act) {
        const double2* src = buf + ridx<D1, D2>(c, 0) + k1 * (D2 + 1);
#pragma unroll
        for (int j = 0; j < D2; ++j) u[j] = src[j];
        rfft<D2>(u, sgn, tab);
    }
    __syncthreads();
    if (act) {
#pragma unroll
        for (int k2 = 0; k2 < D2; ++k2) buf[ridx<D1, D2>(c, k1 + D1 * k2)] = u[k2];
    }
}

// ---- three-level column FFT, D = D1 D2 D3 (small register DFTs, more
// resident warps than a two-level split of the same D; the opt-in engine 8,
// 1200 = 10 x 12 x 10, measured slower than the two-level engine: k_fft.cu
// engine_for).  Layout: element n of column c
// at c S3 + n + n / D3 (one pad per D3 elements), S3 = col_stride3.  With
// n = n1 D2 D3 + n2 D3 + n3 and k = k1 + D1 k2 + D1 D2 k3:
//   pass A, item (c, m = n2 D3 + n3): FFT_D1 over n1, times W_D^{k1 m};
//   pass B, item (c, k1, n3): FFT_D2 over n2, times W_{D2 D3}^{k2 n3};
//   pass C, item (c, k1, k2): FFT_D3 over n3, stored at the natural k.
// Passes A and B work in place on item-local positions; pass C reads all of
// a column group before any store (barrier), `grp` columns at a time.
// WD: W_D^t (t < D, global memory); W23: W_{D2 D3}^t (t < D2 D3); tab: the
// small register tables.  Every thread of the CTA must call it.
__host__ __device__ constexpr int col_stride3(int D, int D3) {
    return D + D / D3 + 1 + ((3 - (D + D / D3 + 1) % 8) + 8) % 8;
}
template <int D1, int D2, int D3>
__device__ __forceinline__ int idx3(int c, int n) {
    return c * col_stride3(D1 * D2 * D3, D3) + n + n / D3;
}
__device__ __forceinline__ double2 twc(const double2* t, int e, int sgn) {
    double2 w = t[e];
    if (sgn > 0) w.y = -w.y;
    return w;
}
template <int D1, int D2, int D3>
__device__ __forceinline__ void fft_cols_3l(double2* buf, int ncol, int sgn,
                                            const double2* __restrict__ WD, const double2* W23,
                                            const double2* tab) {
    constexpr int D = D1 * D2 * D3, M23 = D2 * D3;
    const int T = blockDim.x;
    // pass A
    for (int it = threadIdx.x; it < ncol * M23; it += T) {
        const int c = it / M23, m = it - c * M23;
        double2 v[D1];
#pragma unroll
        for (int n1 = 0; n1 < D1; ++n1) v[n1] = buf[idx3<D1, D2, D3>(c, n1 * M23 + m)];
        rfft<D1>(v, sgn, tab);
        int t = 0;
#pragma unroll
        for (int k1 = 0; k1 < D1; ++k1) {
            if (k1 > 0) v[k1] = cmul(v[k1], twc(WD, t, sgn));
            t += m;
            if (t >= D) t -= D;
        }
#pragma unroll
        for (int k1 = 0; k1 < D1; ++k1) buf[idx3<D1, D2, D3>(c, k1 * M23 + m)] = v[k1];
    }
    __syncthreads();
    // pass B
    for (int it = threadIdx.x; it < ncol * D1 * D3; it += T) {
        const int c = it / (D1 * D3), r = it - c * (D1 * D3);
        const int k1 = r / D3, n3 = r - k1 * D3;
        double2 v[D2];
#pragma unroll
        for (int n2 = 0; n2 < D2; ++n2) v[n2] = buf[idx3<D1, D2, D3>(c, k1 * M23 + n2 * D3 + n3)];
        rfft<D2>(v, sgn, tab);
#pragma unroll
        for (int k2 = 1; k2 < D2; ++k2) v[k2] = cmul(v[k2], twc(W23, k2 * n3, sgn));
#pragma unroll
        for (int k2 = 0; k2 < D2; ++k2) buf[idx3<D1, D2, D3>(c, k1 * M23 + k2 * D3 + n3)] = v[k2];
    }
    __syncthreads();
    // pass C, `grp` columns per round: load + FFT, barrier, natural-order store
    const int grp = T / (D1 * D2) > 0 ? T / (D1 * D2) : 1;
    for (int c0 = 0; c0 < ncol; c0 += grp) {
        const int it = threadIdx.x;
        const int c = c0 + it / (D1 * D2), r = it - (it / (D1 * D2)) * (D1 * D2);
        const bool act = it < grp * D1 * D2 && c < ncol;
        const int k1 = r % D1, k2 = r / D1;
        double2 v[D3];
        if (act) {
#pragma unroll
            for (int n3 = 0; n3 < D3; ++n3) v[n3] = buf[idx3<D1, D2, D3>(c, k1 * M23 + k2 * D3 + n3)];
            rfft<D3>(v, sgn, tab);
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int k3 = 0; k3 < D3; ++k3) buf[idx3<D1, D2, D3>(c, k1 + D1 * k2 + D1 * D2 * k3)] = v[k3];
        }
        __syncthreads();
    }
}

}  // namespace freg
}  // namespace fsecu
