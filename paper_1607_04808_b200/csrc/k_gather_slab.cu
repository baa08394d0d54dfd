// k_gather_slab.cu -- trapezoidal quadrature back to the targets
// (ewald.cpp:349-391) on the FP64 tensor cores (DMMA m8n8k4).
//
// Work item = one z-half of a coarse tile: the <= 32 targets (more => more
// items) whose support start lies in an 8 x 8 x 8 block of starts
// (x0, y0, z0) -- a contiguous key range, since the fine key puts the z-half
// first.  Every support lies in the union box
// [x0, x0+P+7) x [y0, y0+P+7) x [z0, z0+P+7).  The CTA streams the box
// through shared memory one x-plane ("slab") at a time with cp.async double
// buffering.  A slab is the matrix
//     A[(c, y)][z] = g_c[x][y0 + y][z0 + z]        (3 (P+7) rows, 4 KS cols)
// and the z contraction of every row against every target is the GEMM
//     S = A B,   B[z][t] = wz_t[z0 + z]            (zero outside the support)
// done with mma.sync.m8n8k4.f64; each A fragment is one LDS and feeds NT
// MMAs.  wx_t[x] is folded into the B fragments of slab x, so the MMA
// accumulators carry
//     C[(c, y)][t] = sum_x wx_t[x] sum_z g_c[x][y][z] wz_t[z]
// across all slabs, and the item ends with the y contraction through shared
// memory: u_t[c] = h^3 sum_y wy_t[y] C[(c, y)][t].  No atomics; fixed order.
//
// The union box costs (P+7)^2 (4 KS) / P^3 ~ 2.2x the exact FMA count at
// P = 24 and target padding to 8 another ~1.2x, but at 256 FMAs per MMA
// instruction the tensor pipe runs near its (FP64) peak instead of the
// issue- and latency-bound per-lane DFMA loops.  P + 7 <= 32 (P <= 25);
// larger supports use k_gather.cu.
//
// Roofline: FP64 tensor (DMMA) -- same ~37 TFLOP/s peak as DFMA on B200.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

#ifndef FSE_GATHER_SW
#define FSE_GATHER_SW 4
#endif
constexpr int SW = FSE_GATHER_SW;  // warps per CTA
constexpr int MAXT = 32;   // targets per item
constexpr int RS = 34;     // slab row stride (doubles): 32 + 2 keeps A-fragment loads at 2 wavefronts
#ifndef FSE_GATHER_NST
#define FSE_GATHER_NST 2
#endif
constexpr int NST = FSE_GATHER_NST;  // slab buffers (cp.async pipeline depth)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16z(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp8z(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// stage x-plane x of the union box: rows r = c NY + yy, columns z < NZ
// (zero-filled up to 4 KS); pad rows >= 3 NY stay zero from the prologue
template <int KS>
__device__ __forceinline__ void stage_slab(const GridParams& g, const double* __restrict__ X,
                                           int x, int y0, int z0, int NY, int NZ, bool vec16,
                                           double* dst) {
    const double* src0 = X + static_cast<int64_t>(x - g.x_lo) * g.plane +
                         static_cast<int64_t>(y0) * g.rowp + z0;  // slab-local plane
    if (vec16) {
        constexpr int NCH = 2 * KS;  // 16-byte chunks per row
        const int total = 3 * NY * NCH;
        for (int idx = threadIdx.x; idx < total; idx += SW * 32) {
            const int r = idx / NCH, k = idx - r * NCH;
            const int c = (r >= NY) + (r >= 2 * NY);
            const int yy = r - c * NY;
            const double* src = src0 + c * g.comp + static_cast<int64_t>(yy) * g.rowp;
            const int zz = 2 * k;
            const int bytes = zz + 1 < NZ ? 16 : (zz < NZ ? 8 : 0);
            cp16z(dst + r * RS + zz, bytes ? src + zz : src0, bytes);
        }
    } else {
        constexpr int NCH = 4 * KS;
        const int total = 3 * NY * NCH;
        for (int idx = threadIdx.x; idx < total; idx += SW * 32) {
            const int r = idx / NCH, k = idx - r * NCH;
            const int c = (r >= NY) + (r >= 2 * NY);
            const int yy = r - c * NY;
            const double* src = src0 + c * g.comp + static_cast<int64_t>(yy) * g.rowp;
            cp8z(dst + r * RS + k, k < NZ ? src + k : src0, k < NZ ? 8 : 0);
        }
    }
}

// MT: m-tiles (8 rows) per warp; NT: n-tiles (8 targets); KS: k-steps (4 z).
// wx is folded into the B fragments per slab (bs = b0 wx_t[x]), so C
// accumulates sum_x sum_z directly across slabs: no per-slab epilogue and
// MT x NT independent accumulation chains per warp.
template <int MT, int NT, int KS>
__device__ void gather_item(const GridParams& g, const double* __restrict__ X, double* slab,
                            const double* b0s, const double* wxs, int x0, int y0, int z0, int NX,
                            int NY, int NZ, bool vec16, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows_pad = 8 * MT * SW;
    const int buf_elems = rows_pad * RS;
    double C[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) C[mt][nt][0] = C[mt][nt][1] = 0.0;
    const int rbase = 8 * MT * warp + (lane >> 2);
    const int tb = lane >> 2;  // B column (target within an n-tile) of this lane

    // planes of the union box inside this rank's slab (all of them on one GPU);
    // with several slabs every rank adds its planes' share of the sum
    const int xs0 = max(0, g.x_lo - x0), xs1 = min(NX, g.x_lo + g.nx - x0);
    // NST-stage cp.async pipeline: slab xs + NST - 1 is in flight while xs is used
#pragma unroll
    for (int st = 0; st < NST - 1; ++st) {
        if (xs0 + st < xs1)
            stage_slab<KS>(g, X, x0 + xs0 + st, y0, z0, NY, NZ, vec16,
                           slab + ((xs0 + st) % NST) * buf_elems);
        cp_commit();
    }
    for (int xs = xs0; xs < xs1; ++xs) {
        if (xs + NST - 1 < xs1)
            stage_slab<KS>(g, X, x0 + xs + NST - 1, y0, z0, NY, NZ, vec16,
                           slab + ((xs + NST - 1) % NST) * buf_elems);
        cp_commit();
        cp_wait<NST - 1>();
        __syncthreads();
        const double* A = slab + (xs % NST) * buf_elems + rbase * RS + (lane & 3);
        double wxt[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) wxt[nt] = wxs[xs * MAXT + 8 * nt + tb];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            double bs[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) bs[nt] = b0s[(ks * 4 + nt) * 32 + lane] * wxt[nt];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const double a = A[8 * mt * RS + 4 * ks];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(C[mt][nt][0], C[mt][nt][1], a, bs[nt]);
            }
        }
        __syncthreads();
    }
    // red[r][t] = C (rows r = (c, y), columns t)
    const int tc = 2 * (lane & 3);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const int r = rbase + 8 * mt;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            red[r * MAXT + 8 * nt + tc] = C[mt][nt][0];
            red[r * MAXT + 8 * nt + tc + 1] = C[mt][nt][1];
        }
    }
}

template <int MT, int KS>
__global__ void __launch_bounds__(SW * 32, NST == 2 ? 3 : 2) k_gather_mma(
    GridParams g, const int32_t* __restrict__ i0s, const double* __restrict__ w,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ items,
    const int32_t* __restrict__ nitems_dev, const double* __restrict__ X,
    const uint32_t* __restrict__ perm, double scale, double* __restrict__ u) {
    extern __shared__ __align__(16) double gsm[];
    __shared__ int4 tinfo[MAXT];
    if (static_cast<int>(blockIdx.x) >= *nitems_dev) return;  // CTA-uniform
    constexpr int ROWS = 8 * MT * SW;
    double* slab = gsm;                    // [2][ROWS][RS]
    double* wxs = slab + NST * ROWS * RS;  // [nx][MAXT]
    double* b0s = wxs + 32 * MAXT;         // [KS][4][32] B fragments (wz)
    const int e = items[2 * blockIdx.x], bi = items[2 * blockIdx.x + 1];
    const int c = e >> 1, h = e & 1;
    const int cz = c % g.ncz, cy = (c / g.ncz) % g.ncy, cx = c / (g.ncz * g.ncy);
    const int P = g.P, Mt = g.Mt;
    const int x0 = cx * 8, y0 = cy * 8, z0 = cz * 16 + 8 * h;
    const int first = tstart[8 * c + 4 * h] + MAXT * bi;
    const int n = min(MAXT, tstart[8 * c + 4 * h + 4] - first);
    const int NX = min(P + 7, Mt - x0), NY = min(P + 7, Mt - y0), NZ = min(P + 7, Mt - z0);
    const int tid = threadIdx.x;
    if (tid < MAXT) {
        int4 ti = make_int4(0, 0, 0, 0);
        if (tid < n) {
            const int q = first + tid;
            ti = make_int4(q, i0s[3 * q], i0s[3 * q + 1], i0s[3 * q + 2]);
        }
        tinfo[tid] = ti;
    }
    // pad rows of both slab buffers stay zero
    for (int idx = tid; idx < NST * ROWS * RS; idx += SW * 32) {
        const int r = (idx / RS) % ROWS;
        if (r >= 3 * NY) slab[idx] = 0.0;
    }
    __syncthreads();
    // x weights on the union box: wxs[x][t] (zero outside the support)
    for (int idx = tid; idx < 32 * MAXT; idx += SW * 32) {
        const int xx = idx / MAXT, t = idx % MAXT;
        const int4 ti = tinfo[t];
        const int px = x0 + xx - ti.y;
        wxs[idx] = (t < n && xx < NX && px >= 0 && px < P)
                       ? w[static_cast<int64_t>(ti.x) * 3 * P + px]
                       : 0.0;
    }
    // B fragments b0[ks][nt][lane] = wz_t[z0 + 4 ks + lane % 4 - iz_t], t = 8 nt + lane / 4
    for (int idx = tid; idx < KS * 4 * 32; idx += SW * 32) {
        const int l = idx & 31, nt = (idx >> 5) & 3, ks = idx >> 7;
        const int t = 8 * nt + (l >> 2), z = 4 * ks + (l & 3);
        const int4 ti = tinfo[t];
        const int pz = z0 + z - ti.w;
        b0s[idx] = (t < n && z < NZ && pz >= 0 && pz < P)
                       ? w[static_cast<int64_t>(ti.x) * 3 * P + 2 * P + pz]
                       : 0.0;
    }
    __syncthreads();
    const bool vec16 = (Mt % 2) == 0;
    double* red = slab;  // reused after the last slab (ROWS x MAXT <= 2 ROWS RS)
    const int nt = (n + 7) / 8;
    if (nt <= 1)
        gather_item<MT, 1, KS>(g, X, slab, b0s, wxs, x0, y0, z0, NX, NY, NZ, vec16, red);
    else if (nt == 2)
        gather_item<MT, 2, KS>(g, X, slab, b0s, wxs, x0, y0, z0, NX, NY, NZ, vec16, red);
    else if (nt == 3)
        gather_item<MT, 3, KS>(g, X, slab, b0s, wxs, x0, y0, z0, NX, NY, NZ, vec16, red);
    else
        gather_item<MT, 4, KS>(g, X, slab, b0s, wxs, x0, y0, z0, NX, NY, NZ, vec16, red);
    __syncthreads();
    // u_t[c] = h^3 sum_y wy_t[y] red[(c, y)][t]
    if (tid < 3 * MAXT) {
        const int t = tid % MAXT, cc = tid / MAXT;
        if (t < n) {
            const int4 ti = tinfo[t];
            const double* wy = w + static_cast<int64_t>(ti.x) * 3 * P + P;
            const int yo = ti.z - y0;  // support rows yy = yo .. yo + P - 1
            double s = 0.0;
            for (int p = 0; p < P; ++p) s = fma(wy[p], red[(cc * NY + yo + p) * MAXT + t], s);
            u[3 * static_cast<int64_t>(perm[first + t]) + cc] = scale * s;
        }
    }
}

// ---------------------------------------------------------------- TMA variant
// Same item, same MMA loop; the slab (all 3 components x P+7 rows y x 34 z)
// arrives as ONE cp.async.bulk.tensor box per x-plane, issued by one thread
// and completed on an mbarrier, instead of ~1500 16-byte cp.async per plane
// issued by all 128 threads (the staging index math was ~2x the MMA loop's
// instructions).  The box's 34-double rows are exactly the RS = 34 padded
// layout (two extra z columns are fetched and never read), y rows past the
// grid edge and z past M~ arrive as zeros (TMA out-of-bounds fill), so the
// rows are (c, y) with a fixed pitch of P+7 = NYB per component.  Needs an
// even M~ (16-byte row strides) and KS = 8.

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int z, int y, int x, int c) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(z), "r"(y), "r"(x), "r"(c)
        : "memory");
}

// MMAs of one slab for the n-tiles [LO, HI] (compile-time, so the
// accumulators stay in registers and no MMA is predicated)
template <int LO, int HI, int MT, int NT, int KS>
__device__ __forceinline__ void slab_mmas(double (&C)[MT][NT][2], const double* A,
                                          const double* b0s, const double (&wxt)[NT], int lane) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        double bs[NT];
#pragma unroll
        for (int nt = LO; nt <= HI; ++nt) bs[nt] = b0s[(ks * 4 + nt) * 32 + lane] * wxt[nt];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const double a = A[8 * mt * RS + 4 * ks];
#pragma unroll
            for (int nt = LO; nt <= HI; ++nt) dmma(C[mt][nt][0], C[mt][nt][1], a, bs[nt]);
        }
    }
}

// dispatch the run-time n-tile range [lo, hi] (0 <= lo <= hi < NT) to slab_mmas
template <int LO, int HI, int MT, int NT, int KS>
__device__ __forceinline__ void slab_mmas_rt(int lo, int hi, double (&C)[MT][NT][2],
                                             const double* A, const double* b0s,
                                             const double (&wxt)[NT], int lane) {
    if constexpr (LO < NT) {
        if (lo == LO) {
            if constexpr (HI < NT) {
                if (hi == HI) {
                    slab_mmas<LO, HI, MT, NT, KS>(C, A, b0s, wxt, lane);
                    return;
                }
                slab_mmas_rt<LO, HI + 1, MT, NT, KS>(lo, hi, C, A, b0s, wxt, lane);
            }
            return;
        }
        slab_mmas_rt<LO + 1, LO + 1, MT, NT, KS>(lo, hi, C, A, b0s, wxt, lane);
    }
}

// xr[nt] = (first, last + P) plane range of n-tile nt's x supports (targets
// sorted by x start, so the tiles active on one plane are a contiguous range
// [lo, hi]); planes outside every tile's range are not loaded at all
template <int MT, int NT, int KS>
__device__ void gather_item_tma(const GridParams& g, const CUtensorMap* map, double* slab,
                                uint64_t* bars, const double* b0s, const double* wxs, int x0,
                                int y0, int z0, int NX, const int2* xr, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows_pad = 8 * MT * SW;
    const int buf_elems = rows_pad * RS;
    const unsigned bytes = static_cast<unsigned>(sizeof(double)) * RS * (g.P + 7) * 3;
    double C[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) C[mt][nt][0] = C[mt][nt][1] = 0.0;
    const int rbase = 8 * MT * warp + (lane >> 2);
    const int tb = lane >> 2;
    int xlo[NT], xhi[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int2 r = xr[nt];
        xlo[nt] = r.x;
        xhi[nt] = r.y;
    }
    const int xs0 = max(max(0, g.x_lo - x0), xlo[0]);
    const int xs1 = min(min(NX, g.x_lo + g.nx - x0), xhi[NT - 1]);
    auto issue = [&](int xs) {  // one thread: slab xs -> buffer (xs - xs0) & 1
        const int b = (xs - xs0) & 1;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(bars + b, bytes);
        tma_load_4d(slab + b * buf_elems, map, bars + b, z0, y0, x0 + xs - g.x_lo, 0);
    };
    if (threadIdx.x == 0 && xs0 < xs1) issue(xs0);
    for (int xs = xs0; xs < xs1; ++xs) {
        const int i = xs - xs0;
        if (threadIdx.x == 0 && xs + 1 < xs1) issue(xs + 1);
        // n-tiles whose supports contain plane xs (warp-uniform)
        int lo = 0, hi = NT - 1;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            if (xhi[nt] <= xs) lo = nt + 1;
            if (xlo[NT - 1 - nt] > xs) hi = NT - 2 - nt;
        }
        mbar_wait(bars + (i & 1), (i >> 1) & 1);
        const double* A = slab + (i & 1) * buf_elems + rbase * RS + (lane & 3);
        double wxt[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) wxt[nt] = wxs[xs * MAXT + 8 * nt + tb];
        if (lo <= hi) slab_mmas_rt<0, 0, MT, NT, KS>(lo, hi, C, A, b0s, wxt, lane);
        __syncthreads();  // everyone is done with this buffer before it is refilled
    }
    const int tc = 2 * (lane & 3);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const int r = rbase + 8 * mt;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            red[r * MAXT + 8 * nt + tc] = C[mt][nt][0];
            red[r * MAXT + 8 * nt + tc + 1] = C[mt][nt][1];
        }
    }
}

template <int MT, int KS>
__global__ void __launch_bounds__(SW * 32, 3) k_gather_tma(
    const __grid_constant__ CUtensorMap map, GridParams g, const int32_t* __restrict__ i0s,
    const double* __restrict__ w, const int32_t* __restrict__ tstart,
    const int32_t* __restrict__ items, const int32_t* __restrict__ nitems_dev,
    const uint32_t* __restrict__ perm, double scale, double* __restrict__ u) {
    extern __shared__ __align__(128) double gsm[];
    if (static_cast<int>(blockIdx.x) >= *nitems_dev) return;  // CTA-uniform
    constexpr int ROWS = 8 * MT * SW;
    double* slab = gsm;                    // [2][ROWS][RS], 128-byte aligned buffers
    double* wxs = slab + 2 * ROWS * RS;    // [nx][MAXT]
    double* b0s = wxs + 32 * MAXT;         // [KS][4][32] B fragments (wz)
    int4* tinfo = reinterpret_cast<int4*>(b0s + KS * 4 * 32);
    uint64_t* bars = reinterpret_cast<uint64_t*>(tinfo + MAXT);
    int2* xr = reinterpret_cast<int2*>(bars + 2);  // per n-tile plane range
    const int e = items[2 * blockIdx.x], bi = items[2 * blockIdx.x + 1];
    const int c = e >> 1, h = e & 1;
    const int cz = c % g.ncz, cy = (c / g.ncz) % g.ncy, cx = c / (g.ncz * g.ncy);
    const int P = g.P, Mt = g.Mt, NYB = P + 7;
    const int x0 = cx * 8, y0 = cy * 8, z0 = cz * 16 + 8 * h;
    const int first = tstart[8 * c + 4 * h] + MAXT * bi;
    const int n = min(MAXT, tstart[8 * c + 4 * h + 4] - first);
    const int NX = min(P + 7, Mt - x0), NZ = min(P + 7, Mt - z0);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (tid < MAXT) {
        // the item's targets in x-start order (stable counting sort over the
        // 8 starts of the block, one ballot per start), so that each n-tile of
        // 8 targets spans few x starts and skips the planes outside its supports
        int4 ti = make_int4(0, 0, 0, 0);
        int key = 8;  // idle slots sort last
        if (tid < n) {
            const int q = first + tid;
            ti = make_int4(q, i0s[3 * q], i0s[3 * q + 1], i0s[3 * q + 2]);
            key = ti.y - x0;
        }
        int pos = 0, base = 0;
#pragma unroll
        for (int v = 0; v <= 8; ++v) {
            const unsigned bv = __ballot_sync(0xffffffffu, key == v);
            if (key == v) pos = base + __popc(bv & ((1u << tid) - 1u));
            base += __popc(bv);
        }
        tinfo[pos] = ti;
        __syncwarp();
        // plane range [first start, last start + P) of n-tile tid (slab index)
        if (tid < 4) {
            const int t0 = 8 * tid, t1 = min(8 * tid + 7, n - 1);
            xr[tid] = t0 < n ? make_int2(tinfo[t0].y - x0, tinfo[t1].y - x0 + P)
                             : make_int2(0, 0);
        }
    }
    // pad rows (>= 3 NYB) of both buffers stay zero; the boxes never write them
    for (int idx = tid; idx < 2 * ROWS * RS; idx += SW * 32) {
        const int r = (idx / RS) % ROWS;
        if (r >= 3 * NYB) slab[idx] = 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < 32 * MAXT; idx += SW * 32) {
        const int xx = idx / MAXT, t = idx % MAXT;
        const int4 ti = tinfo[t];
        const int px = x0 + xx - ti.y;
        wxs[idx] = (t < n && xx < NX && px >= 0 && px < P)
                       ? w[static_cast<int64_t>(ti.x) * 3 * P + px]
                       : 0.0;
    }
    for (int idx = tid; idx < KS * 4 * 32; idx += SW * 32) {
        const int l = idx & 31, nt = (idx >> 5) & 3, ks = idx >> 7;
        const int t = 8 * nt + (l >> 2), z = 4 * ks + (l & 3);
        const int4 ti = tinfo[t];
        const int pz = z0 + z - ti.w;
        b0s[idx] = (t < n && z < NZ && pz >= 0 && pz < P)
                       ? w[static_cast<int64_t>(ti.x) * 3 * P + 2 * P + pz]
                       : 0.0;
    }
    __syncthreads();
    double* red = slab;  // reused after the last slab (ROWS x MAXT <= 2 ROWS RS)
    const int nt = (n + 7) / 8;
    if (nt <= 1)
        gather_item_tma<MT, 1, KS>(g, &map, slab, bars, b0s, wxs, x0, y0, z0, NX, xr, red);
    else if (nt == 2)
        gather_item_tma<MT, 2, KS>(g, &map, slab, bars, b0s, wxs, x0, y0, z0, NX, xr, red);
    else if (nt == 3)
        gather_item_tma<MT, 3, KS>(g, &map, slab, bars, b0s, wxs, x0, y0, z0, NX, xr, red);
    else
        gather_item_tma<MT, 4, KS>(g, &map, slab, bars, b0s, wxs, x0, y0, z0, NX, xr, red);
    __syncthreads();
    // u_t[c] = h^3 sum_y wy_t[y] red[(c, y)][t]   (rows at the fixed pitch NYB)
    if (tid < 3 * MAXT) {
        const int t = tid % MAXT, cc = tid / MAXT;
        if (t < n) {
            const int4 ti = tinfo[t];
            const double* wy = w + static_cast<int64_t>(ti.x) * 3 * P + P;
            const int yo = ti.z - y0;
            double s = 0.0;
            for (int p = 0; p < P; ++p) s = fma(wy[p], red[(cc * NYB + yo + p) * MAXT + t], s);
            u[3 * static_cast<int64_t>(perm[ti.x]) + cc] = scale * s;
        }
    }
}

// items per (coarse tile, z-half): ceil(n / 32)
// A (coarse tile, z-half) whose union box [x0, x0 + P + 7) misses this
// slab's planes [x_lo, x_lo + nx) gets no items: with several slabs each rank
// only visits the tiles that reach its planes (their targets' partial
// velocities are zero here, the caller clears u first).
__global__ void k_slab_counts(const int32_t* __restrict__ tstart, int64_t nhalf, int ncz,
                              int ncy, int x_lo, int nx, int span, int32_t* __restrict__ cnt) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e < nhalf) {
        const int n = tstart[4 * e + 4] - tstart[4 * e];
        const int64_t c = e >> 1;
        const int x0 = static_cast<int>(c / (static_cast<int64_t>(ncz) * ncy)) * 8;
        const bool meets = x0 < x_lo + nx && x0 + span > x_lo;
        cnt[e] = meets ? (n + MAXT - 1) / MAXT : 0;
    }
    if (e == nhalf) cnt[e] = 0;
}

__global__ void k_slab_fill(const int32_t* __restrict__ off, int64_t nhalf,
                            int32_t* __restrict__ items) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= nhalf) return;
    for (int32_t j = off[e]; j < off[e + 1]; ++j) {
        items[2 * j] = static_cast<int32_t>(e);
        items[2 * j + 1] = j - off[e];
    }
}

int ks_for(int P) { return (P + 7 + 3) / 4; }
int mt_for(int P) { return (3 * (P + 7) + 8 * SW - 1) / (8 * SW); }

}  // namespace

size_t slab_smem_bytes(const GridParams& g) {
    const int rows = 8 * mt_for(g.P) * SW;
    return sizeof(double) * (NST * static_cast<size_t>(rows) * RS + 32 * MAXT + 8 * 4 * 32);
}

bool gather_slab_enabled(const GridParams& g) {
    static const bool off = [] {
        const char* e = std::getenv("FSE_GATHER_SLAB");
        return e && std::atoi(e) == 0;
    }();
    const int ks = ks_for(g.P), mt = mt_for(g.P);
    return !off && g.P + 7 <= 32 && ks >= 4 && ks <= 8 && mt >= 1 && mt <= 3;
}

void launch_slab_counts(const Launch& L, const GridParams& g, const int32_t* tstart,
                        int64_t nhalf, int32_t* cnt) {
    k_slab_counts<<<static_cast<unsigned>((nhalf + 256) / 256), 256, 0, L.s>>>(
        tstart, nhalf, g.ncz, g.ncy, g.x_lo, g.nx, g.P + 7, cnt);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_slab_fill(const Launch& L, const int32_t* off, int64_t nhalf, int32_t* items) {
    k_slab_fill<<<static_cast<unsigned>((nhalf + 255) / 256), 256, 0, L.s>>>(off, nhalf, items);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

template <int MT, int KS>
static void launch_mma(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                       const int32_t* tstart, const int32_t* items, int64_t max_items,
                       const int32_t* nitems_dev, const double* X, const uint32_t* perm,
                       double scale, double* u) {
    const size_t sm = slab_smem_bytes(g);
    FSE_CU(cudaFuncSetAttribute(k_gather_mma<MT, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sm)));
    k_gather_mma<MT, KS><<<static_cast<unsigned>(max_items), SW * 32, sm, L.s>>>(
        g, i0s, w, tstart, items, nitems_dev, X, perm, scale, u);
}

// tensor map of the quadrature grid X[c][x][y][z] (3 components of this slab's
// planes): 4-d, z fastest, box 34 z x (P+7) y x 1 x x 3 c, zero fill outside
bool encode_grid_map(const GridParams& g, const double* X, CUtensorMap* map) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.Mt), static_cast<cuuint64_t>(g.Mt),
                                static_cast<cuuint64_t>(g.nx), 3};
    const cuuint64_t strides[3] = {sizeof(double) * static_cast<cuuint64_t>(g.rowp),
                                   sizeof(double) * static_cast<cuuint64_t>(g.plane),
                                   sizeof(double) * static_cast<cuuint64_t>(g.comp)};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(RS), static_cast<cuuint32_t>(g.P + 7), 1, 3};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(X), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool gather_tma_enabled(const GridParams& g) {
    static const bool off = [] {
        const char* e = std::getenv("FSE_GATHER_TMA");
        return e && std::atoi(e) == 0;
    }();
    return !off && g.Mt % 2 == 0 && g.nx > 0;
}

template <int MT, int KS>
void launch_tma(const Launch& L, const CUtensorMap& map, const GridParams& g, const int32_t* i0s,
                const double* w, const int32_t* tstart, const int32_t* items, int64_t max_items,
                const int32_t* nitems_dev, const uint32_t* perm, double scale, double* u) {
    constexpr int ROWS = 8 * MT * SW;
    const size_t sm = sizeof(double) * (2 * static_cast<size_t>(ROWS) * RS + 32 * MAXT +
                                        KS * 4 * 32) +
                      sizeof(int4) * MAXT + 2 * sizeof(uint64_t) + 4 * sizeof(int2);
    FSE_CU(cudaFuncSetAttribute(k_gather_tma<MT, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sm)));
    k_gather_tma<MT, KS><<<static_cast<unsigned>(max_items), SW * 32, sm, L.s>>>(
        map, g, i0s, w, tstart, items, nitems_dev, perm, scale, u);
}

void launch_gather_slab(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                        const int32_t* tstart, const int32_t* items, int64_t max_items,
                        const int32_t* nitems_dev, const double* X, const uint32_t* perm,
                        double scale, double* u) {
    if (max_items <= 0) return;
    const int ks = ks_for(g.P), mt = mt_for(g.P);
    CUtensorMap map;
    if (gather_tma_enabled(g) && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
        encode_grid_map(g, X, &map)) {
#define FSE_TMA_CASE(M_, K_)                                                                   \
    if (mt == M_ && ks == K_) {                                                                \
        launch_tma<M_, K_>(L, map, g, i0s, w, tstart, items, max_items, nitems_dev, perm,      \
                           scale, u);                                                          \
        FSE_LAUNCH_CHECK();                                                                    \
        ++*L.launches;                                                                         \
        return;                                                                                \
    }
        FSE_TMA_CASE(3, 8)
        FSE_TMA_CASE(2, 8)
        FSE_TMA_CASE(1, 8)
        FSE_TMA_CASE(3, 7)
        FSE_TMA_CASE(3, 6)
        FSE_TMA_CASE(2, 7)
        FSE_TMA_CASE(2, 6)
        FSE_TMA_CASE(2, 5)
        FSE_TMA_CASE(2, 4)
        FSE_TMA_CASE(1, 4)
#undef FSE_TMA_CASE
    }
#define FSE_MMA_CASE(M_, K_)                                                                   \
    if (mt == M_ && ks == K_) {                                                                \
        launch_mma<M_, K_>(L, g, i0s, w, tstart, items, max_items, nitems_dev, X, perm, scale, \
                           u);                                                                 \
    } else
    FSE_MMA_CASE(3, 8)
    FSE_MMA_CASE(3, 7)
    FSE_MMA_CASE(3, 6)
    FSE_MMA_CASE(2, 7)
    FSE_MMA_CASE(2, 6)
    FSE_MMA_CASE(2, 5)
    FSE_MMA_CASE(2, 4)
    FSE_MMA_CASE(1, 4)
    throw Error(FSE_EINVAL, "gather: no tensor-core variant for this support");
#undef FSE_MMA_CASE
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
