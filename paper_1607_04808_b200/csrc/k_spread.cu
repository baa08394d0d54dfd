// k_spread.cu -- Gaussian spreading (ewald.cpp:136-214), atomics-free.
//
// Ownership instead of atomics: one CTA owns an 8 x 8 x 16 tile of grid
// nodes and is the only writer of it.  Each of its 4 warps owns one
// (x-half, z-half) of the tile -- 4 x-rows x 8 y x 8 z -- and accumulates it
// on the FP64 tensor cores: for every group of 4 points (one k-step of
// mma.m8n8k4.f64)
//     G_c[(x, y)][z] += sum_p (wx_p[x] wy_p[y]) (f_{c,p} wz_p[z]),
// 4 x-m-tiles x 3 component-n-tiles = 12 MMAs per group from 7 fragment
// products (1 DMUL each); a group none of whose supports meets the warp's
// domain is skipped (one staged byte per point).  The CTA streams, in
// tile-key order, every point whose P^3 support meets the tile (points are
// pre-sorted by the tile of their support start i0, so those points sit in
// 4 x 4 contiguous key ranges), stages the slices of their separable weights
// that fall on the tile in shared memory (wx[8], wy[8], wz[16], f[3] per
// point; cp.async, double-buffered so the next chunk's copies overlap this
// chunk's MMAs), and every lane accumulates in registers: no shared-memory
// read-modify-write, no global atomics; fixed order (deterministic).
//
// Roofline: FP64 FMA (2 a P^3 flops per point, ~100 flop/B); HBM traffic is
// the weights (3P doubles per point) plus one write of the grid.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

#ifndef FSE_SPREAD_NWARP
#define FSE_SPREAD_NWARP 4
#endif
// NWARP = 2: warp w owns z [8w, 8w + 8) of all 8 x-rows; NWARP = 4: warp w
// owns x-rows [4 (w % 2), +4) and z [8 (w / 2), +8).  CH = 64 points per chunk
// (staged by the first 64 threads).
#ifndef FSE_SPREAD_CH
#define FSE_SPREAD_CH 64
#endif
constexpr int TX = 8, TY = 8, TZ = 16, CH = FSE_SPREAD_CH, NWARP = FSE_SPREAD_NWARP;
constexpr int XS = NWARP / 2, XW = TX / XS;  // x splits, x-rows per warp
// 4 warps: (x-half, z-half) domains, 96 registers for five CTAs per SM
// (cfg2 spread 7.28 -> 6.60 ms against 2 warps with all 8 x-rows each)
#ifndef FSE_SPREAD_MINB
#define FSE_SPREAD_MINB 5
#endif

// element-major staging ([element][point], point stride CHP = CH + 4): the
// per-thread staging writes of a warp are consecutive doubles and the MMA
// fragment reads (4 points x 8 rows) spread over all banks
#ifndef FSE_SPREAD_PAD
#define FSE_SPREAD_PAD 4
#endif
constexpr int CHP = CH + FSE_SPREAD_PAD;
struct Stage {
    // wx and f are read 4 consecutive points of one row at a time (no
    // conflicts unpadded); wy and wz rows are read 8 at a time (padded).
    // Unpadded they bring the CTA to 37.5 KB: six CTAs per SM instead of five.
    double wx[TX][CH];
    double wy[TY][CHP];
    double wz[TZ][CHP];
    double f[3][CH];
    // bit w: the point's z-support meets warp w's 8 z (read 4 points at a time)
    uint32_t zm4[CH / 4];
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa8(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
                 : "memory");
}

// Walk over the CTA's point chunks: the 4 x 4 (x, y) coarse-tile columns
// whose starts can reach the tile, each a contiguous key range.
struct Cursor {
    int kx, ky, base, qend;
};

__global__ void __launch_bounds__(NWARP * 32, FSE_SPREAD_MINB) k_spread(GridParams g, const int32_t* __restrict__ i0s,
                                                       const double* __restrict__ w,
                                                       const double* __restrict__ fs, int a, int c0,
                                                       const int32_t* __restrict__ tstart,
                                                       const int32_t* __restrict__ order,
                                                       double* __restrict__ X) {
    __shared__ __align__(16) Stage st[2];
    __shared__ int cnts[3][NWARP];
    const int P = g.P;
    const int tile = order ? order[blockIdx.x] : static_cast<int>(blockIdx.x);  // heaviest first
    const int tz = tile % g.ncz;
    const int ty = (tile / g.ncz) % g.ncy;
    const int tx = g.x_lo / TX + tile / (g.ncz * g.ncy);  // this slab's x tiles
    const int x0n = tx * TX, y0n = ty * TY, z0n = tz * TZ;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // warp w owns x-rows [wx_off, +XW) and z [wz_lo, +8) of the tile
    const int wx_off = (warp % XS) * XW;
    const int wz_off = (warp / XS) * 8;
    const int wz_lo = z0n + wz_off;

    // MMA accumulators: C[x][c] holds G_c[x0n + wx_off + x][y0n + lane/4][wz_lo + 2 (lane%4) + {0,1}]
    double C[XW][3][2];
#pragma unroll
    for (int r = 0; r < XW; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) C[r][c][0] = C[r][c][1] = 0.0;

    // support starts that reach the tile: i0 in [n0 - P + 1, n0 + T - 1]
    const int ix_lo = x0n - P + 1, iy_lo = y0n - P + 1, iz_lo = z0n - P + 1;
    const int kx_lo = ix_lo < 0 ? 0 : (ix_lo >> 3);
    const int ky_lo = iy_lo < 0 ? 0 : (iy_lo >> 3);
    const int kz_lo = iz_lo < 0 ? 0 : (iz_lo >> 4);
    auto range = [&](Cursor& c) {  // load [base, qend) of column (kx, ky)
        const int64_t kb = (static_cast<int64_t>(c.kx) * g.ncy + c.ky) * g.ncz;
        c.base = tstart[(kb + kz_lo) * 8];
        c.qend = tstart[(kb + tz) * 8 + 8];
    };
    auto next_nonempty = [&](Cursor& c) {  // advance columns until a chunk exists
        while (c.kx <= tx && c.base >= c.qend) {
            if (++c.ky > ty) {
                c.ky = ky_lo;
                ++c.kx;
            }
            if (c.kx <= tx) range(c);
        }
    };
    // per-chunk metadata: which of this thread's point is kept (support meets the tile)
    auto meta = [&](const Cursor& c, int& q, int& ix, int& iy, int& iz) -> bool {
        q = c.base + tid;
        if (tid >= CH || q >= c.qend) return false;
        ix = i0s[3 * q];
        iy = i0s[3 * q + 1];
        iz = i0s[3 * q + 2];
        return ix >= ix_lo && ix <= x0n + TX - 1 && iy >= iy_lo && iy <= y0n + TY - 1 &&
               iz >= iz_lo && iz <= z0n + TZ - 1;
    };
    // asynchronous staging of the kept points' weight slices (zero outside the support)
    auto stage = [&](Stage& S, int slot, int q, int ix, int iy, int iz) {
        const double* wq = w + static_cast<int64_t>(q) * 3 * P;
#pragma unroll
        for (int r = 0; r < TX; ++r) {
            const int p = x0n + r - ix;
            const bool in = p >= 0 && p < P;
            cpa8(&S.wx[r][slot], in ? wq + p : wq, in ? 8 : 0);
        }
#pragma unroll
        for (int r = 0; r < TY; ++r) {
            const int p = y0n + r - iy;
            const bool in = p >= 0 && p < P;
            cpa8(&S.wy[r][slot], in ? wq + P + p : wq, in ? 8 : 0);
        }
#pragma unroll
        for (int r = 0; r < TZ; ++r) {
            const int p = z0n + r - iz;
            const bool in = p >= 0 && p < P;
            cpa8(&S.wz[r][slot], in ? wq + 2 * P + p : wq, in ? 8 : 0);
        }
        const double* fq = fs + static_cast<int64_t>(q) * a + c0;
        cpa8(&S.f[0][slot], fq, 8);
        cpa8(&S.f[1][slot], fq + 1, 8);
        cpa8(&S.f[2][slot], fq + 2, 8);
        uint32_t zb = 0;  // bit w: the support meets warp w's x-rows and z range
#pragma unroll
        for (int ww = 0; ww < NWARP; ++ww) {
            const int xa = x0n + (ww % XS) * XW, za = z0n + (ww / XS) * 8;
            const bool in = !(ix > xa + XW - 1 || ix + P <= xa) && !(iz > za + 7 || iz + P <= za);
            zb |= static_cast<uint32_t>(in) << ww;
        }
        reinterpret_cast<uint8_t*>(S.zm4)[slot] = static_cast<uint8_t>(zb);
    };

    Cursor cur;
    cur.kx = kx_lo;
    cur.ky = ky_lo;
    range(cur);
    next_nonempty(cur);
    int q = 0, ix = 0, iy = 0, iz = 0;
    bool keep = cur.kx <= tx && meta(cur, q, ix, iy, iz);
    unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) cnts[0][warp] = __popc(bal);
    __syncthreads();
    // slot of this thread's kept point: kept points of the staging warps before it
    auto slot_of = [&](int kk) {
        int off = 0;
#pragma unroll
        for (int w = 0; w < CH / 32; ++w)
            if (w < warp) off += cnts[kk][w];
        return off + __popc(bal & ((1u << lane) - 1u));
    };
    if (keep) stage(st[0], slot_of(0), q, ix, iy, iz);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    int k = 0, b = 0;
    while (cur.kx <= tx) {
        // metadata of the next chunk (overlaps the copies in flight)
        Cursor nxt = cur;
        nxt.base += CH;
        next_nonempty(nxt);
        const bool more = nxt.kx <= tx;
        const int kn = k == 2 ? 0 : k + 1;
        keep = more && meta(nxt, q, ix, iy, iz);
        bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) cnts[kn][warp] = __popc(bal);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();  // chunk k staged; everyone is done with buffer b ^ 1
        if (keep)
            stage(st[b ^ 1], slot_of(kn), q, ix, iy, iz);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const Stage& S = st[b];
        int total = 0;
#pragma unroll
        for (int w = 0; w < CH / 32; ++w) total += cnts[k][w];
        // groups of 4 points = one k-step of m8n8k4:
        //   A[(x, y)][p] = wx_p[x] wy_p[y]   (m-tile = one x, rows y)
        //   B[p][(c, z)] = f_{c,p} wz_p[z]   (n-tile = one component, 8 z of this warp)
        // one k-step of 4 points; FULL: all 4 slots hold points of this chunk
        // (every group but possibly the last), so no tail masking/selects
        auto group = [&](int p0, auto full) {
            constexpr bool FULL = decltype(full)::value;
            // warp-uniform skip when no support of the group meets this warp's z
            // range (one byte per point; bytes past `total` are stale: masked)
            uint32_t zm = S.zm4[p0 >> 2] & (0x01010101u << warp);
            if (!FULL) zm &= (1u << (8 * (total - p0))) - 1u;
            if (zm == 0u) return;
            const int p = p0 + (lane & 3);
            const bool pv = FULL || p < total;
            const int pp = pv ? p : p0;
            const double wyv = pv ? S.wy[lane >> 2][pp] : 0.0;
            const double wzv = pv ? S.wz[wz_off + (lane >> 2)][pp] : 0.0;
            const double bf[3] = {S.f[0][pp] * wzv, S.f[1][pp] * wzv, S.f[2][pp] * wzv};
#pragma unroll
            for (int r = 0; r < XW; ++r) {
                const double ar = S.wx[wx_off + r][pp] * wyv;
#pragma unroll
                for (int c = 0; c < 3; ++c) dmma(C[r][c][0], C[r][c][1], ar, bf[c]);
            }
        };
        int p0 = 0;
        for (; p0 + 4 <= total; p0 += 4) group(p0, std::true_type{});
        if (p0 < total) group(p0, std::false_type{});
        cur = nxt;
        k = kn;
        b ^= 1;
    }

    const int y = y0n + (lane >> 2), z = wz_lo + 2 * (lane & 3);
    if (y >= g.Mt || z >= g.Mt) return;
    const bool z1 = z + 1 < g.Mt;
    const bool vec = z1 && (g.Mt % 2 == 0);  // 16-byte aligned pairs
#pragma unroll
    for (int r = 0; r < XW; ++r) {
        const int x = x0n + wx_off + r;
        if (x >= g.x_lo + g.nx) break;
        const int64_t off = (x - g.x_lo) * g.plane + y * g.rowp + z;  // slab-local plane
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double* dst = X + (c0 + c) * g.comp + off;
            if (vec) {
                *reinterpret_cast<double2*>(dst) = make_double2(C[r][c][0], C[r][c][1]);
            } else {
                dst[0] = C[r][c][0];
                if (z1) dst[1] = C[r][c][1];
            }
        }
    }
}

// ---------------------------------------------------------------- warp-specialized
// Same tile, warp domains, staging layout and MMAs as k_spread, but the chunk
// staging is done by a dedicated producer warp into a ring of NSTG stages
// handed over with mbarriers (full: the stage's copies have landed; empty:
// all four MMA warps are done with it), so the MMA warps never wait for each
// other at a CTA barrier (k_spread's per-chunk __syncthreads was ~24 % of its
// stall samples: the warps' skip patterns make their chunk times differ).
#ifndef FSE_SPREAD_NSTG
#define FSE_SPREAD_NSTG 3
#endif
constexpr int NSTG = FSE_SPREAD_NSTG;
struct StageW {
    Stage st;
    int total;  // kept points in the stage; -1: no more chunks
};

__device__ __forceinline__ unsigned su32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(su32(b)), "r"(parity)
            : "memory");
    }
}

#ifndef FSE_SPREAD_WS_MINB
#define FSE_SPREAD_WS_MINB 4
#endif
__global__ void __launch_bounds__((NWARP + 1) * 32, FSE_SPREAD_WS_MINB) k_spread_ws(
    GridParams g, const int32_t* __restrict__ i0s, const double* __restrict__ w,
    const double* __restrict__ fs, int a, int c0, const int32_t* __restrict__ tstart,
    const int32_t* __restrict__ order, double* __restrict__ X) {
    extern __shared__ __align__(16) unsigned char spw_smem[];
    StageW* ring = reinterpret_cast<StageW*>(spw_smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NSTG);
    uint64_t* empty = full + NSTG;
    const int P = g.P;
    const int tile = order ? order[blockIdx.x] : static_cast<int>(blockIdx.x);  // heaviest first
    const int tz = tile % g.ncz;
    const int ty = (tile / g.ncz) % g.ncy;
    const int tx = g.x_lo / TX + tile / (g.ncz * g.ncy);
    const int x0n = tx * TX, y0n = ty * TY, z0n = tz * TZ;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int b = 0; b < NSTG; ++b) {
            mb_init(full + b, 33);
            mb_init(empty + b, NWARP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();  // the only CTA-wide barrier

    if (warp == NWARP) {
        // ---------------- producer: stream the points whose support meets the tile
        const int ix_lo = x0n - P + 1, iy_lo = y0n - P + 1, iz_lo = z0n - P + 1;
        const int kx_lo = ix_lo < 0 ? 0 : (ix_lo >> 3);
        const int ky_lo = iy_lo < 0 ? 0 : (iy_lo >> 3);
        const int kz_lo = iz_lo < 0 ? 0 : (iz_lo >> 4);
        auto range = [&](Cursor& c) {
            const int64_t kb = (static_cast<int64_t>(c.kx) * g.ncy + c.ky) * g.ncz;
            c.base = tstart[(kb + kz_lo) * 8];
            c.qend = tstart[(kb + tz) * 8 + 8];
        };
        auto next_nonempty = [&](Cursor& c) {
            while (c.kx <= tx && c.base >= c.qend) {
                if (++c.ky > ty) {
                    c.ky = ky_lo;
                    ++c.kx;
                }
                if (c.kx <= tx) range(c);
            }
        };
        Cursor cur;
        cur.kx = kx_lo;
        cur.ky = ky_lo;
        range(cur);
        next_nonempty(cur);
        int k = 0;
        for (;; ++k) {
            const int b = k % NSTG;
            if (k >= NSTG) mb_wait(empty + b, ((k / NSTG) - 1) & 1);
            StageW& S = ring[b];
            const bool more = cur.kx <= tx;
            int total = -1;
            if (more) {
                // CH candidates, CH / 32 per lane; kept ones compacted in order
                int off = 0;
#pragma unroll
                for (int h = 0; h < CH / 32; ++h) {
                    const int q = cur.base + h * 32 + lane;
                    int ix = 0, iy = 0, iz = 0;
                    bool keep = false;
                    if (q < cur.qend) {
                        ix = i0s[3 * q];
                        iy = i0s[3 * q + 1];
                        iz = i0s[3 * q + 2];
                        keep = ix >= ix_lo && ix <= x0n + TX - 1 && iy >= iy_lo &&
                               iy <= y0n + TY - 1 && iz >= iz_lo && iz <= z0n + TZ - 1;
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        const int slot = off + __popc(bal & ((1u << lane) - 1u));
                        const double* wq = w + static_cast<int64_t>(q) * 3 * P;
#pragma unroll
                        for (int r = 0; r < TX; ++r) {
                            const int p = x0n + r - ix;
                            const bool in = p >= 0 && p < P;
                            cpa8(&S.st.wx[r][slot], in ? wq + p : wq, in ? 8 : 0);
                        }
#pragma unroll
                        for (int r = 0; r < TY; ++r) {
                            const int p = y0n + r - iy;
                            const bool in = p >= 0 && p < P;
                            cpa8(&S.st.wy[r][slot], in ? wq + P + p : wq, in ? 8 : 0);
                        }
#pragma unroll
                        for (int r = 0; r < TZ; ++r) {
                            const int p = z0n + r - iz;
                            const bool in = p >= 0 && p < P;
                            cpa8(&S.st.wz[r][slot], in ? wq + 2 * P + p : wq, in ? 8 : 0);
                        }
                        const double* fq = fs + static_cast<int64_t>(q) * a + c0;
                        cpa8(&S.st.f[0][slot], fq, 8);
                        cpa8(&S.st.f[1][slot], fq + 1, 8);
                        cpa8(&S.st.f[2][slot], fq + 2, 8);
                        uint32_t zb = 0;
#pragma unroll
                        for (int ww = 0; ww < NWARP; ++ww) {
                            const int xa = x0n + (ww % XS) * XW, za = z0n + (ww / XS) * 8;
                            const bool in = !(ix > xa + XW - 1 || ix + P <= xa) &&
                                            !(iz > za + 7 || iz + P <= za);
                            zb |= static_cast<uint32_t>(in) << ww;
                        }
                        reinterpret_cast<uint8_t*>(S.st.zm4)[slot] = static_cast<uint8_t>(zb);
                    }
                    off += __popc(bal);
                }
                total = off;
                cur.base += CH;
                next_nonempty(cur);
            }
            if (lane == 0) S.total = total;
            // full[b] completes when every lane's copies have landed (32
            // asynchronous arrives) and lane 0 has released the metadata
            // (total, zm) the warp wrote: the producer goes straight on to
            // the next chunk instead of waiting for the copies
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(full + b))
                         : "memory");
            __syncwarp();
            if (lane == 0) mb_arrive(full + b);
            if (!more) break;
        }
        return;
    }

    // ---------------- MMA warps (warp w owns x-rows [wx_off, +XW), z [wz_off, +8))
    const int wx_off = (warp % XS) * XW;
    const int wz_off = (warp / XS) * 8;
    const int wz_lo = z0n + wz_off;
    double C[XW][3][2];
#pragma unroll
    for (int r = 0; r < XW; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) C[r][c][0] = C[r][c][1] = 0.0;
    for (int k = 0;; ++k) {
        const int b = k % NSTG;
        mb_wait(full + b, (k / NSTG) & 1);
        const StageW& SW = ring[b];
        const int total = SW.total;
        if (total < 0) break;
        const Stage& S = SW.st;
        auto group = [&](int p0, auto fullg) {
            constexpr bool FULL = decltype(fullg)::value;
            uint32_t zm = S.zm4[p0 >> 2] & (0x01010101u << warp);
            if (!FULL) zm &= (1u << (8 * (total - p0))) - 1u;
            if (zm == 0u) return;
            const int p = p0 + (lane & 3);
            const bool pv = FULL || p < total;
            const int pp = pv ? p : p0;
            const double wyv = pv ? S.wy[lane >> 2][pp] : 0.0;
            const double wzv = pv ? S.wz[wz_off + (lane >> 2)][pp] : 0.0;
            const double bf[3] = {S.f[0][pp] * wzv, S.f[1][pp] * wzv, S.f[2][pp] * wzv};
#pragma unroll
            for (int r = 0; r < XW; ++r) {
                const double ar = S.wx[wx_off + r][pp] * wyv;
#pragma unroll
                for (int c = 0; c < 3; ++c) dmma(C[r][c][0], C[r][c][1], ar, bf[c]);
            }
        };
        int p0 = 0;
        for (; p0 + 4 <= total; p0 += 4) group(p0, std::true_type{});
        if (p0 < total) group(p0, std::false_type{});
        __syncwarp();
        if (lane == 0) mb_arrive(empty + b);
    }

    const int y = y0n + (lane >> 2), z = wz_lo + 2 * (lane & 3);
    if (y >= g.Mt || z >= g.Mt) return;
    const bool z1 = z + 1 < g.Mt;
    const bool vec = z1 && (g.Mt % 2 == 0);
#pragma unroll
    for (int r = 0; r < XW; ++r) {
        const int x = x0n + wx_off + r;
        if (x >= g.x_lo + g.nx) break;
        const int64_t off = (x - g.x_lo) * g.plane + y * g.rowp + z;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double* dst = X + (c0 + c) * g.comp + off;
            if (vec) {
                *reinterpret_cast<double2*>(dst) = make_double2(C[r][c][0], C[r][c][1]);
            } else {
                dst[0] = C[r][c][0];
                if (z1) dst[1] = C[r][c][1];
            }
        }
    }
}

__global__ void k_extract(GridParams g, const double* __restrict__ X, int a,
                          double* __restrict__ out) {
    const int64_t vol = static_cast<int64_t>(g.Mt) * g.Mt * g.Mt;
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= vol * a) return;
    const int64_t c = q / vol, r = q % vol;
    const int64_t z = r % g.Mt, y = (r / g.Mt) % g.Mt, x = r / (static_cast<int64_t>(g.Mt) * g.Mt);
    out[q] = X[c * g.comp + x * g.plane + y * g.rowp + z];
}

constexpr int kTileBuckets = 32;

// Heavy tiles are scheduled first: the points a tile streams (those whose support
// meets it) vary by two orders of magnitude on clustered input (cfg4), and a heavy
// tile dispatched last leaves the GPU waiting on one CTA.  Tiles with at least
// heavy_min points (four times the mean) go to the front of the order, bucketed by
// log2(points), heaviest bucket first; the others follow in their natural order, which keeps
// neighbouring tiles -- they stream the same points -- close in time (a fully
// bucketed order cost uniform input 5%: cfg2 6.16 -> 6.47 ms).  The order only
// schedules: every tile is still computed by exactly one CTA in its own fixed order.
__global__ void k_tile_flag(GridParams g, const int32_t* __restrict__ tstart, unsigned tiles,
                            long long heavy_min, int32_t* __restrict__ light,
                            uint8_t* __restrict__ hbucket, int32_t* __restrict__ bwork) {
    const unsigned tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= tiles) return;
    const int P = g.P;
    const int tz = tile % g.ncz;
    const int ty = (tile / g.ncz) % g.ncy;
    const int tx = g.x_lo / TX + tile / (g.ncz * g.ncy);
    const int ix_lo = tx * TX - P + 1, iy_lo = ty * TY - P + 1, iz_lo = tz * TZ - P + 1;
    const int kx_lo = ix_lo < 0 ? 0 : (ix_lo >> 3);
    const int ky_lo = iy_lo < 0 ? 0 : (iy_lo >> 3);
    const int kz_lo = iz_lo < 0 ? 0 : (iz_lo >> 4);
    long long work = 0;
    for (int kx = kx_lo; kx <= tx; ++kx)
        for (int ky = ky_lo; ky <= ty; ++ky) {
            const int64_t kb = (static_cast<int64_t>(kx) * g.ncy + ky) * g.ncz;
            work += tstart[(kb + tz) * 8 + 8] - tstart[(kb + kz_lo) * 8];
        }
    const bool heavy = work >= heavy_min;
    light[tile] = heavy ? 0 : 1;
    if (heavy) {  // bucket by log2(points), bucket 0 heaviest
        const int bk = max(0, kTileBuckets - 1 - (63 - __clzll(work)));
        hbucket[tile] = static_cast<uint8_t>(bk);
        atomicAdd(bwork + bk, 1);
    }
}

// one warp: bucket offsets of the heavy tiles and their total
__global__ void k_tile_scan(int32_t* __restrict__ bwork) {
    const int l = threadIdx.x;
    const int v = bwork[l];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += t;
    }
    bwork[kTileBuckets + l] = incl - v;
    if (l == 31) bwork[3 * kTileBuckets] = incl;
}

// heavy tiles bucket by bucket (heaviest first), then the light tiles in natural
// order (pos = exclusive scan of light)
__global__ void k_tile_place(const int32_t* __restrict__ light, const int32_t* __restrict__ pos,
                             const uint8_t* __restrict__ hbucket, int32_t* __restrict__ bwork,
                             unsigned tiles, int32_t* __restrict__ order) {
    const unsigned tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= tiles) return;
    if (light[tile]) {
        order[bwork[3 * kTileBuckets] + pos[tile]] = static_cast<int32_t>(tile);
    } else {
        const int bk = hbucket[tile];
        order[bwork[kTileBuckets + bk] + atomicAdd(bwork + 2 * kTileBuckets + bk, 1)] =
            static_cast<int32_t>(tile);
    }
}

}  // namespace

unsigned spread_tiles(const GridParams& g) {
    return static_cast<unsigned>((g.nx + TX - 1) / TX) * g.ncy * g.ncz;
}

// step 1: light flags (tiles ints), heavy tiles' buckets (tiles bytes) and bucket
// offsets; bwork = 3 * 32 + 1 ints
void launch_spread_flags(const Launch& L, const GridParams& g, const int32_t* tstart, int64_t n,
                         int32_t* light, uint8_t* hbucket, int32_t* bwork) {
    const unsigned tiles = spread_tiles(g);
    if (tiles == 0) return;
    // mean points per tile: each point meets ~ (P + 7) / 8 tiles per axis in x and y
    // and (P + 15) / 16 in z
    const double per_axis = (g.P + 7) / 8.0;
    const double total_tiles = static_cast<double>(g.ncx) * g.ncy * g.ncz;
    const double mean = static_cast<double>(n) * per_axis * per_axis * ((g.P + 15) / 16.0) /
                        std::max(total_tiles, 1.0);
    const long long heavy_min = static_cast<long long>(4.0 * mean) + 64;
    FSE_CU(cudaMemsetAsync(bwork, 0, (3 * kTileBuckets + 1) * sizeof(int32_t), L.s));
    k_tile_flag<<<(tiles + 255) / 256, 256, 0, L.s>>>(g, tstart, tiles, heavy_min, light, hbucket,
                                                      bwork);
    FSE_LAUNCH_CHECK();
    k_tile_scan<<<1, 32, 0, L.s>>>(bwork);
    FSE_LAUNCH_CHECK();
    *L.launches += 2;
}

// step 2, after pos = exclusive scan of light
void launch_spread_place(const Launch& L, const GridParams& g, const int32_t* light,
                         const int32_t* pos, const uint8_t* hbucket, int32_t* bwork,
                         int32_t* order) {
    const unsigned tiles = spread_tiles(g);
    if (tiles == 0) return;
    k_tile_place<<<(tiles + 255) / 256, 256, 0, L.s>>>(light, pos, hbucket, bwork, tiles, order);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_spread(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                   const double* fs, int64_t n, int a, int c0, const int32_t* tstart,
                   double* X, const int32_t* order) {
    (void)n;
    const unsigned tiles = spread_tiles(g);
    if (tiles == 0) return;
    static const int ws = [] {
        const char* e = std::getenv("FSE_SPREAD_WS");
        return e ? std::atoi(e) : 1;
    }();
    if (ws) {
        const size_t sm = sizeof(StageW) * NSTG + 2 * NSTG * sizeof(uint64_t);
        static bool attr = false;
        if (!attr) {
            FSE_CU(cudaFuncSetAttribute(k_spread_ws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sm)));
            attr = true;
        }
        k_spread_ws<<<tiles, (NWARP + 1) * 32, sm, L.s>>>(g, i0s, w, fs, a, c0, tstart, order, X);
    } else {
        k_spread<<<tiles, NWARP * 32, 0, L.s>>>(g, i0s, w, fs, a, c0, tstart, order, X);
    }
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_extract_grid(const Launch& L, const GridParams& g, const double* X, int a,
                         double* out) {
    const int64_t tot = static_cast<int64_t>(g.Mt) * g.Mt * g.Mt * a;
    k_extract<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.s>>>(g, X, a, out);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
