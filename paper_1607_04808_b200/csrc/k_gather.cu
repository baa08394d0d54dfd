// k_gather.cu -- trapezoidal quadrature back to the targets (ewald.cpp:349-391).
//
// One warp per group of up to K = 4 targets whose support starts lie in the
// same 4 x 4 x 8 fine tile (targets are tile-sorted); the register block is
// picked per group (2 or 4 targets; 6 or 8 with FSE_GATHER_K=8).  The group's supports
// fit in a union box of at most (P+3) x (P+3) x (P+7) nodes; lanes span z
// (32 at a time), the warp walks the union's (x, y) rows with RING rows in
// flight and each grid row is loaded ONCE (3 coalesced loads) and reused by
// all K targets:
//     S_t[c] += wy_t[y] g_c[x][y][z_lane]            (per row,  3K DFMA)
//     T_t[c] += wx_t[x] S_t[c]                       (per x)
//     u_t[c]  = h^3 prefac sum_lanes wz_t[z_lane] T_t[c]   (warp reduction)
// Weights outside a target's support are stored as zeros in per-warp
// shared-memory windows, so the inner loop has no compares.  Register
// accumulation, no atomics, deterministic.  Results are scattered to the
// caller's target order.
//
// Roofline: FP64 FMA (2 a P^3 flops per target).
#include <cstdlib>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int WPB = 4;      // warps per CTA
constexpr int MAXU = 72;    // union window (P + 7 <= 72 => P <= 64)

struct GatherWarp {
    double wxu[8][MAXU];
    double wyu[8][MAXU];
    int q[8];
    int ix[8], iy[8], iz[8];
};

constexpr int RING = 4;  // grid rows in flight per lane (hides the L2 latency)

// Contract the group's union box for KK >= cnt targets (KK a compile-time
// bound so S/T stay in registers; the group size picks the smallest).
template <int KK>
__device__ __forceinline__ void gather_box(const GridParams& g, const GatherWarp& s, int cnt,
                                           int X0, int NX, int Y0, int NY, int Z0, int Z1,
                                           const double* __restrict__ w,
                                           const double* __restrict__ X, int lane,
                                           double res[3]) {
    const int P = g.P;
    const int64_t plane = g.plane, rowp = g.rowp, comp = g.comp;
    for (int zc = Z0; zc < Z1; zc += 32) {
        const int z = zc + lane;
        const bool zok = z < Z1;
        double wz[KK];
#pragma unroll
        for (int t = 0; t < KK; ++t) {
            double v = 0.0;
            if (t < cnt && zok) {
                const int pz = z - s.iz[t];
                if (pz >= 0 && pz < P) v = w[static_cast<int64_t>(s.q[t]) * 3 * P + 2 * P + pz];
            }
            wz[t] = v;
        }
        // lanes past Z1 read a valid node (z = Z0) and carry wz = 0
        // lanes past Z1 read a valid node (z = Z0) and carry wz = 0; rows
        // are padded to a multiple of RING (wy = 0 there, y clamped in range)
        const double* zb = X + (zok ? z : Z0) + static_cast<int64_t>(X0) * plane;
        const int NYp = (NY + RING - 1) / RING * RING;
        const int ymax = g.Mt - 1;
        double gb[RING][3];
#pragma unroll
        for (int j = 0; j < RING; ++j) {
            const double* rp = zb + min(Y0 + j, ymax) * rowp;
            gb[j][0] = rp[0];
            gb[j][1] = rp[comp];
            gb[j][2] = rp[2 * comp];
        }
        double T[KK][3];
#pragma unroll
        for (int t = 0; t < KK; ++t) T[t][0] = T[t][1] = T[t][2] = 0.0;
        for (int xx = 0; xx < NX; ++xx) {
            double S[KK][3];
#pragma unroll
            for (int t = 0; t < KK; ++t) S[t][0] = S[t][1] = S[t][2] = 0.0;
            for (int y0 = 0; y0 < NYp; y0 += RING) {
                // the row group RING ahead (next x-plane after the last group)
                int nx = xx, ny = y0 + RING;
                if (ny == NYp) {
                    ny = 0;
                    ++nx;
                }
                const bool more = nx < NX;
                const double* np = zb + nx * plane;
#pragma unroll
                for (int j = 0; j < RING; ++j) {
                    const double g0 = gb[j][0], g1 = gb[j][1], g2 = gb[j][2];
                    if (more) {
                        const double* rp = np + min(Y0 + ny + j, ymax) * rowp;
                        gb[j][0] = rp[0];
                        gb[j][1] = rp[comp];
                        gb[j][2] = rp[2 * comp];
                    }
#pragma unroll
                    for (int t = 0; t < KK; ++t) {
                        const double wy = s.wyu[t][y0 + j];
                        S[t][0] = fma(wy, g0, S[t][0]);
                        S[t][1] = fma(wy, g1, S[t][1]);
                        S[t][2] = fma(wy, g2, S[t][2]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < KK; ++t) {
                const double wx = s.wxu[t][xx];
                T[t][0] = fma(wx, S[t][0], T[t][0]);
                T[t][1] = fma(wx, S[t][1], T[t][1]);
                T[t][2] = fma(wx, S[t][2], T[t][2]);
            }
        }
        // reduce wz_t * T_t over lanes; lane t keeps target t
#pragma unroll
        for (int t = 0; t < KK; ++t) {
            double v0 = wz[t] * T[t][0], v1 = wz[t] * T[t][1], v2 = wz[t] * T[t][2];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, o);
                v1 += __shfl_xor_sync(0xffffffffu, v1, o);
                v2 += __shfl_xor_sync(0xffffffffu, v2, o);
            }
            if (lane == t) {
                res[0] += v0;
                res[1] += v1;
                res[2] += v2;
            }
        }
    }
}

template <int K>
__global__ void __launch_bounds__(WPB * 32) k_gather(
    GridParams g, const int32_t* __restrict__ i0s, const double* __restrict__ w,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ gkey,
    const int32_t* __restrict__ goff, const int32_t* __restrict__ ngroups_dev,
    const double* __restrict__ X,
    const uint32_t* __restrict__ perm, double scale, double* __restrict__ u, int dispatch) {
    __shared__ GatherWarp smw[WPB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t grp = static_cast<int64_t>(blockIdx.x) * WPB + warp;
    if (grp >= *ngroups_dev) return;  // grid is an upper bound (no host sync)
    GatherWarp& s = smw[warp];
    const int P = g.P;
    const int key = gkey[grp];
    const int first = tstart[key] + K * static_cast<int>(grp - goff[key]);
    const int last = min(first + K, static_cast<int>(tstart[key + 1]));
    const int cnt = last - first;

    int ix = 1 << 30, iy = 1 << 30, iz = 1 << 30;
    int ax = -1, ay = -1, az = -1;
    if (lane < cnt) {
        const int q = first + lane;
        ix = i0s[3 * q];
        iy = i0s[3 * q + 1];
        iz = i0s[3 * q + 2];
        ax = ix;
        ay = iy;
        az = iz;
        s.q[lane] = q;
        s.ix[lane] = ix;
        s.iy[lane] = iy;
        s.iz[lane] = iz;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ix = min(ix, __shfl_xor_sync(0xffffffffu, ix, o));
        iy = min(iy, __shfl_xor_sync(0xffffffffu, iy, o));
        iz = min(iz, __shfl_xor_sync(0xffffffffu, iz, o));
        ax = max(ax, __shfl_xor_sync(0xffffffffu, ax, o));
        ay = max(ay, __shfl_xor_sync(0xffffffffu, ay, o));
        az = max(az, __shfl_xor_sync(0xffffffffu, az, o));
    }
    const int X0 = ix, X1 = ax + P, Y0 = iy, Y1 = ay + P, Z0 = iz, Z1 = az + P;
    const int NX = X1 - X0, NY = Y1 - Y0;
    __syncwarp();
    // union windows of wx / wy (zeros outside each target's support)
    for (int e = lane; e < K * MAXU; e += 32) {
        const int t = e / MAXU, uu = e % MAXU;
        double vx = 0.0, vy = 0.0;
        if (t < cnt) {
            const double* wq = w + static_cast<int64_t>(s.q[t]) * 3 * P;
            const int px = X0 + uu - s.ix[t], py = Y0 + uu - s.iy[t];
            if (uu < NX && px >= 0 && px < P) vx = wq[px];
            if (uu < NY && py >= 0 && py < P) vy = wq[P + py];
        }
        s.wxu[t][uu] = vx;
        s.wyu[t][uu] = vy;
    }
    __syncwarp();

    double res[3] = {0.0, 0.0, 0.0};  // lane t < cnt ends up holding target t
    if (!dispatch) {
        gather_box<K>(g, s, cnt, X0, NX, Y0, NY, Z0, Z1, w, X, lane, res);
    } else if (K == 4 || cnt <= 4) {
        if (cnt <= 2)
            gather_box<2>(g, s, cnt, X0, NX, Y0, NY, Z0, Z1, w, X, lane, res);
        else
            gather_box<4>(g, s, cnt, X0, NX, Y0, NY, Z0, Z1, w, X, lane, res);
    } else {
        if (cnt <= 6)
            gather_box<6>(g, s, cnt, X0, NX, Y0, NY, Z0, Z1, w, X, lane, res);
        else
            gather_box<K>(g, s, cnt, X0, NX, Y0, NY, Z0, Z1, w, X, lane, res);
    }
    if (lane < cnt) {
        const int64_t m = perm[first + lane];
        u[3 * m] = scale * res[0];
        u[3 * m + 1] = scale * res[1];
        u[3 * m + 2] = scale * res[2];
    }
}

__global__ void k_group_counts(const int32_t* __restrict__ tstart, int64_t nkeys, int K,
                               int32_t* __restrict__ gcount) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k < nkeys) gcount[k] = (tstart[k + 1] - tstart[k] + K - 1) / K;
    if (k == nkeys) gcount[k] = 0;
}

__global__ void k_fill_groups(const int32_t* __restrict__ goff, int64_t nkeys,
                              int32_t* __restrict__ gkey) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nkeys) return;
    for (int32_t gi = goff[k]; gi < goff[k + 1]; ++gi) gkey[gi] = static_cast<int32_t>(k);
}

}  // namespace

// pick the register block by group size (FSE_GATHER_DISPATCH=0: always K)
int gather_dispatch() {
    static const int d = [] {
        const char* e = std::getenv("FSE_GATHER_DISPATCH");
        return (e && std::atoi(e) == 0) ? 0 : 1;
    }();
    return d;
}

// targets per warp group (FSE_GATHER_K=8 trades occupancy for L2 traffic)
int gather_group_size() {
    static const int k = [] {
        const char* e = std::getenv("FSE_GATHER_K");
        return (e && std::atoi(e) == 8) ? 8 : 4;
    }();
    return k;
}

void launch_group_counts(const Launch& L, const int32_t* tstart, int64_t nkeys, int32_t* gcount) {
    k_group_counts<<<static_cast<unsigned>((nkeys + 256) / 256), 256, 0, L.s>>>(
        tstart, nkeys, gather_group_size(), gcount);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_fill_groups(const Launch& L, const int32_t* tstart, const int32_t* goff,
                        int64_t nkeys, int32_t* gkey) {
    (void)tstart;
    k_fill_groups<<<static_cast<unsigned>((nkeys + 255) / 256), 256, 0, L.s>>>(goff, nkeys, gkey);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_gather(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                   const int32_t* tstart, const int32_t* gkey, const int32_t* goff,
                   int64_t max_groups, const double* X, const uint32_t* perm, double scale,
                   double* u) {
    if (max_groups <= 0) return;
    const unsigned blocks = static_cast<unsigned>((max_groups + WPB - 1) / WPB);
    if (gather_group_size() == 4)
        k_gather<4><<<blocks, WPB * 32, 0, L.s>>>(g, i0s, w, tstart, gkey, goff, goff + g.nkeys, X,
                                                  perm, scale, u, gather_dispatch());
    else
        k_gather<8><<<blocks, WPB * 32, 0, L.s>>>(g, i0s, w, tstart, gkey, goff, goff + g.nkeys, X,
                                                  perm, scale, u, gather_dispatch());
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
