// k_gather.cu -- trapezoidal quadrature back to the targets (ewald.cpp:349-391).
//
// One warp per group of up to K = 8 targets whose support starts lie in the
// same 4 x 4 x 8 fine tile (targets are tile-sorted).  The group's supports
// fit in a union box of at most (P+3) x (P+3) x (P+7) nodes; lanes span z
// (32 at a time), the warp walks the union's (x, y) rows and each grid row is
// loaded ONCE (3 coalesced loads) and reused by all K targets:
//     S_t[c] += wy_t[y] g_c[x][y][z_lane]            (per row,  3K DFMA)
//     T_t[c] += wx_t[x] S_t[c]                       (per x)
//     u_t[c]  = h^3 prefac sum_lanes wz_t[z_lane] T_t[c]   (warp reduction)
// Weights outside a target's support are stored as zeros in per-warp
// shared-memory windows, so the inner loop has no compares.  Register
// accumulation, no atomics, deterministic.  Results are scattered to the
// caller's target order.
//
// Roofline: FP64 FMA (2 a P^3 flops per target).
#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int K = 8;        // targets per warp group
constexpr int WPB = 4;      // warps per CTA
constexpr int MAXU = 72;    // union window (P + 7 <= 72 => P <= 64)

struct GatherWarp {
    double wxu[K][MAXU];
    double wyu[K][MAXU];
    int q[K];
    int ix[K], iy[K], iz[K];
};

__global__ void __launch_bounds__(WPB * 32) k_gather(
    GridParams g, const int32_t* __restrict__ i0s, const double* __restrict__ w,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ gkey,
    const int32_t* __restrict__ goff, const int32_t* __restrict__ ngroups_dev,
    const double* __restrict__ X,
    const uint32_t* __restrict__ perm, double scale, double* __restrict__ u) {
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

    const int64_t rowpitch = g.rowp;
    double res[3] = {0.0, 0.0, 0.0};  // lane t < cnt ends up holding target t
    for (int zc = Z0; zc < Z1; zc += 32) {
        const int z = zc + lane;
        const bool zok = z < Z1;
        double wz[K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
            double v = 0.0;
            if (t < cnt && zok) {
                const int pz = z - s.iz[t];
                if (pz >= 0 && pz < P) v = w[static_cast<int64_t>(s.q[t]) * 3 * P + 2 * P + pz];
            }
            wz[t] = v;
        }
        double T[K][3];
#pragma unroll
        for (int t = 0; t < K; ++t) T[t][0] = T[t][1] = T[t][2] = 0.0;
        const double* base0 = X + (zok ? z : 0);
        for (int xx = 0; xx < NX; ++xx) {
            double S[K][3];
#pragma unroll
            for (int t = 0; t < K; ++t) S[t][0] = S[t][1] = S[t][2] = 0.0;
            const double* rowp = base0 + (X0 + xx) * g.plane + static_cast<int64_t>(Y0) * rowpitch;
            double g0 = 0, g1 = 0, g2 = 0;
            if (zok) {
                g0 = rowp[0];
                g1 = rowp[g.comp];
                g2 = rowp[2 * g.comp];
            }
            for (int yy = 0; yy < NY; ++yy) {
                // prefetch the next row before using this one
                double n0 = 0, n1 = 0, n2 = 0;
                if (zok && yy + 1 < NY) {
                    const double* nx = rowp + (yy + 1) * rowpitch;
                    n0 = nx[0];
                    n1 = nx[g.comp];
                    n2 = nx[2 * g.comp];
                }
#pragma unroll
                for (int t = 0; t < K; ++t) {
                    const double wy = s.wyu[t][yy];
                    S[t][0] = fma(wy, g0, S[t][0]);
                    S[t][1] = fma(wy, g1, S[t][1]);
                    S[t][2] = fma(wy, g2, S[t][2]);
                }
                g0 = n0;
                g1 = n1;
                g2 = n2;
            }
#pragma unroll
            for (int t = 0; t < K; ++t) {
                const double wx = s.wxu[t][xx];
                T[t][0] = fma(wx, S[t][0], T[t][0]);
                T[t][1] = fma(wx, S[t][1], T[t][1]);
                T[t][2] = fma(wx, S[t][2], T[t][2]);
            }
        }
        // reduce wz_t * T_t over lanes; lane t keeps target t
#pragma unroll
        for (int t = 0; t < K; ++t) {
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
    if (lane < cnt) {
        const int64_t m = perm[first + lane];
        u[3 * m] = scale * res[0];
        u[3 * m + 1] = scale * res[1];
        u[3 * m + 2] = scale * res[2];
    }
}

// ---------------------------------------------------------------------------
// Plane-streamed variant (P + 7 <= 32): one CTA per 8 x 8 x 8 region of
// support starts (coarse tile, z half) = 4 fine tiles.  The region's union
// box (<= 31 x 31 x 31 nodes) is streamed x-plane by x-plane into shared
// memory with cp.async (double-buffered, 3 x 32 x 32 doubles per plane), and
// the CTA's 8 warps -- each owning one group of <= 8 targets as above --
// read every grid value from shared memory.  Each plane crosses L2 once per
// CTA instead of once per warp (the L2->SM traffic of the warp-per-group
// kernel was ~100 GB per cfg2 step).  Lanes map to region-relative z.
constexpr int PW = 8;  // warps per CTA

struct PlaneSmem {
    double plane[2][3][32][32];  // [buf][comp][y - y0n][z - z0n]
    double wxu[PW][K][32];
    double wyu[PW][K][32];
    int q[PW][K], ix[PW][K], iy[PW][K], iz[PW][K];
    int gfirst[4], gcount[4], key[4];
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int n = ok ? 8 : 0;  // zero-fill outside the grid
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}

__global__ void __launch_bounds__(PW * 32, 2) k_gather_planes(
    GridParams g, const int32_t* __restrict__ i0s, const double* __restrict__ w,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ goff,
    const double* __restrict__ X, const uint32_t* __restrict__ perm, double scale,
    double* __restrict__ u) {
    extern __shared__ __align__(16) unsigned char gsm_raw[];
    PlaneSmem& S = *reinterpret_cast<PlaneSmem*>(gsm_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = g.P;
    const int zhalf = blockIdx.x & 1;
    const int coarse = blockIdx.x >> 1;
    const int tz = coarse % g.ncz, ty = (coarse / g.ncz) % g.ncy, tx = coarse / (g.ncz * g.ncy);
    const int x0n = tx * 8, y0n = ty * 8, z0n = tz * 16 + zhalf * 8;
    if (threadIdx.x < 4) {
        const int k = coarse * 8 + (threadIdx.x >> 1) * 4 + (threadIdx.x & 1) * 2 + zhalf;
        S.key[threadIdx.x] = k;
        S.gfirst[threadIdx.x] = goff[k];
        S.gcount[threadIdx.x] = goff[k + 1] - goff[k];
    }
    __syncthreads();
    const int ng = S.gcount[0] + S.gcount[1] + S.gcount[2] + S.gcount[3];
    if (ng == 0) return;
    const int NYc = min(P + 7, g.Mt - y0n);           // region rows
    const int X1c = min(x0n + P + 7, g.Mt);             // region x-range end
    const int64_t rowp = g.rowp;

    for (int round = 0; round < ng; round += PW) {
        // ---- my group: (key, index within key)
        const int gi = round + warp;
        int cnt = 0, first = 0;
        if (gi < ng) {
            int kk = 0, rem = gi;
            while (rem >= S.gcount[kk]) rem -= S.gcount[kk++];
            const int key = S.key[kk];
            first = tstart[key] + K * rem;
            cnt = min(first + K, static_cast<int>(tstart[key + 1])) - first;
        }
        int mx = 1 << 30, my = 1 << 30, Mx = -1, My = -1;
        if (lane < cnt) {
            const int q = first + lane;
            const int ix = i0s[3 * q], iy = i0s[3 * q + 1], iz = i0s[3 * q + 2];
            S.q[warp][lane] = q;
            S.ix[warp][lane] = ix;
            S.iy[warp][lane] = iy;
            S.iz[warp][lane] = iz;
            mx = Mx = ix;
            my = My = iy;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = min(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            my = min(my, __shfl_xor_sync(0xffffffffu, my, o));
            Mx = max(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
            My = max(My, __shfl_xor_sync(0xffffffffu, My, o));
        }
        const int X0 = mx, X1 = Mx + P, Y0 = my, Y1 = My + P;
        __syncwarp();
        for (int e = lane; e < K * 32; e += 32) {
            const int t = e >> 5, uu = e & 31;
            double vx = 0.0, vy = 0.0;
            if (t < cnt) {
                const double* wq = w + static_cast<int64_t>(S.q[warp][t]) * 3 * P;
                const int px = X0 + uu - S.ix[warp][t], py = Y0 + uu - S.iy[warp][t];
                if (px >= 0 && px < P) vx = wq[px];
                if (py >= 0 && py < P) vy = wq[P + py];
            }
            S.wxu[warp][t][uu] = vx;
            S.wyu[warp][t][uu] = vy;
        }
        // per-lane z weights (region-relative lane z = z0n + lane)
        double wz[K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
            double v = 0.0;
            if (t < cnt) {
                const int pz = z0n + lane - S.iz[warp][t];
                if (pz >= 0 && pz < P) v = w[static_cast<int64_t>(S.q[warp][t]) * 3 * P + 2 * P + pz];
            }
            wz[t] = v;
        }
        double T[K][3];
#pragma unroll
        for (int t = 0; t < K; ++t) T[t][0] = T[t][1] = T[t][2] = 0.0;

        // ---- stream the region's x-planes
        auto issue = [&](int x, int buf) {
            const double* base = X + static_cast<int64_t>(x) * g.plane;
            for (int e = threadIdx.x; e < 3 * 32 * 32; e += PW * 32) {
                const int c = e >> 10, yy = (e >> 5) & 31, zz = e & 31;
                const int y = y0n + yy, z = z0n + zz;
                const bool ok = yy < NYc && z < g.Mt;
                const double* src = ok ? base + c * g.comp + y * rowp + z : X;
                cp_async8(&S.plane[buf][c][yy][zz], src, ok);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        issue(x0n, 0);
        for (int x = x0n; x < X1c; ++x) {
            const int buf = (x - x0n) & 1;
            if (x + 1 < X1c) {
                issue(x + 1, buf ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncthreads();
            if (x >= X0 && x < X1) {
                double Sacc[K][3];
#pragma unroll
                for (int t = 0; t < K; ++t) Sacc[t][0] = Sacc[t][1] = Sacc[t][2] = 0.0;
                const double* p0 = &S.plane[buf][0][0][lane];
                for (int y = Y0; y < Y1; ++y) {
                    const int yy = y - y0n;
                    const double g0 = p0[yy * 32], g1 = p0[1024 + yy * 32], g2 = p0[2048 + yy * 32];
                    const int uy = y - Y0;
#pragma unroll
                    for (int t = 0; t < K; ++t) {
                        const double wy = S.wyu[warp][t][uy];
                        Sacc[t][0] = fma(wy, g0, Sacc[t][0]);
                        Sacc[t][1] = fma(wy, g1, Sacc[t][1]);
                        Sacc[t][2] = fma(wy, g2, Sacc[t][2]);
                    }
                }
#pragma unroll
                for (int t = 0; t < K; ++t) {
                    const double wx = S.wxu[warp][t][x - X0];
                    T[t][0] = fma(wx, Sacc[t][0], T[t][0]);
                    T[t][1] = fma(wx, Sacc[t][1], T[t][1]);
                    T[t][2] = fma(wx, Sacc[t][2], T[t][2]);
                }
            }
            __syncthreads();  // buffer reuse
        }
        // ---- reduce wz_t * T_t over lanes; lane t writes target t
        double res0 = 0, res1 = 0, res2 = 0;
#pragma unroll
        for (int t = 0; t < K; ++t) {
            double v0 = wz[t] * T[t][0], v1 = wz[t] * T[t][1], v2 = wz[t] * T[t][2];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, o);
                v1 += __shfl_xor_sync(0xffffffffu, v1, o);
                v2 += __shfl_xor_sync(0xffffffffu, v2, o);
            }
            if (lane == t) {
                res0 = v0;
                res1 = v1;
                res2 = v2;
            }
        }
        if (lane < cnt) {
            const int64_t m = perm[first + lane];
            u[3 * m] = scale * res0;
            u[3 * m + 1] = scale * res1;
            u[3 * m + 2] = scale * res2;
        }
        __syncwarp();
    }
}

__global__ void k_group_counts(const int32_t* __restrict__ tstart, int64_t nkeys,
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

void launch_group_counts(const Launch& L, const int32_t* tstart, int64_t nkeys, int32_t* gcount) {
    k_group_counts<<<static_cast<unsigned>((nkeys + 256) / 256), 256, 0, L.s>>>(tstart, nkeys,
                                                                              gcount);
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

bool gather_planes_ok(const GridParams& g) { return g.P + 7 <= 32; }

void launch_gather_planes(const Launch& L, const GridParams& g, const int32_t* i0s,
                          const double* w, const int32_t* tstart, const int32_t* goff,
                          const double* X, const uint32_t* perm, double scale, double* u) {
    const size_t sm = sizeof(PlaneSmem);
    FSE_CU(cudaFuncSetAttribute(k_gather_planes, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sm)));
    const unsigned blocks = static_cast<unsigned>(g.ncx) * g.ncy * g.ncz * 2;
    k_gather_planes<<<blocks, PW * 32, sm, L.s>>>(g, i0s, w, tstart, goff, X, perm, scale, u);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_gather(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                   const int32_t* tstart, const int32_t* gkey, const int32_t* goff,
                   int64_t max_groups, const double* X, const uint32_t* perm, double scale,
                   double* u) {
    if (max_groups <= 0) return;
    const unsigned blocks = static_cast<unsigned>((max_groups + WPB - 1) / WPB);
    k_gather<<<blocks, WPB * 32, 0, L.s>>>(g, i0s, w, tstart, gkey, goff, goff + g.nkeys, X, perm,
                                           scale, u);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
