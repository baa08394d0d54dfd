// k_spread.cu -- Gaussian spreading (ewald.cpp:136-214), atomics-free.
//
// Ownership instead of atomics: one CTA owns an 8 x 8 x 16 tile of grid
// nodes and is the only writer of it.  Each of its 4 warps owns a 4 (y) x 8 (z)
// patch of lanes and all 8 x-rows of the tile, so every lane keeps 8 x 3
// fp64 accumulators in registers.  The CTA streams, in tile-key order, every
// point whose P^3 support meets the tile (points are pre-sorted by the tile
// of their support start i0, so those points sit in 4 x 4 contiguous
// key ranges), stages the slices of their separable weights that fall on the
// tile in shared memory (wx[8], wy[8], wz[16], f[3] per point), and every lane
// applies acc[x][c] += wx[x] * (wy * wz * f_c): three DFMAs per grid node per
// point, no shared-memory read-modify-write, no global atomics.  The per-node
// summation order is the stable point order, so results are deterministic.
//
// Roofline: FP64 FMA (2 a P^3 flops per point, ~100 flop/B); HBM traffic is
// the weights (3P doubles per point) plus one write of the grid.
#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int TX = 8, TY = 8, TZ = 16, CH = 128;

struct SpreadSmem {
    double wx[CH][TX];
    double wy[CH][TY];
    double wz[CH][TZ];
    double f[CH][3];
    int iy[CH], iz[CH];
    int warp_cnt[4];
};

__global__ void __launch_bounds__(128) k_spread(GridParams g, const int32_t* __restrict__ i0s,
                                                const double* __restrict__ w,
                                                const double* __restrict__ fs, int a, int c0,
                                                const int32_t* __restrict__ tstart,
                                                double* __restrict__ X) {
    __shared__ SpreadSmem sm;
    const int P = g.P;
    const int tile = blockIdx.x;
    const int tz = tile % g.ncz;
    const int ty = (tile / g.ncz) % g.ncy;
    const int tx = tile / (g.ncz * g.ncy);
    const int x0n = tx * TX, y0n = ty * TY, z0n = tz * TZ;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wy_off = (warp & 1) * 4, wz_off = (warp >> 1) * 8;
    const int ly = lane >> 3, lz = lane & 7;
    const int wy_lo = y0n + wy_off, wz_lo = z0n + wz_off;

    double acc[TX][3];
#pragma unroll
    for (int r = 0; r < TX; ++r) acc[r][0] = acc[r][1] = acc[r][2] = 0.0;

    // support starts that reach the tile: i0 in [n0 - P + 1, n0 + T - 1]
    const int ix_lo = x0n - P + 1, iy_lo = y0n - P + 1, iz_lo = z0n - P + 1;
    const int kx_lo = ix_lo < 0 ? 0 : (ix_lo >> 3);
    const int ky_lo = iy_lo < 0 ? 0 : (iy_lo >> 3);
    const int kz_lo = iz_lo < 0 ? 0 : (iz_lo >> 4);

    for (int kx = kx_lo; kx <= tx; ++kx)
        for (int ky = ky_lo; ky <= ty; ++ky) {
            const int64_t kb = (static_cast<int64_t>(kx) * g.ncy + ky) * g.ncz;
            const int qbeg = tstart[(kb + kz_lo) * 8];
            const int qend = tstart[(kb + tz) * 8 + 8];
            for (int base = qbeg; base < qend; base += CH) {
                const int q = base + tid;
                int ix = 0, iy = 0, iz = 0;
                bool keep = false;
                if (q < qend) {
                    ix = i0s[3 * q];
                    iy = i0s[3 * q + 1];
                    iz = i0s[3 * q + 2];
                    keep = ix >= ix_lo && ix <= x0n + TX - 1 && iy >= iy_lo &&
                           iy <= y0n + TY - 1 && iz >= iz_lo && iz <= z0n + TZ - 1;
                }
                // deterministic compaction: warp ballot + per-warp prefix
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (lane == 0) sm.warp_cnt[warp] = __popc(bal);
                __syncthreads();
                int wbase = 0, total = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = sm.warp_cnt[k];
                    wbase += (k < warp) ? c : 0;
                    total += c;
                }
                if (keep) {
                    const int slot = wbase + __popc(bal & ((1u << lane) - 1u));
                    const double* wq = w + static_cast<int64_t>(q) * 3 * P;
#pragma unroll
                    for (int r = 0; r < TX; ++r) {
                        const int p = x0n + r - ix;
                        sm.wx[slot][r] = (p >= 0 && p < P) ? wq[p] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < TY; ++r) {
                        const int p = y0n + r - iy;
                        sm.wy[slot][r] = (p >= 0 && p < P) ? wq[P + p] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < TZ; ++r) {
                        const int p = z0n + r - iz;
                        sm.wz[slot][r] = (p >= 0 && p < P) ? wq[2 * P + p] : 0.0;
                    }
                    const double* fq = fs + static_cast<int64_t>(q) * a + c0;
                    sm.f[slot][0] = fq[0];
                    sm.f[slot][1] = fq[1];
                    sm.f[slot][2] = fq[2];
                    sm.iy[slot] = iy;
                    sm.iz[slot] = iz;
                }
                __syncthreads();
                for (int p = 0; p < total; ++p) {
                    const int iyp = sm.iy[p], izp = sm.iz[p];
                    // warp-uniform skip when the support misses this warp's patch
                    if (iyp > wy_lo + 3 || iyp + P <= wy_lo || izp > wz_lo + 7 ||
                        izp + P <= wz_lo)
                        continue;
                    const double wyz = sm.wy[p][wy_off + ly] * sm.wz[p][wz_off + lz];
                    const double u0 = wyz * sm.f[p][0];
                    const double u1 = wyz * sm.f[p][1];
                    const double u2 = wyz * sm.f[p][2];
#pragma unroll
                    for (int r = 0; r < TX; ++r) {
                        const double wxr = sm.wx[p][r];
                        acc[r][0] = fma(wxr, u0, acc[r][0]);
                        acc[r][1] = fma(wxr, u1, acc[r][1]);
                        acc[r][2] = fma(wxr, u2, acc[r][2]);
                    }
                }
                __syncthreads();
            }
        }

    const int y = wy_lo + ly, z = wz_lo + lz;
    if (y >= g.Mt || z >= g.Mt) return;
    const int64_t rowpitch = g.rowp;
#pragma unroll
    for (int r = 0; r < TX; ++r) {
        const int x = x0n + r;
        if (x >= g.Mt) break;
        const int64_t off = x * g.plane + y * rowpitch + z;
#pragma unroll
        for (int c = 0; c < 3; ++c) X[(c0 + c) * g.comp + off] = acc[r][c];
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

}  // namespace

void launch_spread(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                   const double* fs, int64_t n, int a, int c0, const int32_t* tstart,
                   double* X) {
    (void)n;
    const unsigned tiles = static_cast<unsigned>(g.ncx) * g.ncy * g.ncz;
    k_spread<<<tiles, 128, 0, L.s>>>(g, i0s, w, fs, a, c0, tstart, X);
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
