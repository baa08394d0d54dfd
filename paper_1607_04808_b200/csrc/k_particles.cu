// k_particles.cu -- per-point preparation kernels (HBM-bound, one thread per
// point): support start indices and tile keys, the FGG axis weights in
// tile-sorted order, cell ids for the real-space cell list, SoA permutes.
//
// Bit-exactness: i0 = (int)ceil((x - origin)/h - P/2) (ewald.cpp:38-39) and
// cell = clamp(floor((x - origin)/side)) (realspace.cpp:60-63) are computed
// with explicitly rounded IEEE ops (__dsub_rn/__ddiv_rn), so they match the
// reference's x86-64 doubles exactly.
#include "fse_internal.cuh"

namespace fsecu {

namespace {

constexpr int TPB = 256;

inline unsigned blocks_for(int64_t n, int tpb = TPB) {
    return static_cast<unsigned>((n + tpb - 1) / tpb);
}

__device__ __forceinline__ int support_start(double x, double origin, double h, int P) {
    const double s = __ddiv_rn(__dsub_rn(x, origin), h);
    return static_cast<int>(ceil(__dsub_rn(s, 0.5 * P)));
}

__global__ void k_support_keys(GridParams g, const double* __restrict__ pos, int64_t n,
                               int check_box, uint32_t* __restrict__ key,
                               int32_t* __restrict__ i0out, int* __restrict__ flags) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= n) return;
    int ii[3];
    bool bad = false, outside = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = pos[3 * q + a];
        if (!(x >= 0.0 && x <= g.L)) outside = true;
        int f = support_start(x, g.origin, g.h, g.P);
        if (f < 0 || f + g.P > g.Mt || x != x) {
            bad = true;
            f = f < 0 ? 0 : g.Mt - g.P;
        }
        ii[a] = f;
    }
    if (check_box && outside) atomicOr(flags, FLAG_TARGET_BOX);
    if (bad) atomicOr(flags, FLAG_SUPPORT);
    if (i0out) {
        i0out[3 * q] = ii[0];
        i0out[3 * q + 1] = ii[1];
        i0out[3 * q + 2] = ii[2];
    }
    if (key) {
        const uint32_t cx = ii[0] >> 3, cy = ii[1] >> 3, cz = ii[2] >> 4;
        const uint32_t coarse = (cx * g.ncy + cy) * g.ncz + cz;
        // z-half first, so each 8 x 8 x 8 half of a coarse tile is a
        // contiguous key range (the slab gather's work item)
        const uint32_t fine = (((ii[2] >> 3) & 1) << 2) | (((ii[0] >> 2) & 1) << 1) |
                              ((ii[1] >> 2) & 1);
        key[q] = coarse * 8u + fine;
    }
}

__global__ void k_quad_table(GridParams g, double* q) {
    const int p = threadIdx.x;
    if (p < g.P) q[p] = exp(-g.alpha * (p * g.h) * (p * g.h));  // ewald.cpp:154-156
}

// FGG axis weights (ewald.cpp:33-51) for point perm[q], stored at sorted slot q.
// Three threads per point, one per axis (the 3 P weights are three independent
// chains of P products), PT points per block.  The weights are built in shared
// memory (row stride 3P+1) and the block then writes its points' rows, which
// are one contiguous run of w, with consecutive threads on consecutive doubles.
__global__ void k_payload(GridParams g, const double* __restrict__ pos,
                          const double* __restrict__ str, int a, const uint32_t* __restrict__ perm,
                          int64_t n, const double* __restrict__ qtab, int32_t* __restrict__ i0s,
                          double* __restrict__ w, double* __restrict__ fs, bool fold_prefac,
                          int slab_only, bool naive) {
    extern __shared__ double stage[];
    __shared__ int fx_s[128];
    __shared__ bool keep_row[128];
    const int P = g.P, W3 = 3 * P, RS = W3 + 1;
    const int PT = static_cast<int>(blockDim.x) / 3;
    const int ax = static_cast<int>(threadIdx.x) / PT, pt = static_cast<int>(threadIdx.x) - ax * PT;
    const int64_t q0 = blockIdx.x * static_cast<int64_t>(PT);
    const int64_t q = q0 + pt;
    const bool valid = q < n;
    int64_t idx = 0;
    double s = 0.0;
    int first = 0;
    if (valid) {
        idx = perm[q];
        s = __ddiv_rn(__dsub_rn(pos[3 * idx + ax], g.origin), g.h);
        first = static_cast<int>(ceil(__dsub_rn(s, 0.5 * P)));
        int f = first < 0 ? 0 : first;
        if (f + P > g.Mt) f = g.Mt - P;
        i0s[3 * q + ax] = f;
        if (ax == 0) fx_s[pt] = f;
    }
    __syncthreads();
    // slab_only 1 (sources): a point whose x support misses this slab's
    // planes is never read by its spread tiles; 2 (targets): a target whose
    // coarse tile's union box misses them is in no quadrature item
    // (k_slab_counts).  Such points get no weights.
    bool keep = false;
    if (valid) {
        const int fx = fx_s[pt];
        const int x0 = (fx >> 3) * 8;
        keep = slab_only == 0 ||
               (slab_only == 1 ? (fx + P > g.x_lo && fx < g.x_lo + g.nx)
                               : (x0 < g.x_lo + g.nx && x0 + P + 7 > g.x_lo));
    }
    if (ax == 0) keep_row[pt] = keep;
    if (keep) {
        double* row = stage + pt * RS + ax * P;
        const double scale = (fold_prefac && ax == 0) ? g.prefac : 1.0;
        if (naive) {
            // axis_weights_naive (ewald.cpp:53-66): one exp per node
            for (int p = 0; p < P; ++p) {
                const double dx = (static_cast<double>(first + p) - s) * g.h;
                row[p] = scale * exp(-g.alpha * dx * dx);
            }
        } else {
            const double x0 = (first - s) * g.h;
            const double e0 = exp(-g.alpha * x0 * x0);
            const double ratio = exp(-2.0 * g.alpha * x0 * g.h);
            double r = 1.0;
            for (int p = 0; p < P; ++p) {
                row[p] = scale * (e0 * r * qtab[p]);
                r *= ratio;
            }
        }
        if (fs)
            for (int c = ax; c < a; c += 3) fs[q * a + c] = str[idx * a + c];
    }
    __syncthreads();
    const int64_t left = n - q0;
    const int cnt = static_cast<int>(left < PT ? left : PT);
    double* out = w + q0 * W3;
    for (int e = threadIdx.x; e < cnt * W3; e += blockDim.x) {
        const int t = e / W3;
        if (keep_row[t]) out[e] = stage[t * RS + (e - t * W3)];
    }
}

__global__ void k_histogram(const uint32_t* __restrict__ keys, int64_t n, int32_t* counts) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q < n) atomicAdd(&counts[keys[q]], 1);
}

// sub = 8 or 64: key = sub * cell + sub-cell, the real-space kernels' own ordering
// (k_realspace.cu).  The top three sub-cell bits are the octant, one bit per axis
// = (coordinate >= cell centre) -- the octant items' culling rule rests on exactly
// this comparison; sub = 64 appends the quarter bits (ordering only: the 32 targets
// of an item are neighbours).  The cell itself is the reference's
// (realspace.cpp:78-84) for every sub.
__global__ void k_cell_ids(const double* __restrict__ pos, int64_t n, double origin, double side,
                           int dim, int sub, uint32_t* __restrict__ cell) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= n) return;
    int c[3];
    uint32_t oct = 0, quad = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = pos[3 * q + a];
        int v = static_cast<int>(floor(__ddiv_rn(__dsub_rn(x, origin), side)));
        c[a] = v < 0 ? 0 : (v > dim - 1 ? dim - 1 : v);
        const bool hi = x >= origin + (c[a] + 0.5) * side;
        oct = (oct << 1) | (hi ? 1u : 0u);
        quad = (quad << 1) | (x >= origin + (c[a] + (hi ? 0.75 : 0.25)) * side ? 1u : 0u);
    }
    const uint32_t id = (static_cast<uint32_t>(c[0]) * dim + c[1]) * dim + c[2];
    cell[q] = sub == 64 ? id * 64u + oct * 8u + quad : (sub == 8 ? id * 8u + oct : id);
}

__global__ void k_permute_soa(const double* __restrict__ pos, const double* __restrict__ str,
                              int a, const uint32_t* __restrict__ perm, int64_t n,
                              double* __restrict__ px, double* __restrict__ py,
                              double* __restrict__ pz, double* __restrict__ fs) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= n) return;
    const int64_t idx = perm[q];
    px[q] = pos[3 * idx];
    py[q] = pos[3 * idx + 1];
    pz[q] = pos[3 * idx + 2];
    if (fs)
        for (int c = 0; c < a; ++c) fs[q * a + c] = str[idx * a + c];
}

__global__ void k_iota(uint32_t* v, int64_t n) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q < n) v[q] = static_cast<uint32_t>(q);
}

__global__ void k_u32_to_i64(const uint32_t* in, int64_t* out, int64_t n) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q < n) out[q] = in[q];
}

__global__ void k_i32_to_i64(const int32_t* in, int64_t* out, int64_t n) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q < n) out[q] = in[q];
}

}  // namespace

void launch_support_keys(const Launch& L, const GridParams& g, const double* pos, int64_t n,
                         int check_box, uint32_t* key, int32_t* i0, int* flags) {
    if (n <= 0) return;
    k_support_keys<<<blocks_for(n), TPB, 0, L.s>>>(g, pos, n, check_box, key, i0, flags);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_quad_table(const Launch& L, const GridParams& g, double* q) {
    k_quad_table<<<1, 128, 0, L.s>>>(g, q);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_gather_payload(const Launch& L, const GridParams& g, const double* pos,
                           const double* str, int a, const uint32_t* perm, int64_t n,
                           const double* qtab, int32_t* i0s, double* w, double* fs,
                           bool fold_prefac, int slab_only, bool naive) {
    if (n <= 0) return;
    // points per block: up to 64 (three threads each) whose staged weight rows
    // fit 48 KB; wider supports take fewer points and opt-in shared memory
    const size_t row_bytes = sizeof(double) * (3 * g.P + 1);
    int pt = static_cast<int>((48 * 1024) / row_bytes) / 32 * 32;
    pt = pt < 32 ? 32 : (pt > 64 ? 64 : pt);
    if (row_bytes * pt > 48 * 1024) {
        if (row_bytes * pt > 227 * 1024)
            throw Error(FSE_EINVAL, "k_payload: Gaussian support too wide");
        FSE_CU(cudaFuncSetAttribute(k_payload, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(row_bytes * pt)));
    }
    k_payload<<<static_cast<unsigned>((n + pt - 1) / pt), 3 * pt, row_bytes * pt, L.s>>>(
        g, pos, str, a, perm, n, qtab, i0s, w, fs, fold_prefac, slab_only, naive);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_histogram(const Launch& L, const uint32_t* keys, int64_t n, int32_t* counts) {
    if (n <= 0) return;
    k_histogram<<<blocks_for(n), TPB, 0, L.s>>>(keys, n, counts);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_cell_ids(const Launch& L, const double* pos, int64_t n, double origin, double side,
                     int dim, uint32_t* cell, int sub) {
    if (n <= 0) return;
    k_cell_ids<<<blocks_for(n), TPB, 0, L.s>>>(pos, n, origin, side, dim, sub, cell);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_permute_soa(const Launch& L, const double* pos, const double* str, int a,
                        const uint32_t* perm, int64_t n, double* px, double* py, double* pz,
                        double* fs) {
    if (n <= 0) return;
    k_permute_soa<<<blocks_for(n), TPB, 0, L.s>>>(pos, str, a, perm, n, px, py, pz, fs);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_iota(const Launch& L, uint32_t* v, int64_t n) {
    if (n <= 0) return;
    k_iota<<<blocks_for(n), TPB, 0, L.s>>>(v, n);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_u32_to_i64(const Launch& L, const uint32_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    k_u32_to_i64<<<blocks_for(n), TPB, 0, L.s>>>(in, out, n);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

void launch_i32_to_i64(const Launch& L, const int32_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    k_i32_to_i64<<<blocks_for(n), TPB, 0, L.s>>>(in, out, n);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
