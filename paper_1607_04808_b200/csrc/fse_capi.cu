// fse_capi.cu -- host orchestration and the C-ABI (include/fse_cuda.h).
//
// One evaluation of fse::total_sum (ewald.cpp:394-415) on one B200:
//
//   stream s0 (Fourier part, ewald.cpp:295-392)
//     support starts + tile keys -> stable radix sort -> tile starts
//     -> FGG weights in sorted order (prefac folded)              [prep]
//     -> k_spread_ws: tile-owned DMMA spreading, no atomics; a producer
//        warp feeds four MMA warps through an mbarrier ring        [spread]
//     -> k_zfwd (R2C along z, two real rows per complex FFT) and
//        k_ypass (y), pruned: zero planes x >= Mtilde are never stored [fft]
//     -> k_xscale*: forward x-FFT, Nyquist-exact multiplier A_eff G / D^3,
//        inverse x-FFT, in shared memory / registers                [scale]
//     -> k_ypass<inverse>, k_zinv (C2R): only the Mtilde^3 window   [fft]
//     -> target prep (reuses the source sort when targets == sources)
//     -> k_gather_tma: TMA-staged x-planes, DMMA z-contraction, targets
//        x-sorted per item, n-tiles skip planes outside their supports [quadrature]
//   stream s1 (real part, realspace.cpp:86-149), concurrent with s0
//     cell ids -> stable radix sort -> bucket starts (the reference CellList)
//     -> SoA permute -> work items heaviest cell first -> k_realspace [realspace]
//   s0 waits for s1 -> k_epilogue: u = (uF + uR) + self term
//
// All FFTs of the hot path are the hand-written engines of k_fft.cu (no cuFFT);
// the Green's precompute uses cuBLAS DGEMMs for its cosine passes and the
// fse::fft3d drop-in uses cuFFT.  Device buffers are cached per context and grow
// on demand.
#include <cublas_v2.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "fse_internal.cuh"
#include "fse_host.h"
#include "k_fft.cuh"

namespace fsecu {

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    throw Error(e == cudaErrorMemoryAllocation ? FSE_ENOMEM : FSE_ECUDA, buf);
}

[[noreturn]] void throw_cufft(cufftResult r, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "cuFFT error %d in %s at %s:%d", static_cast<int>(r), what,
                  file, line);
    throw Error(r == CUFFT_ALLOC_FAILED ? FSE_ENOMEM : FSE_ECUFFT, buf);
}

GridParams make_grid_params(const fse_config& c) {
    GridParams g{};
    g.P = c.P;
    g.Mt = c.Mtilde;
    g.D = 2 * c.Mtilde;
    g.Dh = g.D / 2 + 1;
    g.rowp = g.Mt;
    g.plane = static_cast<int64_t>(g.Mt) * g.Mt;
    g.comp = static_cast<int64_t>(g.Mt) * g.plane;
    g.h = c.h;
    g.origin = -c.deltaL / 2;                                     // ewald.cpp:147
    g.alpha = 2.0 * c.xi * c.xi / c.eta;                          // ewald.cpp:152
    g.prefac = std::pow(2.0 * c.xi * c.xi / (M_PI * c.eta), 1.5);  // ewald.cpp:153
    g.L = c.L;
    g.dk = M_PI / c.Ltilde;                                       // ewald.cpp:232
    g.inv4xi2 = 1.0 / (4.0 * c.xi * c.xi);                        // ewald.cpp:233
    g.eta = c.eta;
    g.invD3 = 1.0 / (static_cast<double>(g.D) * g.D * g.D);        // fft.cpp:34
    g.ncx = (g.Mt + 7) / 8;
    g.ncy = (g.Mt + 7) / 8;
    g.ncz = (g.Mt + 15) / 16;
    g.nkeys = static_cast<int64_t>(g.ncx) * g.ncy * g.ncz * 8;
    g.x_lo = 0;
    g.nx = g.Mt;
    g.nxs = g.Mt;
    g.ky_lo = 0;
    g.nky = g.D;
    g.nkys = g.D;
    return g;
}

void set_slab(GridParams& g, int r, int G) {
    if (G <= 1) return;
    g.nxs = ((g.Mt + G - 1) / G + 7) / 8 * 8;  // x-planes per slab, whole spread tiles
    g.x_lo = std::min(r * g.nxs, g.Mt);
    g.nx = std::min(g.nxs, g.Mt - g.x_lo);
    g.comp = static_cast<int64_t>(g.nx) * g.plane;
    g.nkys = (g.D + G - 1) / G;
    g.ky_lo = std::min(r * g.nkys, g.D);
    g.nky = std::min(g.nkys, g.D - g.ky_lo);
}

namespace {
__global__ void k_not_equal(const double* a, const double* b, int64_t n, int* flag) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q < n && !(a[q] == b[q])) atomicOr(flag, 1);
}
}  // namespace

}  // namespace fsecu

using namespace fsecu;

struct fse_green {
    int kind;
    double Ltilde, h, R;
    int Mtilde;
    int device;
    double* d_half;  // [D][D][D/2+1]
};

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

constexpr int NEV = 16;
constexpr int NKMS = 11;

}  // namespace

struct FftPlanDev {
    HostFftPlan host;
    double2* tw = nullptr;
};

struct fse_cuda_ctx {
    int device = 0;
    std::map<int, FftPlanDev> fft_plans;
    cudaStream_t s0 = nullptr, s1 = nullptr;
    cudaEvent_t ev[NEV] = {};
    cudaEvent_t mark[2] = {};
    int mark_n = 0;
    std::mutex mu;
    std::string err;
    uint64_t launches = 0;
    double kms[NKMS] = {};  // per-kernel device ms of the last evaluation
    std::map<std::string, DevBuf> bufs;
    int* d_flags = nullptr;  // [0] s0 flags, [1] s1 flags, [2] equality flag
    int* h_flags = nullptr;  // pinned
    bool overlap = std::getenv("FSE_SERIAL") == nullptr;  // real space on s1 alongside s0
    unsigned long long* d_counts = nullptr;  // real-space candidates / accepted pairs
    bool str_pending = false;  // strengths still copying on s1 (EV_H2D marks the end)
};

namespace {

struct Guard {
    explicit Guard(fse_cuda_ctx* c) : lk(c->mu) { FSE_CU(cudaSetDevice(c->device)); }
    std::unique_lock<std::mutex> lk;
};

template <class F>
fse_status api(fse_cuda_ctx* ctx, F&& f) {
    if (!ctx) return FSE_EINVAL;
    try {
        Guard g(ctx);
        ctx->err.clear();
        f();
        return FSE_OK;
    } catch (const Error& e) {
        ctx->err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failed";
        return FSE_ENOMEM;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return FSE_ERUNTIME;
    }
}

[[noreturn]] void invalid(const std::string& m) { throw Error(FSE_EINVAL, m); }

void sync_all(fse_cuda_ctx* c) { FSE_CU(cudaDeviceSynchronize()); }

template <class T>
T* buf(fse_cuda_ctx* c, const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    DevBuf& b = c->bufs[name];
    if (b.bytes < bytes) {
        sync_all(c);
        if (b.p) FSE_CU(cudaFree(b.p));
        b.p = nullptr;
        b.bytes = 0;
        // headroom for neighbouring sizes; none on multi-GB buffers (cfg5t's spectra
        // are 62 GB: the headroom alone would be 8 GB)
        const size_t alloc = bytes + (bytes < (size_t(2) << 30) ? bytes / 8 : 0);
        FSE_CU(cudaMalloc(&b.p, alloc));
        b.bytes = alloc;
    }
    return static_cast<T*>(b.p);
}

void release_plans(fse_cuda_ctx* c) {
    for (auto& kv : c->fft_plans)
        if (kv.second.tw) cudaFree(kv.second.tw);
    c->fft_plans.clear();
}

// hand-written FFT plan (radices + long-double twiddle tables), cached per D
const FftPlanDev& fft_plan(fse_cuda_ctx* c, int D) {
    auto it = c->fft_plans.find(D);
    if (it != c->fft_plans.end()) return it->second;
    FftPlanDev p;
    p.host = make_fft_plan(D);
    FSE_CU(cudaMalloc(&p.tw, sizeof(double2) * p.host.tw.size()));
    FSE_CU(cudaMemcpy(p.tw, p.host.tw.data(), sizeof(double2) * p.host.tw.size(),
                      cudaMemcpyHostToDevice));
    return c->fft_plans.emplace(D, std::move(p)).first->second;
}

Launch L0(fse_cuda_ctx* c) { return Launch{c->s0, &c->launches}; }
Launch L1(fse_cuda_ctx* c) { return Launch{c->s1, &c->launches}; }

void check_cfg(const fse_config* cfg) {
    if (!cfg) invalid("null config");
    if (!(cfg->L > 0) || !(cfg->xi > 0) || !(cfg->rc > 0) || cfg->M < 1 || cfg->P < 2 ||
        cfg->P % 2 || cfg->Mtilde < cfg->P || !(cfg->h > 0) || !(cfg->eta > 0))
        invalid("config was not produced by make_config");
}

void check_kind(int kind) {
    if (kind < FSE_STOKESLET || kind > FSE_ROTLET) invalid("unknown kernel kind");
}

// ewald.cpp:93-99
void check_green(const fse_config* cfg, int kind, const fse_green* g) {
    if (!g) invalid("fourier_sum: null green");
    const int want = kind == FSE_ROTLET ? FSE_HARMONIC : FSE_BIHARMONIC;
    if (g->kind != want) invalid("fourier_sum: green kind does not match kernel");
    if (g->Mtilde != cfg->Mtilde || std::abs(g->Ltilde - cfg->Ltilde) > 1e-12 * cfg->Ltilde)
        invalid("fourier_sum: green grid does not match config");
}

void exclusive_scan(fse_cuda_ctx* c, cudaStream_t s, const char* tag, const int32_t* in,
                    int32_t* out, int64_t n) {
    size_t tb = 0;
    FSE_CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, static_cast<int>(n), s));
    void* tmp = buf<char>(c, std::string("cubtmp_") + tag, tb);
    FSE_CU(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, static_cast<int>(n), s));
}

void sort_pairs(fse_cuda_ctx* c, cudaStream_t s, const char* tag, const uint32_t* kin,
                uint32_t* kout, const uint32_t* vin, uint32_t* vout, int64_t n, int bits) {
    size_t tb = 0;
    FSE_CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, static_cast<int>(n),
                                           0, bits, s));
    void* tmp = buf<char>(c, std::string("cubtmp_") + tag, tb);
    FSE_CU(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, static_cast<int>(n), 0,
                                           bits, s));
}

int bits_for(int64_t nkeys) {
    int b = 1;
    while ((int64_t{1} << b) < nkeys) ++b;
    return b;
}

// Sorted point set for the Fourier stages (support-tile order).
enum {
    EV_START, EV_PREP, EV_MEMSET, EV_SPREAD, EV_FFT1, EV_SCALE, EV_FFT2, EV_TPREP, EV_QUAD,
    EV_R0, EV_RPAIR, EV_R1, EV_JOIN, EV_END, EV_H2D, EV_COUNT
};
static_assert(EV_COUNT <= NEV, "event pool");

struct Sorted {
    uint32_t* perm = nullptr;
    int32_t* tstart = nullptr;  // nkeys + 1
    int32_t* i0s = nullptr;
    double* w = nullptr;
    double* fs = nullptr;
};

Sorted prep_points(fse_cuda_ctx* c, const GridParams& g, const std::string& tag,
                   const double* d_pos, const double* d_str, int a, int64_t n, int check_box,
                   const double* qtab, bool naive = false) {
    Launch L = L0(c);
    Sorted s;
    uint32_t* keys = buf<uint32_t>(c, tag + "keys", n);
    uint32_t* keys2 = buf<uint32_t>(c, tag + "keys2", n);
    uint32_t* iota = buf<uint32_t>(c, tag + "iota", n);
    s.perm = buf<uint32_t>(c, tag + "perm", n);
    int32_t* counts = buf<int32_t>(c, tag + "counts", g.nkeys + 1);
    s.tstart = buf<int32_t>(c, tag + "tstart", g.nkeys + 1);
    s.i0s = buf<int32_t>(c, tag + "i0s", 3 * n);
    s.w = buf<double>(c, tag + "w", 3 * g.P * n);
    s.fs = d_str ? buf<double>(c, tag + "fs", a * n) : nullptr;
    launch_support_keys(L, g, d_pos, n, check_box, keys, nullptr, c->d_flags);
    launch_iota(L, iota, n);
    if (n > 0) sort_pairs(c, c->s0, "s0", keys, keys2, iota, s.perm, n, bits_for(g.nkeys));
    FSE_CU(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (g.nkeys + 1), c->s0));
    launch_histogram(L, keys2, n, counts);
    exclusive_scan(c, c->s0, "s0", counts, s.tstart, g.nkeys + 1);
    if (d_str && c->str_pending) FSE_CU(cudaStreamWaitEvent(c->s0, c->ev[EV_H2D], 0));
    // one z-slab: weights only for the sources whose support reaches its planes
    // and the targets of the quadrature items that do (k_slab_counts)
    launch_gather_payload(L, g, d_pos, d_str, a, s.perm, n, qtab, s.i0s, s.w, s.fs, true,
                          g.nx < g.Mt ? (d_str != nullptr ? 1 : 2) : 0, naive);
    return s;
}

// Reference CellList geometry (realspace.cpp:65-76), computed on the host
// with the same libm calls so dims and cell_side are bit-identical.
CellGrid cell_grid(int64_t n, double box_side, double rc, double pad) {
    if (!(rc > 0)) invalid("build_cell_list: rc must be positive");
    CellGrid cg;
    cg.origin = -pad;
    const double extent = box_side + 2.0 * pad;
    const int cap =
        1 + static_cast<int>(std::cbrt(8.0 * static_cast<double>(std::max<int64_t>(n, 1))));
    const int want = std::max(1, static_cast<int>(std::floor(extent / rc)));
    cg.dim = std::min(want, cap);
    cg.side = extent / cg.dim;
    cg.ncell = static_cast<int64_t>(cg.dim) * cg.dim * cg.dim;
    return cg;
}

struct Cells {
    uint32_t* perm = nullptr;
    int32_t* start = nullptr;  // ncell + 1
    double *px = nullptr, *py = nullptr, *pz = nullptr, *fs = nullptr;
};

// sub > 1: sorted by (cell, sub-cell) with sub * ncell + 1 bucket starts (the
// real-space kernels' own order; cell c is [start[sub c], start[sub c + sub]));
// sub = 1: the reference's CellList order (build_cell_list)
Cells bin_cells(fse_cuda_ctx* c, const CellGrid& cg, const std::string& tag, const double* d_pos,
                const double* d_str, int a, int64_t n, int sub = 1) {
    Launch L = L1(c);
    Cells r;
    const int64_t nkeys = sub * cg.ncell;
    uint32_t* cell = buf<uint32_t>(c, tag + "cell", n);
    uint32_t* cell2 = buf<uint32_t>(c, tag + "cell2", n);
    uint32_t* iota = buf<uint32_t>(c, tag + "iota", n);
    r.perm = buf<uint32_t>(c, tag + "perm", n);
    int32_t* counts = buf<int32_t>(c, tag + "counts", nkeys + 1);
    r.start = buf<int32_t>(c, tag + "start", nkeys + 1);
    launch_cell_ids(L, d_pos, n, cg.origin, cg.side, cg.dim, cell, sub);
    launch_iota(L, iota, n);
    if (n > 0) sort_pairs(c, c->s1, "s1", cell, cell2, iota, r.perm, n, bits_for(nkeys));
    FSE_CU(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (nkeys + 1), c->s1));
    launch_histogram(L, cell2, n, counts);
    exclusive_scan(c, c->s1, "s1", counts, r.start, nkeys + 1);
    r.px = buf<double>(c, tag + "px", n);
    r.py = buf<double>(c, tag + "py", n);
    r.pz = buf<double>(c, tag + "pz", n);
    r.fs = d_str ? buf<double>(c, tag + "fs", a * n) : nullptr;
    launch_permute_soa(L, d_pos, d_str, a, r.perm, n, r.px, r.py, r.pz, r.fs);
    return r;
}


// real-space pair sum on s1 into d_uR (caller order).  No host sync: the
// pair kernel is launched over an upper bound of work items and reads the
// true count from device memory.
// part / nparts > 1: only the targets in x-slice `part` of the cell grid
// (whole cells, so work items stay full); the others' d_uR entries are zero
// n_geom >= 0: the point count that fixes the cell geometry (the global N when
// d_pos holds one rank's local sources, so the bins are the reference's)
void real_part(fse_cuda_ctx* c, int kind, const double* d_pos, const double* d_str, int64_t n,
               double box_side, double xi, double rc, const double* d_tgt, int64_t nt, bool tas,
               double* d_uR, int part = 0, int nparts = 1, int64_t n_geom = -1) {
    if (!(xi > 0) || !(rc > 0)) invalid("real_space_sum: xi and rc must be positive");
    const int a = arity_of(kind);
    const CellGrid cg = cell_grid(n_geom >= 0 ? n_geom : n, box_side, rc, 0.0);
    // sub-cell buckets per cell: 64 (octant + quarter bits) while the bucket tables
    // stay small next to the points, else 8, else the plain cell order
    const int64_t room = 16 * std::max(n, nt) + (int64_t(1) << 20);
    const int sub = 64 * cg.ncell <= room ? 64 : (8 * cg.ncell <= room ? 8 : 1);
    Cells src = bin_cells(c, cg, "rs_", d_pos, d_str, a, n, sub);
    Cells tgt = tas ? src : bin_cells(c, cg, "rt_", d_tgt, nullptr, 0, nt, sub);
    Launch L = L1(c);
    const int per = realspace_item_size(nt, cg.ncell);
    // octant items of dense cells (k_realspace.cu) need side > rc by a margin far
    // above the rounding of the cell centres
    const int oct_min =
        (per == 32 && sub >= 8 && cg.side >= rc * (1.0 + 1e-9)) ? realspace_octant_threshold() : 0;
    int64_t c_lo = 0, c_hi = -1;
    if (nparts > 1) {  // cells are (i dim + j) dim + k: x-slices are contiguous
        const int64_t plane = static_cast<int64_t>(cg.dim) * cg.dim;
        c_lo = plane * (static_cast<int64_t>(cg.dim) * part / nparts);
        c_hi = plane * (static_cast<int64_t>(cg.dim) * (part + 1) / nparts);
        if (nt > 0) FSE_CU(cudaMemsetAsync(d_uR, 0, sizeof(double) * 3 * nt, c->s1));
    }
    // one partial item per non-empty cell (octant), plus the full ones
    const int64_t max_items =
        std::min<int64_t>((oct_min > 0 ? 8 : 1) * cg.ncell, nt) + (nt + per - 1) / per;
    int32_t* items = buf<int32_t>(c, "rs_items", 2 * static_cast<size_t>(max_items));
    uint8_t* bucket = buf<uint8_t>(c, "rs_bucket", cg.ncell);
    int32_t* bwork = buf<int32_t>(c, "rs_bwork", 3 * realspace_work_buckets() + 1);
    int32_t* nitems = bwork + 3 * realspace_work_buckets();
    launch_realspace_items(L, src.start, tgt.start, cg.dim, cg.ncell, per, c_lo, c_hi, bucket,
                           bwork, items, nitems, oct_min, sub);
    FSE_CU(cudaEventRecord(c->ev[EV_RPAIR], c->s1));
    FSE_CU(cudaMemsetAsync(c->d_counts, 0, 2 * sizeof(unsigned long long), c->s1));
    if (nt > 0 && n > 0)
        launch_realspace(L, kind, cg, src.px, src.py, src.pz, src.fs, n, src.start, tgt.px, tgt.py,
                         tgt.pz, tgt.start, items, max_items, nitems, tgt.perm, xi, rc,
                         c->d_counts, d_uR, per, sub);
    else if (nt > 0)
        FSE_CU(cudaMemsetAsync(d_uR, 0, sizeof(double) * 3 * nt, c->s1));
}

double ev_sec(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    FSE_CU(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
}


void raise_flags(fse_cuda_ctx* c) {
    FSE_CU(cudaMemcpyAsync(c->h_flags, c->d_flags, 3 * sizeof(int), cudaMemcpyDeviceToHost,
                           c->s0));
    FSE_CU(cudaStreamSynchronize(c->s0));
    const int f = c->h_flags[0] | c->h_flags[1];
    if (f & FLAG_TARGET_BOX) invalid("fourier_sum: target outside [0,L]^3");
    if (f & FLAG_SUPPORT) invalid("spread/quadrature: point support exceeds grid");
    if (f & FLAG_COINCIDENT) throw Error(FSE_EDOMAIN, "direct_sum: coincident target/source point");
}

bool detect_tas_dev(fse_cuda_ctx* c, const double* a, const double* b, int64_t n, int64_t nt) {
    if (n != nt) return false;
    if (a == b || n == 0) return true;
    FSE_CU(cudaMemsetAsync(c->d_flags + 2, 0, sizeof(int), c->s0));
    k_not_equal<<<static_cast<unsigned>((3 * n + 255) / 256), 256, 0, c->s0>>>(a, b, 3 * n,
                                                                                c->d_flags + 2);
    FSE_LAUNCH_CHECK();
    ++c->launches;
    FSE_CU(cudaMemcpyAsync(c->h_flags + 2, c->d_flags + 2, sizeof(int), cudaMemcpyDeviceToHost,
                           c->s0));
    FSE_CU(cudaStreamSynchronize(c->s0));
    return c->h_flags[2] == 0;
}

// quadrature (ewald.cpp:349-391) of nt prepared targets from the real grid X
// into u (caller order via tg.perm): the TMA/DMMA slab gather (P <= 25), else
// the warp-group gather; EV_TPREP marks the end of the target preparation
void quadrature(fse_cuda_ctx* c, const GridParams& g, const Sorted& tg, int64_t nt,
                const double* X, double h3, double* u, bool record_events) {
    Launch L = L0(c);
    if (gather_slab_enabled(g)) {
        const int64_t nhalf = g.nkeys / 4;  // (coarse tile, z-half) pairs
        int32_t* scnt = buf<int32_t>(c, "scnt", nhalf + 1);
        int32_t* soff = buf<int32_t>(c, "soff", nhalf + 1);
        launch_slab_counts(L, g, tg.tstart, nhalf, scnt);
        exclusive_scan(c, c->s0, "s0", scnt, soff, nhalf + 1);
        const int64_t max_items = std::min<int64_t>(nhalf, nt) + (nt + 31) / 32;
        int32_t* sitems = buf<int32_t>(c, "sitems", 2 * static_cast<size_t>(max_items));
        launch_slab_fill(L, soff, nhalf, sitems);
        if (record_events) FSE_CU(cudaEventRecord(c->ev[EV_TPREP], c->s0));
        launch_gather_slab(L, g, tg.i0s, tg.w, tg.tstart, sitems, max_items, soff + nhalf, X,
                           tg.perm, h3, u);
    } else {
        if (g.nx < g.Mt) invalid("slab: the decomposition needs the tensor-core quadrature (P <= 25)");
        int32_t* gcnt = buf<int32_t>(c, "gcnt", g.nkeys + 1);
        int32_t* goff = buf<int32_t>(c, "goff", g.nkeys + 1);
        launch_group_counts(L, tg.tstart, g.nkeys, gcnt);
        exclusive_scan(c, c->s0, "s0", gcnt, goff, g.nkeys + 1);
        // upper bound on groups: one partial group per non-empty key + nt/8
        const int gk = gather_group_size();
        const int64_t max_groups = std::min<int64_t>(g.nkeys, nt) + (nt + gk - 1) / gk;
        int32_t* gkey = buf<int32_t>(c, "gkey", max_groups);
        launch_fill_groups(L, tg.tstart, goff, g.nkeys, gkey);
        if (record_events) FSE_CU(cudaEventRecord(c->ev[EV_TPREP], c->s0));
        launch_gather(L, g, tg.i0s, tg.w, tg.tstart, gkey, goff, max_groups, X, tg.perm, h3, u);
    }
}

// heavy-tiles-first order of the spread (k_spread.cu) on s0
const int32_t* spread_order(fse_cuda_ctx* c, const GridParams& g, const int32_t* tstart,
                            int64_t n) {
    const unsigned tiles = spread_tiles(g);
    if (tiles == 0) return nullptr;
    int32_t* order = buf<int32_t>(c, "sp_order", tiles);
    int32_t* light = buf<int32_t>(c, "sp_light", tiles + 1);
    int32_t* pos = buf<int32_t>(c, "sp_pos", tiles + 1);
    uint8_t* hbucket = buf<uint8_t>(c, "sp_hbucket", tiles);
    int32_t* bwork = buf<int32_t>(c, "sp_bwork", 97);
    launch_spread_flags(L0(c), g, tstart, n, light, hbucket, bwork);
    exclusive_scan(c, c->s0, "s0", light, pos, tiles);
    launch_spread_place(L0(c), g, light, pos, hbucket, bwork, order);
    return order;
}

// The whole hot path on device pointers.  u (caller order) = fourier (if
// want_f) + real (if want_r) + self (stokeslet, targets == sources, full sum).
void run_sum(fse_cuda_ctx* c, const fse_config* cfg, int kind, const double* d_pos,
             const double* d_str, int64_t n, double box_side, const double* d_tgt, int64_t nt,
             int tas_flag, const fse_green* green, double* d_u, fse_timings* tm, bool want_f,
             bool want_r) {
    check_kind(kind);
    if (n < 0 || nt < 0) invalid("negative point count");
    const int a = arity_of(kind);
    if (want_f) {
        check_cfg(cfg);
        check_green(cfg, kind, green);
        if (green->device != c->device) invalid("green lives on another device");
    }
    const bool tas = tas_flag < 0 ? detect_tas_dev(c, d_pos, d_tgt, n, nt) : tas_flag != 0;
    FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
    FSE_CU(cudaEventRecord(c->ev[EV_START], c->s0));
    FSE_CU(cudaStreamWaitEvent(c->s1, c->ev[EV_START], 0));

    double* uR = nullptr;
    // The FP64-bound real-space sum runs on stream s1.  With the Fourier part
    // it is enqueued after the source preparation (below), so the short,
    // latency-bound prep kernels do not queue behind its CTAs.
    auto enqueue_real = [&]() {
        uR = want_f ? buf<double>(c, "uR", 3 * nt) : d_u;
        FSE_CU(cudaEventRecord(c->ev[EV_R0], c->s1));
        real_part(c, kind, d_pos, d_str, n, box_side, cfg->xi, cfg->rc, d_tgt, nt, tas, uR);
        FSE_CU(cudaEventRecord(c->ev[EV_R1], c->s1));
    };
    if (want_r && !want_f) enqueue_real();

    double* uF = nullptr;
    if (want_f) {
        if (std::abs(box_side - cfg->L) > 1e-12 * cfg->L)
            invalid("spread: config box does not match system");
        const GridParams g = make_grid_params(*cfg);
        fft_xscale_check(fft_plan(c, g.D).host, kind);  // refuse before any work is queued
        Launch L = L0(c);
        double* qtab = buf<double>(c, "qtab", g.P);
        launch_quad_table(L, g, qtab);
        Sorted src = prep_points(c, g, "fs_", d_pos, d_str, a, n, tas ? 1 : 0, qtab);
        FSE_CU(cudaEventRecord(c->ev[EV_PREP], c->s0));
        const bool serial = !c->overlap;
        if (want_r && !serial) {
            FSE_CU(cudaStreamWaitEvent(c->s1, c->ev[EV_PREP], 0));
            enqueue_real();
        }
        // R: a compact Mt^3 real grids (every node is written by exactly one
        // spread tile, so no memset); B, C: pruned spectra (k_fft.cu)
        const int64_t Dh = g.Dh;
        double* X = buf<double>(c, "R", static_cast<size_t>(a) * g.comp);
        double2* Bs = buf<double2>(c, "B", static_cast<size_t>(a) * g.Mt * g.Mt * Dh);
        double2* Cs = buf<double2>(c, "C", static_cast<size_t>(a) * g.Mt * g.D * Dh);
        const FftPlanDev& fp = fft_plan(c, g.D);
        FSE_CU(cudaEventRecord(c->ev[EV_MEMSET], c->s0));
        const int32_t* order = spread_order(c, g, src.tstart, n);
        for (int c0 = 0; c0 < a; c0 += 3)
            launch_spread(L, g, src.i0s, src.w, src.fs, n, a, c0, src.tstart, X, order);
        FSE_CU(cudaEventRecord(c->ev[EV_SPREAD], c->s0));
        launch_fft_forward_zy(L, fp.host, fp.tw, g, a, X, Bs, Cs);
        FSE_CU(cudaEventRecord(c->ev[EV_FFT1], c->s0));
        launch_fft_xscale(L, fp.host, fp.tw, g, kind, green->d_half, Cs,
                          buf<double>(c, "ex_axis", g.D));
        FSE_CU(cudaEventRecord(c->ev[EV_SCALE], c->s0));
        launch_fft_inverse_yz(L, fp.host, fp.tw, g, a, Cs, Bs, X);
        FSE_CU(cudaEventRecord(c->ev[EV_FFT2], c->s0));

        Sorted tg = tas ? src : prep_points(c, g, "ft_", d_tgt, nullptr, 0, nt, 1, qtab);
        uF = want_r ? buf<double>(c, "uF", 3 * nt) : d_u;
        const double h3 = g.h * g.h * g.h;  // prefac is folded into the x weights
        quadrature(c, g, tg, nt, X, h3, uF, true);
        FSE_CU(cudaEventRecord(c->ev[EV_QUAD], c->s0));
        if (want_r && serial) {
            FSE_CU(cudaStreamWaitEvent(c->s1, c->ev[EV_QUAD], 0));
            enqueue_real();
        }
    }

    if (want_r) {
        FSE_CU(cudaEventRecord(c->ev[EV_JOIN], c->s1));
        FSE_CU(cudaStreamWaitEvent(c->s0, c->ev[EV_JOIN], 0));
    }
    if (want_f && want_r) {
        const bool self = tas && kind == FSE_STOKESLET;
        launch_epilogue(L0(c), nt, uF, uR, self ? d_str : nullptr,
                        self ? -4.0 * cfg->xi / std::sqrt(M_PI) : 0.0, d_u);
    }
    FSE_CU(cudaEventRecord(c->ev[EV_END], c->s0));
    raise_flags(c);
    for (double& v : c->kms) v = 0;
    auto ms = [&](int a0, int b0) { return 1e3 * ev_sec(c->ev[a0], c->ev[b0]); };
    if (want_f) {
        c->kms[0] = ms(EV_START, EV_PREP);
        c->kms[1] = ms(EV_PREP, EV_MEMSET);
        c->kms[2] = ms(EV_MEMSET, EV_SPREAD);
        c->kms[3] = ms(EV_SPREAD, EV_FFT1);
        c->kms[4] = ms(EV_FFT1, EV_SCALE);
        c->kms[5] = ms(EV_SCALE, EV_FFT2);
        c->kms[6] = ms(EV_FFT2, EV_TPREP);
        c->kms[7] = ms(EV_TPREP, EV_QUAD);
    }
    if (want_r) {
        c->kms[8] = ms(EV_R0, EV_RPAIR);
        c->kms[9] = ms(EV_RPAIR, EV_R1);
    }
    c->kms[10] = ms(EV_START, EV_END);
    if (tm) {
        FSE_CU(cudaEventSynchronize(c->ev[EV_END]));
        if (want_f) {
            tm->spread += ev_sec(c->ev[EV_START], c->ev[EV_SPREAD]);
            tm->fft += ev_sec(c->ev[EV_SPREAD], c->ev[EV_FFT1]) +
                       ev_sec(c->ev[EV_SCALE], c->ev[EV_FFT2]);
            tm->scale += ev_sec(c->ev[EV_FFT1], c->ev[EV_SCALE]);
            tm->quadrature += ev_sec(c->ev[EV_FFT2], c->ev[EV_QUAD]);
        }
        if (want_r) tm->realspace += ev_sec(c->ev[EV_R0], c->ev[EV_R1]);
        tm->total += ev_sec(c->ev[EV_START], c->ev[EV_END]);
    }
}

// host-pointer front end: H2D (pinned or pageable), run, D2H
bool host_equal(const double* a, const double* b, int64_t n) {
    if (a == b) return true;
    for (int64_t q = 0; q < 3 * n; ++q)
        if (!(a[q] == b[q])) return false;
    return true;
}

void h2d(fse_cuda_ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes) FSE_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s0));
}

void d2h(fse_cuda_ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes) FSE_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->s0));
    FSE_CU(cudaStreamSynchronize(c->s0));
}

void run_sum_host(fse_cuda_ctx* c, const fse_config* cfg, int kind, const double* pos,
                  const double* str, int64_t n, double box_side, const double* tgt, int64_t nt,
                  int tas_flag, const fse_green* green, double* u, fse_timings* tm, bool want_f,
                  bool want_r) {
    check_kind(kind);
    if (n < 0 || nt < 0) invalid("negative point count");
    if ((n > 0 && (!pos || !str)) || (nt > 0 && (!tgt || !u))) invalid("null pointer");
    const int a = arity_of(kind);
    const bool tas = tas_flag < 0 ? (n == nt && host_equal(pos, tgt, n)) : tas_flag != 0;
    double* d_pos = buf<double>(c, "in_pos", 3 * n);
    double* d_str = buf<double>(c, "in_str", a * n);
    double* d_tgt = tas ? d_pos : buf<double>(c, "in_tgt", 3 * nt);
    double* d_u = buf<double>(c, "in_u", 3 * nt);
    // positions (and targets) on s0, strengths on s1: the support keys and sort
    // of the positions overlap the strengths' transfer (pinned host memory)
    h2d(c, d_pos, pos, sizeof(double) * 3 * n);
    if (n > 0) {
        FSE_CU(cudaMemcpyAsync(d_str, str, sizeof(double) * a * n, cudaMemcpyHostToDevice, c->s1));
        FSE_CU(cudaEventRecord(c->ev[EV_H2D], c->s1));
        c->str_pending = true;
    }
    if (!tas) h2d(c, d_tgt, tgt, sizeof(double) * 3 * nt);
    struct Clear {
        fse_cuda_ctx* c;
        ~Clear() { c->str_pending = false; }
    } clear{c};
    run_sum(c, cfg, kind, d_pos, d_str, n, box_side, d_tgt, nt, tas ? 1 : 0, green, d_u, tm,
            want_f, want_r);
    d2h(c, u, d_u, sizeof(double) * 3 * nt);
}

// ---------------------------------------------------------------- Green
fse_green* new_green(fse_cuda_ctx* c, int kind, double Ltilde, int Mt, double h, double R) {
    auto* g = new fse_green;
    g->kind = kind;
    g->Ltilde = Ltilde;
    g->Mtilde = Mt;
    g->h = h;
    g->R = R;
    g->device = c->device;
    g->d_half = nullptr;
    const int64_t D = 2 * static_cast<int64_t>(Mt);
    cudaError_t e = cudaMalloc(&g->d_half, sizeof(double) * D * D * (D / 2 + 1));
    if (e != cudaSuccess) {
        delete g;
        throw_cuda(e, "cudaMalloc(green)", __FILE__, __LINE__);
    }
    return g;
}

// One device buffer owned for the duration of a call (one-off scratch that must
// not stay cached in the context).
struct DevScratch {
    void* p = nullptr;
    DevScratch() = default;
    DevScratch(const DevScratch&) = delete;
    DevScratch& operator=(const DevScratch&) = delete;
    ~DevScratch() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* alloc(size_t count) {
        if (p) FSE_CU(cudaFree(p));
        p = nullptr;
        FSE_CU(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        return static_cast<T*>(p);
    }
};

struct Cublas {
    cublasHandle_t h = nullptr;
    ~Cublas() {
        if (h) cublasDestroy(h);
    }
};

#define FSE_CUBLAS(x)                                                                  \
    do {                                                                               \
        cublasStatus_t st_ = (x);                                                      \
        if (st_ != CUBLAS_STATUS_SUCCESS) {                                            \
            char b_[256];                                                              \
            std::snprintf(b_, sizeof b_, "cuBLAS error %d in %s", static_cast<int>(st_), #x); \
            throw Error(st_ == CUBLAS_STATUS_ALLOC_FAILED ? FSE_ENOMEM : FSE_ECUDA, b_);    \
        }                                                                              \
    } while (0)

// even-sequence cosine matrix, row-major [nout][nin]:
//   C[n][q] = w_q cos(2 pi q n / len) * scale, w_q = 1 at q = 0 and q = len/2, else 2
// (the length-len DFT of a real sequence even in q, evaluated at n, folded onto
// q in [0, len/2]); angles reduced exactly in integers, cosl in long double.
std::vector<double> cos_matrix(int nout, int nin, int len, long double scale) {
    std::vector<double> m(static_cast<size_t>(nout) * nin);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int n = 0; n < nout; ++n)
        for (int q = 0; q < nin; ++q) {
            const int64_t r = (static_cast<int64_t>(q) * n) % len;
            const long double w = (q == 0 || 2 * q == len) ? 1.0L : 2.0L;
            m[static_cast<size_t>(n) * nin + q] =
                static_cast<double>(w * scale * cosl(two_pi * static_cast<long double>(r) / len));
        }
    return m;
}

// One separable pass: out[n][ab] = sum_q Cm[n][q] in[ab][q] (row-major); the
// summed axis is the fastest of `in` and becomes the slowest of `out`, so three
// passes rotate the axes back to their original order.  A plain DGEMM (cuBLAS).
void cos_pass(cublasHandle_t hb, const double* in, int64_t AB, int K, const double* Cm, int N,
              double* out) {
    const double one = 1.0, zero = 0.0;
    FSE_CUBLAS(cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(AB), N, K, &one, in,
                           K, Cm, K, &zero, out, static_cast<int>(AB)));
}

// greens.cpp:48-113 on the GPU, pruned and symmetry-aware.
// The reference fills Ghat(|k|) on the sM^3 wavenumber grid, inverse-FFTs it,
// keeps the real (2 Mt)^3 window of offsets [-Mt, Mt) and forward-FFTs that.
// Ghat is real and even in every axis, so the inverse DFT is a product of
// cosine sums over q in [0, sM/2] and is only needed at |offset| <= Mt; the
// windowed grid is again real and even, so the forward DFT is a product of
// cosine sums over n in [0, Mt] evaluated at k in [0, D/2]:
//   octant Ghat (sM/2+1)^3 -> 3 cosine passes -> g (Mt+1)^3 -> 3 cosine passes
//   -> T (D/2+1)^3 -> unfolded to the D x D x (D/2+1) half table.
// Six DGEMMs on arrays of at most (sM/2+1)^3 doubles instead of an sM^3 grid
// (cfg5: 4.4 GB instead of 35 GB; cfg5t: 13 GB instead of 105 GB).
fse_green* green_precompute(fse_cuda_ctx* c, int gkind, double Ltilde, int Mt, double sf) {
    const double sf_min = 1.0 + std::sqrt(3.0);
    if (!(Ltilde > 0) || Mt < 1) invalid("precompute_mollified_green: bad domain");
    if (sf < sf_min - 1e-12) invalid("precompute_mollified_green: sf below 1 + sqrt(3)");
    if (gkind != FSE_HARMONIC && gkind != FSE_BIHARMONIC) invalid("unknown green kind");
    const double h = Ltilde / Mt;
    const double R = std::sqrt(3.0) * Ltilde;
    int sM = static_cast<int>(std::ceil(sf * Mt));
    if (sM % 2 != 0) ++sM;
    const double dk = 2.0 * M_PI / (sM * h);
    const int D = 2 * Mt;
    const int nq = sM / 2 + 1, nm = Mt + 1;  // D/2 + 1 == Mt + 1
    Launch L = L0(c);
    fse_green* g = new_green(c, gkind, Ltilde, Mt, h, R);
    try {
        Cublas cb;
        FSE_CUBLAS(cublasCreate(&cb.h));
        FSE_CUBLAS(cublasSetStream(cb.h, c->s0));
        FSE_CUBLAS(cublasSetMathMode(cb.h, CUBLAS_DEFAULT_MATH));
        // inverse transform matrix [n][q] (1/sM per axis = the 1/sM^3 of fft3d_inverse)
        // and forward matrix [k][n] over the D-periodic windowed grid
        const std::vector<double> ci = cos_matrix(nm, nq, sM, 1.0L / sM);
        const std::vector<double> cf = cos_matrix(nm, nm, D, 1.0L);
        DevScratch sci, scf, sa, sb;
        double* dci = sci.alloc<double>(ci.size());
        double* dcf = scf.alloc<double>(cf.size());
        FSE_CU(cudaMemcpyAsync(dci, ci.data(), ci.size() * sizeof(double),
                               cudaMemcpyHostToDevice, c->s0));
        FSE_CU(cudaMemcpyAsync(dcf, cf.data(), cf.size() * sizeof(double),
                               cudaMemcpyHostToDevice, c->s0));
        const int64_t q3 = static_cast<int64_t>(nq) * nq * nq;
        const int64_t big = std::max<int64_t>(q3, static_cast<int64_t>(nm) * nm * nq);
        double* A = sa.alloc<double>(static_cast<size_t>(big));
        double* B = sb.alloc<double>(static_cast<size_t>(static_cast<int64_t>(nm) * nq * nq));
        launch_green_octant(L, gkind, sM, dk, R, A);                                  // [qx][qy][qz]
        cos_pass(cb.h, A, static_cast<int64_t>(nq) * nq, nq, dci, nm, B);           // [nz][qx][qy]
        cos_pass(cb.h, B, static_cast<int64_t>(nm) * nq, nq, dci, nm, A);           // [ny][nz][qx]
        cos_pass(cb.h, A, static_cast<int64_t>(nm) * nm, nq, dci, nm, B);           // [nx][ny][nz]
        cos_pass(cb.h, B, static_cast<int64_t>(nm) * nm, nm, dcf, nm, A);           // [kz][nx][ny]
        cos_pass(cb.h, A, static_cast<int64_t>(nm) * nm, nm, dcf, nm, B);           // [ky][kz][nx]
        cos_pass(cb.h, B, static_cast<int64_t>(nm) * nm, nm, dcf, nm, A);           // [kx][ky][kz]
        launch_green_unfold(L, Mt, A, g->d_half);
        FSE_CU(cudaStreamSynchronize(c->s0));
    } catch (...) {
        cudaFree(g->d_half);
        delete g;
        throw;
    }
    return g;
}

}  // namespace

// ======================================================================= C-ABI
extern "C" {

int fse_cuda_abi_version(void) { return FSE_CUDA_ABI_VERSION; }
int fse_arity(int kind) { return arity_of(kind); }

fse_status fse_cuda_create(int device, fse_cuda_ctx** out) {
    if (!out) return FSE_EINVAL;
    *out = nullptr;
    auto* c = new fse_cuda_ctx;
    c->device = device;
    try {
        FSE_CU(cudaSetDevice(device));
        // FSE_S1_PRIORITY=high|low: scheduling priority of the real-space stream
        // relative to the Fourier stream (default: equal)
        int lo = 0, hi = 0;
        FSE_CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const char* pr = std::getenv("FSE_S1_PRIORITY");
        const int p1 = pr && std::strcmp(pr, "high") == 0 ? hi : lo;
        const int p0 = pr && std::strcmp(pr, "low") == 0 ? hi : lo;
        FSE_CU(cudaStreamCreateWithPriority(&c->s0, cudaStreamNonBlocking, p0));
        FSE_CU(cudaStreamCreateWithPriority(&c->s1, cudaStreamNonBlocking, p1));
        for (auto& e : c->ev) FSE_CU(cudaEventCreate(&e));
        for (auto& e : c->mark) FSE_CU(cudaEventCreate(&e));
        FSE_CU(cudaMalloc(&c->d_flags, 8 * sizeof(int)));
        FSE_CU(cudaMalloc(&c->d_counts, 2 * sizeof(unsigned long long)));
        FSE_CU(cudaMemset(c->d_counts, 0, 2 * sizeof(unsigned long long)));
        FSE_CU(cudaMallocHost(&c->h_flags, 8 * sizeof(int)));
    } catch (const Error& e) {
        fse_status st = e.code;
        fse_cuda_destroy(c);
        return st;
    }
    *out = c;
    return FSE_OK;
}

void fse_cuda_destroy(fse_cuda_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    release_plans(c);
    for (auto& kv : c->bufs)
        if (kv.second.p) cudaFree(kv.second.p);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->mark)
        if (e) cudaEventDestroy(e);
    if (c->d_flags) cudaFree(c->d_flags);
    if (c->d_counts) cudaFree(c->d_counts);
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->s0) cudaStreamDestroy(c->s0);
    if (c->s1) cudaStreamDestroy(c->s1);
    delete c;
}

const char* fse_cuda_last_error(const fse_cuda_ctx* c) { return c ? c->err.c_str() : "null context"; }

fse_status fse_cuda_trim(fse_cuda_ctx* c) {
    return api(c, [&] {
        sync_all(c);
        release_plans(c);
        for (auto& kv : c->bufs)
            if (kv.second.p) FSE_CU(cudaFree(kv.second.p));
        c->bufs.clear();
    });
}

fse_status fse_cuda_host_alloc(fse_cuda_ctx* c, size_t bytes, void** out) {
    return api(c, [&] { FSE_CU(cudaMallocHost(out, std::max<size_t>(bytes, 1))); });
}
void fse_cuda_host_free(void* p) {
    if (p) cudaFreeHost(p);
}
fse_status fse_cuda_dev_alloc(fse_cuda_ctx* c, size_t bytes, void** out) {
    return api(c, [&] { FSE_CU(cudaMalloc(out, std::max<size_t>(bytes, 1))); });
}
void fse_cuda_dev_free(fse_cuda_ctx* c, void* p) {
    if (c && p) {
        cudaSetDevice(c->device);
        cudaFree(p);
    }
}
fse_status fse_cuda_memcpy(fse_cuda_ctx* c, void* dst, const void* src, size_t bytes) {
    return api(c, [&] {
        FSE_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->s0));
        FSE_CU(cudaStreamSynchronize(c->s0));
    });
}
fse_status fse_cuda_mark(fse_cuda_ctx* c) {
    return api(c, [&] {
        FSE_CU(cudaEventRecord(c->mark[c->mark_n & 1], c->s0));
        ++c->mark_n;
    });
}
fse_status fse_cuda_elapsed_ms(fse_cuda_ctx* c, double* ms) {
    return api(c, [&] {
        if (c->mark_n < 2) invalid("need two marks");
        cudaEvent_t a = c->mark[(c->mark_n - 2) & 1], b = c->mark[(c->mark_n - 1) & 1];
        FSE_CU(cudaEventSynchronize(b));
        float f = 0;
        FSE_CU(cudaEventElapsedTime(&f, a, b));
        *ms = f;
    });
}
uint64_t fse_cuda_launch_count(const fse_cuda_ctx* c) { return c ? c->launches : 0; }

fse_status fse_cuda_fp64_peak(fse_cuda_ctx* c, double* tflops) {
    return api(c, [&] {
        if (!tflops) invalid("null pointer");
        *tflops = measure_dfma_tflops(L0(c), buf<double>(c, "peak_scratch", 1));
    });
}

fse_status fse_cuda_realspace_counts(fse_cuda_ctx* c, uint64_t* candidates, uint64_t* pairs) {
    return api(c, [&] {
        if (!candidates || !pairs) invalid("null pointer");
        unsigned long long h[2] = {0, 0};
        FSE_CU(cudaStreamSynchronize(c->s1));
        FSE_CU(cudaMemcpy(h, c->d_counts, sizeof h, cudaMemcpyDeviceToHost));
        *candidates = h[0];
        *pairs = h[1];
    });
}

fse_status fse_cuda_set_overlap(fse_cuda_ctx* c, int on) {
    return api(c, [&] { c->overlap = on != 0; });
}

fse_status fse_cuda_kernel_ms(fse_cuda_ctx* c, double* out, int n) {
    return api(c, [&] {
        if (!out) invalid("null pointer");
        for (int k = 0; k < n && k < NKMS; ++k) out[k] = c->kms[k];
    });
}

// ewald.cpp:103-134
fse_status fse_make_config(double L, double xi, double rc, int M, int P, double sf,
                           fse_config* out, char* err, size_t errlen) {
    auto fail = [&](const char* m) {
        if (err && errlen) std::snprintf(err, errlen, "%s", m);
        return FSE_EINVAL;
    };
    if (!out) return fail("null output");
    if (!(L > 0) || !(xi > 0) || !(rc > 0) || M < 1 || P < 2)
        return fail("make_config: all parameters must be positive");
    if (P % 2 != 0) return fail("make_config: P must be even");
    fse_config c;
    std::memset(&c, 0, sizeof c);
    c.L = L;
    c.xi = xi;
    c.rc = rc;
    c.M = M;
    c.P = P;
    c.h = L / M;
    c.d = c.h * P;
    c.m = 0.976 * std::sqrt(M_PI * P);
    c.eta = (xi * c.d / c.m) * (xi * c.d / c.m);
    double raw = c.d;
    if (c.eta < 1.0) raw = std::max(c.d, std::sqrt(2.0 * (1.0 - c.eta)) * c.m / xi);
    const int pad = static_cast<int>(std::ceil(raw / c.h - 1e-12));
    c.deltaL = pad * c.h;
    c.Mtilde = M + pad;
    c.Ltilde = c.Mtilde * c.h;
    c.kinf = M_PI * c.Mtilde / c.Ltilde;
    c.R = std::sqrt(3.0) * c.Ltilde;
    c.sf = sf > 0 ? sf : 1.0 + std::sqrt(3.0);
    if (c.sf < 1.0 + std::sqrt(3.0) - 1e-12) return fail("make_config: sf below 1 + sqrt(3)");
    if (P > c.Mtilde) return fail("make_config: Gaussian support exceeds grid");
    *out = c;
    return FSE_OK;
}

fse_status fse_cuda_green_precompute(fse_cuda_ctx* c, int green_kind, double Ltilde, int Mtilde,
                                     double sf, fse_green** out) {
    return api(c, [&] {
        if (!out) invalid("null output");
        *out = green_precompute(c, green_kind, Ltilde, Mtilde, sf);
    });
}

fse_status fse_cuda_green_upload(fse_cuda_ctx* c, int green_kind, double Ltilde, int Mtilde,
                                 double h, double R, const double* full, fse_green** out) {
    return api(c, [&] {
        if (!out || !full) invalid("null pointer");
        if (Mtilde < 1 || !(Ltilde > 0)) invalid("bad green geometry");
        if (green_kind != FSE_HARMONIC && green_kind != FSE_BIHARMONIC)
            invalid("unknown green kind");
        fse_green* g = new_green(c, green_kind, Ltilde, Mtilde, h, R);
        try {
            const int D = 2 * Mtilde;
            const size_t n = static_cast<size_t>(D) * D * D;
            DevScratch scratch;
            double* tmp = scratch.alloc<double>(n);
            h2d(c, tmp, full, n * sizeof(double));
            launch_green_full_to_half(L0(c), D, tmp, g->d_half);
            FSE_CU(cudaStreamSynchronize(c->s0));
        } catch (...) {
            cudaFree(g->d_half);
            delete g;
            throw;
        }
        *out = g;
    });
}

fse_status fse_cuda_green_download(fse_cuda_ctx* c, const fse_green* g, double* full) {
    return api(c, [&] {
        if (!g || !full) invalid("null pointer");
        const int D = 2 * g->Mtilde;
        const size_t n = static_cast<size_t>(D) * D * D;
        DevScratch scratch;
        double* tmp = scratch.alloc<double>(n);
        launch_green_half_to_full(L0(c), D, g->d_half, tmp);
        d2h(c, full, tmp, n * sizeof(double));
    });
}

// fse::freespace_solve (greens.cpp:115-139): zero-pad the M~^3 right-hand side
// to D^3, multiply its transform by the Green's table, transform back and keep
// the M~^3 window -- the hot path's pruned FFT passes with one component and
// the scalar multiplier (G / D^3; G is real and even, so the real-to-complex
// transforms are exact).
fse_status fse_cuda_freespace_solve(fse_cuda_ctx* c, const fse_green* green, const double* rhs,
                                    double* out) {
    return api(c, [&] {
        if (!green || !rhs || !out) invalid("null pointer");
        if (green->device != c->device) invalid("green lives on another device");
        GridParams g{};
        g.Mt = green->Mtilde;
        g.D = 2 * g.Mt;
        g.Dh = g.D / 2 + 1;
        g.P = 2;
        g.rowp = g.Mt;
        g.plane = static_cast<int64_t>(g.Mt) * g.Mt;
        g.comp = static_cast<int64_t>(g.Mt) * g.plane;
        g.h = green->h;
        g.dk = M_PI / green->Ltilde;
        g.invD3 = 1.0 / (static_cast<double>(g.D) * g.D * g.D);  // fft.cpp:34
        g.x_lo = 0;
        g.nx = g.nxs = g.Mt;
        g.ky_lo = 0;
        g.nky = g.nkys = g.D;
        const size_t vol = static_cast<size_t>(g.comp);
        double* R = buf<double>(c, "R", vol);
        double2* Bs = buf<double2>(c, "B", static_cast<size_t>(g.Mt) * g.Mt * g.Dh);
        double2* Cs = buf<double2>(c, "C", static_cast<size_t>(g.Mt) * g.D * g.Dh);
        FSE_CU(cudaMemcpyAsync(R, rhs, vol * sizeof(double), cudaMemcpyHostToDevice, c->s0));
        const FftPlanDev& fp = fft_plan(c, g.D);
        Launch L = L0(c);
        launch_fft_forward_zy(L, fp.host, fp.tw, g, 1, R, Bs, Cs);
        launch_fft_xscale(L, fp.host, fp.tw, g, KIND_SCALAR_X, green->d_half, Cs,
                          buf<double>(c, "ex_axis", g.D));
        launch_fft_inverse_yz(L, fp.host, fp.tw, g, 1, Cs, Bs, R, 1);
        d2h(c, out, R, vol * sizeof(double));
    });
}

fse_status fse_cuda_green_info(const fse_green* g, int* kind, double* Ltilde, double* h,
                               double* R, int* Mtilde) {
    if (!g) return FSE_EINVAL;
    if (kind) *kind = g->kind;
    if (Ltilde) *Ltilde = g->Ltilde;
    if (h) *h = g->h;
    if (R) *R = g->R;
    if (Mtilde) *Mtilde = g->Mtilde;
    return FSE_OK;
}

void fse_cuda_green_free(fse_green* g) {
    if (!g) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    cudaFree(g->d_half);
    cudaSetDevice(cur);
    delete g;
}

// greens.cpp:141-171: "FSEG", u32 version 1, u8 kind, f64 Ltilde/h/R, u64 x3 extents, payload
fse_status fse_cuda_green_save(fse_cuda_ctx* c, const fse_green* g, const char* path) {
    return api(c, [&] {
        if (!g || !path) invalid("null pointer");
        const uint64_t D = 2 * static_cast<uint64_t>(g->Mtilde);
        std::vector<double> full(D * D * D);
        DevScratch scratch;  // one-off D^3 staging, not cached in the context
        double* tmp = scratch.alloc<double>(full.size());
        launch_green_half_to_full(L0(c), static_cast<int>(D), g->d_half, tmp);
        d2h(c, full.data(), tmp, full.size() * sizeof(double));
        std::ofstream os(path, std::ios::binary);
        if (!os) throw Error(FSE_ERUNTIME, std::string("save_mollified_green: cannot open ") + path);
        const uint32_t version = 1;
        const uint8_t kind = static_cast<uint8_t>(g->kind);
        os.write("FSEG", 4);
        os.write(reinterpret_cast<const char*>(&version), 4);
        os.write(reinterpret_cast<const char*>(&kind), 1);
        os.write(reinterpret_cast<const char*>(&g->Ltilde), 8);
        os.write(reinterpret_cast<const char*>(&g->h), 8);
        os.write(reinterpret_cast<const char*>(&g->R), 8);
        for (int k = 0; k < 3; ++k) os.write(reinterpret_cast<const char*>(&D), 8);
        os.write(reinterpret_cast<const char*>(full.data()),
                 static_cast<std::streamsize>(full.size() * sizeof(double)));
        if (!os) throw Error(FSE_ERUNTIME, std::string("save_mollified_green: write failed for ") + path);
    });
}

// greens.cpp:173-203
fse_status fse_cuda_green_load(fse_cuda_ctx* c, const char* path, fse_green** out) {
    return api(c, [&] {
        if (!path || !out) invalid("null pointer");
        std::ifstream is(path, std::ios::binary);
        if (!is) throw Error(FSE_ERUNTIME, std::string("load_mollified_green: cannot open ") + path);
        char magic[4];
        is.read(magic, 4);
        if (!is || std::memcmp(magic, "FSEG", 4) != 0)
            throw Error(FSE_ERUNTIME, std::string("load_mollified_green: bad magic in ") + path);
        uint32_t version = 0;
        is.read(reinterpret_cast<char*>(&version), 4);
        if (version != 1) throw Error(FSE_ERUNTIME, "load_mollified_green: unsupported version");
        uint8_t kind = 0;
        double Lt = 0, h = 0, R = 0;
        uint64_t d[3] = {0, 0, 0};
        is.read(reinterpret_cast<char*>(&kind), 1);
        is.read(reinterpret_cast<char*>(&Lt), 8);
        is.read(reinterpret_cast<char*>(&h), 8);
        is.read(reinterpret_cast<char*>(&R), 8);
        is.read(reinterpret_cast<char*>(d), 24);
        if (!is || d[0] != d[1] || d[0] != d[2] || d[0] == 0 || d[0] % 2 != 0)
            throw Error(FSE_ERUNTIME, "load_mollified_green: bad extents");
        // the reference stores whatever byte it finds (greens.cpp:189); a table of
        // an unknown kind could never pass check_green, so reject it here
        if (kind != FSE_HARMONIC && kind != FSE_BIHARMONIC)
            throw Error(FSE_ERUNTIME, "load_mollified_green: unknown green kind");
        std::vector<double> full(d[0] * d[1] * d[2]);
        is.read(reinterpret_cast<char*>(full.data()),
                static_cast<std::streamsize>(full.size() * sizeof(double)));
        if (!is) throw Error(FSE_ERUNTIME, "load_mollified_green: truncated payload");
        const int Mt = static_cast<int>(d[0] / 2);
        fse_green* g = new_green(c, kind, Lt, Mt, h, R);
        DevScratch scratch;
        double* tmp = scratch.alloc<double>(full.size());
        h2d(c, tmp, full.data(), full.size() * sizeof(double));
        launch_green_full_to_half(L0(c), static_cast<int>(d[0]), tmp, g->d_half);
        FSE_CU(cudaStreamSynchronize(c->s0));
        *out = g;
    });
}

fse_status fse_cuda_total_sum(fse_cuda_ctx* c, const fse_config* cfg, int kind, const double* pos,
                              const double* str, int64_t n, double box_side, const double* targets,
                              int64_t nt, int tas, const fse_green* green, double* u,
                              fse_timings* tm) {
    return api(c, [&] {
        run_sum_host(c, cfg, kind, pos, str, n, box_side, targets, nt, tas, green, u, tm, true,
                     true);
    });
}

fse_status fse_cuda_total_sum_dev(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                  const double* d_pos, const double* d_str, int64_t n,
                                  double box_side, const double* d_tgt, int64_t nt, int tas,
                                  const fse_green* green, double* d_u, fse_timings* tm) {
    return api(c, [&] {
        run_sum(c, cfg, kind, d_pos, d_str, n, box_side, d_tgt, nt, tas, green, d_u, tm, true,
                true);
    });
}

// ------------------------------------------------------------------ z-slabs
// slab r of G owns x-planes [x_lo, x_lo + nx) of the M~ grid and the
// ky rows [ky_lo, ky_lo + nky) of the x-pass.  Every rank holds all points; the
// exchanges are the two spectrum all-to-alls and one sum of the per-rank
// partial velocities (the caller runs them, e.g. NCCL via torch.distributed).
namespace {

GridParams slab_params(const fse_config* cfg, int rank, int nslabs) {
    check_cfg(cfg);
    if (nslabs < 1 || rank < 0 || rank >= nslabs) invalid("slab: need 0 <= rank < nslabs");
    if (nslabs > kMaxSlabs) invalid("slab: at most 16 slabs");
    GridParams g = make_grid_params(*cfg);
    set_slab(g, rank, nslabs);
    if (nslabs > 1 && !gather_slab_enabled(g))
        invalid("slab: the decomposition needs the tensor-core quadrature (P <= 25)");
    return g;
}

int64_t slab_block_elems(const GridParams& g, int a) {
    return static_cast<int64_t>(a) * g.nxs * g.nkys * g.Dh;
}

}  // namespace

fse_status fse_cuda_slab_info(const fse_config* cfg, int kind, int rank, int nslabs,
                              fse_slab_info* out) {
    try {
        check_kind(kind);
        if (!out) invalid("null pointer");
        const GridParams g = slab_params(cfg, rank, nslabs);
        out->x_lo = g.x_lo;
        out->nx = g.nx;
        out->nxs = g.nxs;
        out->ky_lo = g.ky_lo;
        out->nky = g.nky;
        out->nkys = g.nkys;
        out->block_complex = slab_block_elems(g, arity_of(kind));
        return FSE_OK;
    } catch (const Error& e) {
        return e.code;
    } catch (...) {
        return FSE_ERUNTIME;
    }
}

namespace {

// block table of a peer-direct exchange: block s -> dst_bufs[s] at block
// `rank`, uploaded to a small device array (stream-ordered)
BlockDest peer_blocks(fse_cuda_ctx* c, const GridParams& g, int a, int rank, int nslabs,
                      double* const* dst_bufs, const char* name) {
    if (!dst_bufs) invalid("null pointer");
    if (nslabs > kMaxSlabs) invalid("slab: at most 16 slabs");
    const int64_t block = slab_block_elems(g, a);
    double2* h[kMaxSlabs] = {};
    for (int s = 0; s < nslabs; ++s) {
        if (!dst_bufs[s]) invalid("null peer buffer");
        h[s] = reinterpret_cast<double2*>(dst_bufs[s]) + rank * block;
    }
    double2** d_tab = buf<double2*>(c, name, kMaxSlabs);
    FSE_CU(cudaMemcpyAsync(d_tab, h, sizeof h, cudaMemcpyHostToDevice, c->s0));
    BlockDest d{};
    d.tab = d_tab;
    return d;
}

void slab_forward_impl(fse_cuda_ctx* c, const fse_config* cfg, int kind, const double* d_pos,
                       const double* d_str, int64_t n, int rank, int nslabs, double* d_spec,
                       double* const* dst_bufs) {
    check_kind(kind);
    if ((!d_spec && !dst_bufs) || (n > 0 && (!d_pos || !d_str))) invalid("null pointer");
    const int a = arity_of(kind);
    const GridParams g = slab_params(cfg, rank, nslabs);
    BlockDest peers{};
    if (dst_bufs) peers = peer_blocks(c, g, a, rank, nslabs, dst_bufs, "peer_fwd");
    FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
    Launch L = L0(c);
    double* qtab = buf<double>(c, "qtab", g.P);
    launch_quad_table(L, g, qtab);
    Sorted src = prep_points(c, g, "fs_", d_pos, d_str, a, n, 0, qtab);
    double* X = buf<double>(c, "R", static_cast<size_t>(a) * g.comp);
    double2* Bs = buf<double2>(c, "B", static_cast<size_t>(a) * g.nx * g.Mt * g.Dh);
    const FftPlanDev& fp = fft_plan(c, g.D);
    for (int c0 = 0; c0 < a; c0 += 3)
        launch_spread(L, g, src.i0s, src.w, src.fs, n, a, c0, src.tstart, X);
    launch_fft_forward_zy(L, fp.host, fp.tw, g, a, X, Bs, reinterpret_cast<double2*>(d_spec),
                          dst_bufs ? &peers : nullptr);
    raise_flags(c);  // synchronises s0
}

void slab_scale_impl(fse_cuda_ctx* c, const fse_config* cfg, int kind, const fse_green* green,
                     int rank, int nslabs, double* d_spec, double* const* dst_bufs) {
    check_kind(kind);
    if (!d_spec) invalid("null pointer");
    const GridParams g = slab_params(cfg, rank, nslabs);
    check_green(cfg, kind, green);
    if (green->device != c->device) invalid("green lives on another device");
    BlockDest peers{};
    if (dst_bufs) peers = peer_blocks(c, g, arity_of(kind), rank, nslabs, dst_bufs, "peer_bwd");
    const FftPlanDev& fp = fft_plan(c, g.D);
    launch_fft_xscale(L0(c), fp.host, fp.tw, g, kind, green->d_half,
                      reinterpret_cast<double2*>(d_spec), buf<double>(c, "ex_axis", g.D),
                      dst_bufs ? &peers : nullptr);
    FSE_CU(cudaStreamSynchronize(c->s0));
}

}  // namespace

fse_status fse_cuda_slab_forward(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                 const double* d_pos, const double* d_str, int64_t n, int rank,
                                 int nslabs, double* d_spec) {
    return api(c, [&] {
        if (!d_spec) invalid("null pointer");
        slab_forward_impl(c, cfg, kind, d_pos, d_str, n, rank, nslabs, d_spec, nullptr);
    });
}

fse_status fse_cuda_slab_forward_peers(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                       const double* d_pos, const double* d_str, int64_t n,
                                       int rank, int nslabs, double* const* dst_bufs) {
    return api(c, [&] {
        if (!dst_bufs) invalid("null pointer");
        slab_forward_impl(c, cfg, kind, d_pos, d_str, n, rank, nslabs, nullptr, dst_bufs);
    });
}

fse_status fse_cuda_slab_scale(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                               const fse_green* green, int rank, int nslabs, double* d_spec) {
    return api(c, [&] { slab_scale_impl(c, cfg, kind, green, rank, nslabs, d_spec, nullptr); });
}

fse_status fse_cuda_slab_scale_peers(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                     const fse_green* green, int rank, int nslabs,
                                     double* d_spec, double* const* dst_bufs) {
    return api(c, [&] {
        if (!dst_bufs) invalid("null pointer");
        slab_scale_impl(c, cfg, kind, green, rank, nslabs, d_spec, dst_bufs);
    });
}

fse_status fse_cuda_slab_inverse(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                 const double* d_pos, const double* d_str, int64_t n,
                                 double* d_spec, int rank, int nslabs, const double* d_tgt,
                                 int64_t nt, int tas, double* d_u) {
    return api(c, [&] {
        check_kind(kind);
        if (!d_spec || !d_u || (nt > 0 && !d_tgt) || (n > 0 && (!d_pos || !d_str)))
            invalid("null pointer");
        const int a = arity_of(kind);
        const GridParams g = slab_params(cfg, rank, nslabs);
        FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
        Launch L = L0(c);
        // real space for the targets in this rank's x-slice of the cell grid
        // (stream s1); rank 0 adds the self term
        double* uR = buf<double>(c, "uR", 3 * std::max<int64_t>(nt, 1));
        FSE_CU(cudaEventRecord(c->ev[EV_START], c->s0));
        FSE_CU(cudaStreamWaitEvent(c->s1, c->ev[EV_START], 0));
        if (nt > 0)
            real_part(c, kind, d_pos, d_str, n, cfg->L, cfg->xi, cfg->rc, d_tgt, nt, tas != 0, uR,
                      rank, nslabs);
        FSE_CU(cudaEventRecord(c->ev[EV_JOIN], c->s1));
        // inverse y/z passes of this slab, then its planes' share of the quadrature
        double* qtab = buf<double>(c, "qtab", g.P);
        launch_quad_table(L, g, qtab);
        double* W = buf<double>(c, "R", static_cast<size_t>(a) * g.comp);
        double2* Bs = buf<double2>(c, "B", static_cast<size_t>(a) * g.nx * g.Mt * g.Dh);
        const FftPlanDev& fp = fft_plan(c, g.D);
        launch_fft_inverse_yz(L, fp.host, fp.tw, g, a, reinterpret_cast<double2*>(d_spec), Bs, W);
        Sorted tg = prep_points(c, g, "ft_", d_tgt, nullptr, 0, nt, 1, qtab);
        const int64_t nhalf = g.nkeys / 4;
        int32_t* scnt = buf<int32_t>(c, "scnt", nhalf + 1);
        int32_t* soff = buf<int32_t>(c, "soff", nhalf + 1);
        launch_slab_counts(L, g, tg.tstart, nhalf, scnt);
        exclusive_scan(c, c->s0, "s0", scnt, soff, nhalf + 1);
        const int64_t max_items = std::min<int64_t>(nhalf, nt) + (nt + 31) / 32;
        int32_t* sitems = buf<int32_t>(c, "sitems", 2 * static_cast<size_t>(max_items));
        launch_slab_fill(L, soff, nhalf, sitems);
        // tiles whose union box misses this slab get no items: their targets'
        // partial velocities are zero
        if (nslabs > 1 && nt > 0)
            FSE_CU(cudaMemsetAsync(d_u, 0, sizeof(double) * 3 * nt, c->s0));
        if (nt > 0)
            launch_gather_slab(L, g, tg.i0s, tg.w, tg.tstart, sitems, max_items, soff + nhalf, W,
                               tg.perm, g.h * g.h * g.h, d_u);
        FSE_CU(cudaStreamWaitEvent(c->s0, c->ev[EV_JOIN], 0));
        if (nt > 0) {
            const bool self = tas && kind == FSE_STOKESLET && rank == 0;
            launch_epilogue(L, nt, d_u, uR, self ? d_str : nullptr,
                            self ? -4.0 * cfg->xi / std::sqrt(M_PI) : 0.0, d_u);
        }
        raise_flags(c);
    });
}

fse_status fse_cuda_fourier_sum(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                const double* pos, const double* str, int64_t n, double box_side,
                                const double* targets, int64_t nt, const fse_green* green,
                                double* u, fse_timings* tm) {
    return api(c, [&] {
        run_sum_host(c, cfg, kind, pos, str, n, box_side, targets, nt, -1, green, u, tm, true,
                     false);
    });
}

fse_status fse_cuda_real_space_sum(fse_cuda_ctx* c, int kind, const double* pos,
                                   const double* str, int64_t n, double box_side, double xi,
                                   double rc, const double* targets, int64_t nt, double* u) {
    return api(c, [&] {
        if (!(xi > 0) || !(rc > 0)) invalid("real_space_sum: xi and rc must be positive");
        fse_config cfg;
        std::memset(&cfg, 0, sizeof cfg);
        cfg.xi = xi;
        cfg.rc = rc;
        run_sum_host(c, &cfg, kind, pos, str, n, box_side, targets, nt, -1, nullptr, u, nullptr,
                     false, true);
    });
}

fse_status fse_cuda_spread(fse_cuda_ctx* c, const fse_config* cfg, int kind, const double* pos,
                           const double* str, int64_t n, double box_side, double* grid) {
    return fse_cuda_spread_ex(c, cfg, kind, pos, str, n, box_side, 1, grid);
}

fse_status fse_cuda_spread_ex(fse_cuda_ctx* c, const fse_config* cfg, int kind, const double* pos,
                              const double* str, int64_t n, double box_side, int use_fgg,
                              double* grid) {
    return api(c, [&] {
        check_kind(kind);
        check_cfg(cfg);
        if (std::abs(box_side - cfg->L) > 1e-12 * cfg->L)
            invalid("spread: config box does not match system");
        if (n < 0 || (n > 0 && (!pos || !str)) || !grid) invalid("null pointer");
        const int a = arity_of(kind);
        const GridParams g = make_grid_params(*cfg);
        double* d_pos = buf<double>(c, "in_pos", 3 * n);
        double* d_str = buf<double>(c, "in_str", a * n);
        h2d(c, d_pos, pos, sizeof(double) * 3 * n);
        h2d(c, d_str, str, sizeof(double) * a * n);
        FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
        double* qtab = buf<double>(c, "qtab", g.P);
        launch_quad_table(L0(c), g, qtab);
        Sorted src = prep_points(c, g, "fs_", d_pos, d_str, a, n, 0, qtab, use_fgg == 0);
        double* X = buf<double>(c, "R", static_cast<size_t>(a) * g.comp);
        for (int c0 = 0; c0 < a; c0 += 3)
            launch_spread(L0(c), g, src.i0s, src.w, src.fs, n, a, c0, src.tstart, X);
        const size_t vol = static_cast<size_t>(g.Mt) * g.Mt * g.Mt;
        double* out = buf<double>(c, "grid_out", a * vol);
        launch_extract_grid(L0(c), g, X, a, out);
        raise_flags(c);
        d2h(c, grid, out, sizeof(double) * a * vol);
    });
}

fse_status fse_cuda_kspace_scale(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                 const fse_green* green, const double* ghat, double* out) {
    return api(c, [&] {
        check_kind(kind);
        check_cfg(cfg);
        check_green(cfg, kind, green);
        if (!ghat || !out) invalid("null pointer");
        const int a = arity_of(kind);
        const GridParams g = make_grid_params(*cfg);
        const size_t T = static_cast<size_t>(g.D) * g.D * g.D;
        double* Gf = buf<double>(c, "ks_G", T);
        double2* gh = buf<double2>(c, "ks_in", a * T);
        double2* o = buf<double2>(c, "ks_out", 3 * T);
        launch_green_half_to_full(L0(c), g.D, green->d_half, Gf);
        h2d(c, gh, ghat, sizeof(double2) * a * T);
        launch_kscale_full(L0(c), g, kind, Gf, gh, o);
        d2h(c, out, o, sizeof(double2) * 3 * T);
    });
}

fse_status fse_cuda_build_cell_list(fse_cuda_ctx* c, const double* pos, int64_t n,
                                    double box_side, double rc, double pad, int* dims,
                                    double* cell_side, double* origin, int64_t* bstart,
                                    int64_t* perm) {
    return api(c, [&] {
        if (n < 0 || (n > 0 && !pos) || !dims || !cell_side || !origin) invalid("null pointer");
        const CellGrid cg = cell_grid(n, box_side, rc, pad);
        dims[0] = dims[1] = dims[2] = cg.dim;
        *cell_side = cg.side;
        *origin = cg.origin;
        if (!bstart) return;
        double* d_pos = buf<double>(c, "in_pos", 3 * n);
        FSE_CU(cudaMemcpyAsync(d_pos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->s1));
        Cells cl = bin_cells(c, cg, "rs_", d_pos, nullptr, 0, n);
        int64_t* b64 = buf<int64_t>(c, "cl_b64", cg.ncell + 1);
        int64_t* p64 = buf<int64_t>(c, "cl_p64", n);
        launch_i32_to_i64(L1(c), cl.start, b64, cg.ncell + 1);
        launch_u32_to_i64(L1(c), cl.perm, p64, n);
        FSE_CU(cudaMemcpyAsync(bstart, b64, sizeof(int64_t) * (cg.ncell + 1),
                               cudaMemcpyDeviceToHost, c->s1));
        if (n > 0 && perm)
            FSE_CU(cudaMemcpyAsync(perm, p64, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->s1));
        FSE_CU(cudaStreamSynchronize(c->s1));
    });
}

fse_status fse_cuda_support_index(fse_cuda_ctx* c, const fse_config* cfg, const double* pos,
                                  int64_t n, int32_t* i0) {
    return api(c, [&] {
        check_cfg(cfg);
        if (n < 0 || (n > 0 && (!pos || !i0))) invalid("null pointer");
        const GridParams g = make_grid_params(*cfg);
        double* d_pos = buf<double>(c, "in_pos", 3 * n);
        int32_t* d_i0 = buf<int32_t>(c, "si_i0", 3 * n);
        h2d(c, d_pos, pos, sizeof(double) * 3 * n);
        FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
        launch_support_keys(L0(c), g, d_pos, n, 0, nullptr, d_i0, c->d_flags);
        d2h(c, i0, d_i0, sizeof(int32_t) * 3 * n);
        raise_flags(c);
    });
}

fse_status fse_cuda_direct_sum(fse_cuda_ctx* c, int kind, const double* pos, const double* str,
                               int64_t n, const double* targets, int64_t nt, int exclude_self,
                               double* u) {
    return api(c, [&] {
        check_kind(kind);
        if (n < 0 || nt < 0 || (n > 0 && (!pos || !str)) || (nt > 0 && (!targets || !u)))
            invalid("null pointer");
        const int a = arity_of(kind);
        double* d_pos = buf<double>(c, "in_pos", 3 * n);
        double* d_str = buf<double>(c, "in_str", a * n);
        double* d_tgt = buf<double>(c, "in_tgt", 3 * nt);
        double* d_u = buf<double>(c, "in_u", 3 * nt);
        h2d(c, d_pos, pos, sizeof(double) * 3 * n);
        h2d(c, d_str, str, sizeof(double) * a * n);
        h2d(c, d_tgt, targets, sizeof(double) * 3 * nt);
        FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
        launch_direct(L0(c), kind, d_pos, d_str, n, d_tgt, nt, exclude_self, d_u, c->d_flags);
        raise_flags(c);
        d2h(c, u, d_u, sizeof(double) * 3 * nt);
    });
}

// fft.cpp:13-37 over cuFFT Z2Z (in place, inverse scaled by 1/(n0 n1 n2))
// diagnostics for the hand-written FFT engine: ncols contiguous length-D columns
fse_status fse_cuda_fft_columns(fse_cuda_ctx* c, int D, int ncols, double* data, int inverse) {
    return api(c, [&] {
        if (!data || D < 1 || ncols < 1) invalid("fft_columns: bad arguments");
        const FftPlanDev& fp = fft_plan(c, D);
        const size_t n = static_cast<size_t>(D) * ncols;
        double2* d = buf<double2>(c, "fftcol", n);
        h2d(c, d, data, n * sizeof(double2));
        fft_test_columns(L0(c), fp.host, fp.tw, d, ncols, inverse);
        d2h(c, data, d, n * sizeof(double2));
    });
}

// diagnostics: the fused x pass (k_xscale*: FFT_x -> multiplier -> IFFT_x) of the
// hot path on a pseudo-random spectrum, probed at chosen (ky, kz) columns
fse_status fse_cuda_xscale_probe(fse_cuda_ctx* c, const fse_config* cfg, int kind,
                                 const fse_green* green, uint64_t seed, int nprobe,
                                 const int* ky, const int* kz, double* out, double* gcol) {
    return api(c, [&] {
        check_cfg(cfg);
        check_kind(kind);
        if (green) check_green(cfg, kind, green);
        if (nprobe < 1 || !ky || !kz || !out || !gcol) invalid("xscale_probe: bad arguments");
        const GridParams g = make_grid_params(*cfg);
        for (int p = 0; p < nprobe; ++p)
            if (ky[p] < 0 || ky[p] >= g.D || kz[p] < 0 || kz[p] >= g.Dh)
                invalid("xscale_probe: column out of range");
        const int a = arity_of(kind);
        const Launch L = L0(c);
        fft_xscale_check(fft_plan(c, g.D).host, kind);  // before the big buffers
        const int64_t nC = static_cast<int64_t>(a) * g.Mt * g.D * g.Dh;
        double2* C = buf<double2>(c, "C", static_cast<size_t>(nC));
        launch_probe_fill(L, C, nC, seed);
        const double* G = nullptr;
        if (green) {
            G = green->d_half;
        } else {
            const int64_t nG = static_cast<int64_t>(g.D) * g.D * g.Dh;
            double* Gs = buf<double>(c, "probe_G", static_cast<size_t>(nG));
            launch_probe_green(L, Gs, nG, seed ^ 0x5DEECE66Dull);
            G = Gs;
        }
        const FftPlanDev& fp = fft_plan(c, g.D);
        launch_fft_xscale(L, fp.host, fp.tw, g, kind, G, C, buf<double>(c, "ex_axis", g.D));
        int* dk = buf<int>(c, "probe_k", 2 * static_cast<size_t>(nprobe));
        h2d(c, dk, ky, sizeof(int) * nprobe);
        h2d(c, dk + nprobe, kz, sizeof(int) * nprobe);
        const size_t no = static_cast<size_t>(nprobe) * 3 * g.Mt;
        double2* dout = buf<double2>(c, "probe_out", no);
        double* dg = buf<double>(c, "probe_gcol", static_cast<size_t>(nprobe) * g.D);
        launch_probe_extract(L, C, G, g.Mt, g.D, nprobe, dk, dk + nprobe, dout, dg);
        d2h(c, out, dout, no * sizeof(double2));
        d2h(c, gcol, dg, sizeof(double) * nprobe * g.D);
    });
}

// host-only: the FFT planner's verdict for a grid size (include/fse_host.h)
fse_status fse_fft_plan_query(int D, int kind, int* engine, int* generic_stage) {
    try {
        if (D < 2 || D % 2) throw Error(FSE_EINVAL, "fft_plan_query: D must be even and >= 2");
        check_kind(kind);
        const HostFftPlan h = make_fft_plan(D);
        if (engine) *engine = h.eng;
        if (generic_stage) *generic_stage = h.generic ? 1 : 0;
        fft_xscale_check(h, kind);
        return FSE_OK;
    } catch (const Error& e) {
        return e.code;
    } catch (const std::exception&) {
        return FSE_ERUNTIME;
    }
}

fse_status fse_cuda_fft3d(fse_cuda_ctx* c, double* data, int n0, int n1, int n2, int inverse) {
    return api(c, [&] {
        if (!data || n0 < 1 || n1 < 1 || n2 < 1) invalid("fft3d: bad arguments");
        const size_t n = static_cast<size_t>(n0) * n1 * n2;
        double2* d = buf<double2>(c, "fft_data", n);
        h2d(c, d, data, n * sizeof(double2));
        cufftHandle p;
        FSE_CUFFT(cufftPlan3d(&p, n0, n1, n2, CUFFT_Z2Z));
        cufftSetStream(p, c->s0);
        const cufftResult r = cufftExecZ2Z(p, reinterpret_cast<cufftDoubleComplex*>(d),
                                           reinterpret_cast<cufftDoubleComplex*>(d),
                                           inverse ? CUFFT_INVERSE : CUFFT_FORWARD);
        if (r != CUFFT_SUCCESS) {
            cufftDestroy(p);
            throw_cufft(r, "cufftExecZ2Z", __FILE__, __LINE__);
        }
        if (inverse) launch_scale_complex(L0(c), d, static_cast<int64_t>(n), 1.0 / static_cast<double>(n));
        d2h(c, data, d, n * sizeof(double2));
        cufftDestroy(p);
    });
}

}  // extern "C"

static_assert(sizeof(fse_config) == 120, "fse_config must mirror fse::EwaldConfig (120 bytes)");
static_assert(offsetof(fse_config, Mtilde) == 80, "EwaldConfig layout");
static_assert(offsetof(fse_config, kinf) == 88, "EwaldConfig layout");
static_assert(offsetof(fse_config, deterministic) == 112, "EwaldConfig layout");

#include "fse_dist.cuh"
