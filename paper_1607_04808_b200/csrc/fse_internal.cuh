// fse_internal.cuh -- shared declarations of the B200 (sm_100a) free-space
// Spectral Ewald library.  Host orchestration lives in fse_capi.cu; kernels
// live in one .cu per stage.  Only plain device pointers cross these
// interfaces; the C-ABI (include/fse_cuda.h) is the only public surface.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "fse_cuda.h"

namespace fsecu {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    fse_status code;
    Error(fse_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
[[noreturn]] void throw_cufft(cufftResult r, const char* what, const char* file, int line);

#define FSE_CU(x)                                                             \
    do {                                                                      \
        cudaError_t e_ = (x);                                                 \
        if (e_ != cudaSuccess) ::fsecu::throw_cuda(e_, #x, __FILE__, __LINE__); \
    } while (0)
#define FSE_CUFFT(x)                                                              \
    do {                                                                          \
        cufftResult r_ = (x);                                                     \
        if (r_ != CUFFT_SUCCESS) ::fsecu::throw_cufft(r_, #x, __FILE__, __LINE__); \
    } while (0)
#define FSE_LAUNCH_CHECK() FSE_CU(cudaGetLastError())

// device-side error flags (bit set => condition hit)
enum : int {
    FLAG_SUPPORT = 1,      // ewald.cpp:87-91 point support exceeds grid
    FLAG_TARGET_BOX = 2,   // ewald.cpp:299-302 target outside [0,L]^3
    FLAG_COINCIDENT = 4,   // kernels.cpp:79-80 coincident target/source
};

inline int arity_of(int kind) { return kind == FSE_STRESSLET ? 9 : 3; }

// ------------------------------------------------------------ grid params
// Everything a Fourier-stage kernel needs, derived once per evaluation from
// fse_config exactly as the reference derives it (ewald.cpp:147,152-157,
// 232-235, 351-357).
struct GridParams {
    int P;          // support
    int Mt;         // Mtilde
    int D;          // 2 Mtilde (FFT size, exact: SURVEY 8a A6)
    int Dh;         // D/2 + 1 (half spectrum)
    // real grids (spread output R, quadrature input W) are compact Mt^3 per component
    int64_t rowp;   // doubles per row: Mt
    int64_t plane;  // doubles per x-plane: Mt * Mt
    int64_t comp;   // doubles per component: Mt^3
    double h, origin, alpha, prefac, L;
    double dk, inv4xi2, eta, invD3;
    // spread/gather tiling of the support-start space (i0x, i0y, i0z)
    int ncx, ncy, ncz;  // coarse tiles: 8 x 8 x 16
    int64_t nkeys;      // ncx*ncy*ncz*8 fine keys (4 x 4 x 8 sub-tiles)
    // z-slab decomposition (one GPU: the whole grid, one block).
    // Real grids hold this slab's x-planes [x_lo, x_lo + nx) (comp = nx*plane);
    // the spectrum is blocked by nxs x-planes / nkys ky-rows, and this rank's
    // x-pass covers ky rows [ky_lo, ky_lo + nky).
    int x_lo, nx, nxs;
    int ky_lo, nky, nkys;
};
// restrict g to slab r of G (x-planes in multiples of 8, ky rows balanced)
void set_slab(GridParams& g, int r, int G);

// Destination of each spectrum block that crosses the slab exchange (block b
// goes to rank b).  Local exchange buffer (one GPU, NCCL path): base + b *
// stride; peer-direct: tab[b] (a device array) = block `rank` of rank b's
// buffer, mapped into this process over NVLink, so the pass that produces a
// block stores it straight into its owner's memory (no send buffer, no NCCL
// all-to-all).  (A pointer array passed by value would be copied to local
// memory by the dynamic block index.)
constexpr int kMaxSlabs = 16;
struct BlockDest {
    double2* base;
    int64_t stride;
    double2* const* tab;
};
__device__ __forceinline__ double2* block_ptr(const BlockDest& d, int b) {
    return d.tab ? d.tab[b] : d.base + b * d.stride;
}

GridParams make_grid_params(const fse_config& cfg);

// Device-side constant tables (per call, small): q[p] = exp(-alpha (p h)^2)
// (ewald.cpp:154-156) lives in a device buffer passed to the weight kernel.

// --------------------------------------------------------------- launches
// Every launcher enqueues on `s` and bumps *launches by the number of kernels.
struct Launch {
    cudaStream_t s;
    uint64_t* launches;
};

// k_particles.cu ------------------------------------------------------------
// support start + tile key per point; flags FLAG_SUPPORT / FLAG_TARGET_BOX
void launch_support_keys(const Launch& L, const GridParams& g, const double* pos, int64_t n,
                         int check_box, uint32_t* key, int32_t* i0, int* flags);
// q[p] table
void launch_quad_table(const Launch& L, const GridParams& g, double* q);
// sorted payload: i0s (n x 3), weights (n x 3P, prefac folded into x when
// fold_prefac), strengths (a x n SoA), from perm; naive: one exp per node
// (axis_weights_naive, ewald.cpp:53-66) instead of the FGG recurrence
void launch_gather_payload(const Launch& L, const GridParams& g, const double* pos,
                           const double* str, int a, const uint32_t* perm, int64_t n,
                           const double* qtab, int32_t* i0s, double* w, double* fs,
                           bool fold_prefac, int slab_only = 0, bool naive = false);
// histogram of keys into counts (size nkeys, zeroed by caller)
void launch_histogram(const Launch& L, const uint32_t* keys, int64_t n, int32_t* counts);
// cell ids of points for the reference cell list (realspace.cpp:60-63,80)
void launch_cell_ids(const Launch& L, const double* pos, int64_t n, double origin, double side,
                     int dim, uint32_t* cell, int sub = 1);
// SoA permute of positions (+ strengths) by perm
void launch_permute_soa(const Launch& L, const double* pos, const double* str, int a,
                        const uint32_t* perm, int64_t n, double* px, double* py, double* pz,
                        double* fs);
void launch_iota(const Launch& L, uint32_t* v, int64_t n);
void launch_u32_to_i64(const Launch& L, const uint32_t* in, int64_t* out, int64_t n);
void launch_i32_to_i64(const Launch& L, const int32_t* in, int64_t* out, int64_t n);

// k_spread.cu ---------------------------------------------------------------
// writes the Mt^3 grid of components [c0, c0+3) into X (real view, x-planes
// of pitch plane, rows of pitch D+2)
// (tiles of this slab's x-planes only; X holds the slab: x - x_lo)
void launch_spread(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                   const double* fs, int64_t n, int a, int c0, const int32_t* tstart,
                   double* X, const int32_t* order = nullptr);
// heavy-tiles-first order for launch_spread (spread_tiles(g) ints): flags, then the
// caller's exclusive scan of `light` into pos, then place
unsigned spread_tiles(const GridParams& g);
void launch_spread_flags(const Launch& L, const GridParams& g, const int32_t* tstart, int64_t n,
                         int32_t* light, uint8_t* hbucket, int32_t* bwork);
void launch_spread_place(const Launch& L, const GridParams& g, const int32_t* light,
                         const int32_t* pos, const uint8_t* hbucket, int32_t* bwork,
                         int32_t* order);
// Mt^3 compact copy out of the real view (for the fse::spread API)
void launch_extract_grid(const Launch& L, const GridParams& g, const double* X, int a,
                         double* out);

// k_kscale.cu ---------------------------------------------------------------
// full D^3 C2C, reference multiplier verbatim (ewald.cpp:216-293)
void launch_kscale_full(const Launch& L, const GridParams& g, int kind, const double* Gfull,
                        const double2* ghat, double2* out);
void launch_scale_complex(const Launch& L, double2* data, int64_t n, double s);

// k_gather.cu ---------------------------------------------------------------
// groups of <= 8 targets per fine tile; group table built by caller
void launch_gather(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                   const int32_t* tstart, const int32_t* gkey, const int32_t* goff,
                   int64_t max_groups, const double* X, const uint32_t* perm, double scale,
                   double* u);
void launch_group_counts(const Launch& L, const int32_t* tstart, int64_t nkeys, int32_t* gcount);
int gather_group_size();
// slab-staged gather (k_gather.cu): items = (coarse tile, z-half, batch of 32)
bool gather_slab_enabled(const GridParams& g);
size_t slab_smem_bytes(const GridParams& g);
void launch_slab_counts(const Launch& L, const GridParams& g, const int32_t* tstart,
                        int64_t nhalf, int32_t* cnt);
void launch_slab_fill(const Launch& L, const int32_t* off, int64_t nhalf, int32_t* items);
void launch_gather_slab(const Launch& L, const GridParams& g, const int32_t* i0s, const double* w,
                        const int32_t* tstart, const int32_t* items, int64_t max_items,
                        const int32_t* nitems_dev, const double* X, const uint32_t* perm,
                        double scale, double* u);
void launch_fill_groups(const Launch& L, const int32_t* tstart, const int32_t* goff,
                        int64_t nkeys, int32_t* gkey);

// k_realspace.cu ------------------------------------------------------------
struct CellGrid {
    int dim;
    double origin, side;
    int64_t ncell;
};
void launch_realspace(const Launch& L, int kind, const CellGrid& cg, const double* spx,
                      const double* spy, const double* spz, const double* sfs, int64_t ns,
                      const int32_t* bstart, const double* tpx, const double* tpy,
                      const double* tpz, const int32_t* tcell_start, const int32_t* items,
                      int64_t max_items, const int32_t* nitems_dev, const uint32_t* tperm,
                      double xi, double rc, unsigned long long* counts, double* uR, int per,
                      int sub);
// targets per work item (selects the pair kernel: 32 = warp items, else CTA-shared)
int realspace_item_size(int64_t nt, int64_t ncell);
// items per cell; only cells in [c_lo, c_hi) get any (c_hi < 0: all cells)
// the pair kernel's work items (cell, 32-target chunk), heaviest cells first;
// *nitems (device) = item count; bwork: 3 x realspace_work_buckets() ints
int realspace_work_buckets();
void launch_realspace_items(const Launch& L, const int32_t* sstart, const int32_t* tstart,
                            int dim, int64_t ncell, int per, int64_t c_lo, int64_t c_hi,
                            uint8_t* bucket, int32_t* bwork, int32_t* items, int32_t* nitems,
                            int oct_min, int sub);
// cells with at least this many targets are split into octant items (0: never)
int realspace_octant_threshold();

// epilogue: u[perm] = uF + uR (+ self) -------------------------------------
// u = uF + uR (+ self_coef * f for the stokeslet self term), caller order
void launch_epilogue(const Launch& L, int64_t nt, const double* uF, const double* uR,
                     const double* str_self, double self_coef, double* u);

// k_green.cu ----------------------------------------------------------------
// Hhat^R / Bhat^R (greens.cpp:62-79) on the octant q in [0, sM/2]^3 of the sM^3
// wavenumber grid, [qx][qy][qz] (the grid is even in every axis)
void launch_green_octant(const Launch& L, int gkind, int sM, double dk, double R, double* oct);
// T[kx][ky][kz] (k in [0, Mt]^3, even table) -> D x D x (D/2+1) half table
void launch_green_unfold(const Launch& L, int Mt, const double* T, double* half);
// full <-> half conversions of the reference layout
void launch_green_full_to_half(const Launch& L, int D, const double* full, double* half);
void launch_green_half_to_full(const Launch& L, int D, const double* half, double* full);

// k_direct.cu ---------------------------------------------------------------
double measure_dfma_tflops(const Launch& L, double* scratch);
void launch_direct(const Launch& L, int kind, const double* pos, const double* str, int64_t n,
                   const double* tgt, int64_t nt, int exclude_self, double* u, int* flags);

// x-pass probe (fse_cuda_xscale_probe, diagnostics) ------------------------------
void launch_probe_fill(const Launch& L, double2* C, int64_t n, uint64_t seed);
void launch_probe_green(const Launch& L, double* G, int64_t n, uint64_t seed);
void launch_probe_extract(const Launch& L, const double2* C, const double* G, int Mt, int D,
                          int nprobe, const int* ky, const int* kz, double2* out, double* gcol);

}  // namespace fsecu
