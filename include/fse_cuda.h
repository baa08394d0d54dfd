/*
 * fse_cuda.h -- C-ABI of the B200-native free-space Spectral Ewald library
 * (libfse_b200.so).  Plain pointers, sizes and PODs; no C++ or torch types.
 *
 * This is the drop-in boundary for the reference's hot path,
 * fse::total_sum (/root/reference/proj/src/ewald.cpp:394-415) and the
 * functions under it.  Each entry point names the reference interface it
 * replaces.  The C++ wrapper (paper_1607_04808_b200/cpp/include/fse/*.hpp,
 * namespace fse) re-exposes the reference's C++ signatures over this ABI.
 *
 * Conventions
 *   - positions / targets: N x 3 doubles, AoS (x,y,z), like std::vector<fse::Vec3>
 *     (vec3.hpp:8-17);
 *   - strengths: N x a doubles, a = fse_arity(kind) (3, or 9 for the stresslet with
 *     f_lm at 3l+m), i.e. the first `arity` slots of fse::Strength::c (kernels.hpp:25-56);
 *   - velocities: NT x 3 doubles;
 *   - kinds: FSE_STOKESLET / FSE_STRESSLET / FSE_ROTLET (kernels.hpp:16 order);
 *   - every call returns an fse_status; FSE_EINVAL maps to std::invalid_argument,
 *     FSE_EDOMAIN to std::domain_error, the rest to std::runtime_error.
 *     fse_cuda_last_error(ctx) holds the message (per context, per thread).
 *   - calls are blocking (results are complete on return) and thread-safe per
 *     context (one mutex per context); use one context per host thread for
 *     concurrency, as the reference allows concurrent calls.
 *   - "_dev" variants take device pointers on the context's device and do no
 *     host<->device copies.
 */
#ifndef FSE_CUDA_H
#define FSE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSE_CUDA_ABI_VERSION 1

typedef enum {
    FSE_OK = 0,
    FSE_EINVAL = 1,   /* std::invalid_argument */
    FSE_EDOMAIN = 2,  /* std::domain_error */
    FSE_ERUNTIME = 3, /* std::runtime_error (I/O) */
    FSE_ECUDA = 4,
    FSE_ECUFFT = 5,
    FSE_ENOMEM = 6,
    FSE_ENCCL = 7
} fse_status;

typedef enum { FSE_STOKESLET = 0, FSE_STRESSLET = 1, FSE_ROTLET = 2 } fse_kernel_kind;
typedef enum { FSE_HARMONIC = 0, FSE_BIHARMONIC = 1 } fse_green_kind;

/* Bitwise mirror of fse::EwaldConfig (ewald.hpp:16-35), 120 bytes. */
typedef struct {
    double L, xi, rc;
    int32_t M, P;
    double h, d, m, eta, deltaL, Ltilde;
    int32_t Mtilde;
    int32_t _pad0;
    double kinf, R, sf;
    uint8_t deterministic;
    uint8_t _pad1[7];
} fse_config;

/* Mirror of fse::StageTimings (ewald.hpp:56-64), seconds; calls ACCUMULATE (+=). */
typedef struct {
    double precompute, spread, fft, scale, quadrature, realspace, total;
} fse_timings;

typedef struct fse_cuda_ctx fse_cuda_ctx;
typedef struct fse_green fse_green; /* device-resident MollifiedGreen */

/* ---- context ------------------------------------------------------------ */
fse_status fse_cuda_create(int device, fse_cuda_ctx** out);
void fse_cuda_destroy(fse_cuda_ctx* ctx);
const char* fse_cuda_last_error(const fse_cuda_ctx* ctx);
int fse_cuda_abi_version(void);
int fse_arity(int kind);
/* release cached device buffers and FFT plans (the context stays usable) */
fse_status fse_cuda_trim(fse_cuda_ctx* ctx);
/* pinned host memory for fast copies (optional) */
fse_status fse_cuda_host_alloc(fse_cuda_ctx* ctx, size_t bytes, void** out);
void fse_cuda_host_free(void* p);
/* device memory on the context's device (for the _dev entry points) */
fse_status fse_cuda_dev_alloc(fse_cuda_ctx* ctx, size_t bytes, void** out);
void fse_cuda_dev_free(fse_cuda_ctx* ctx, void* p);
fse_status fse_cuda_memcpy(fse_cuda_ctx* ctx, void* dst, const void* src, size_t bytes);
/* device time (ms) between the last two fse_cuda_mark() calls on the context stream */
fse_status fse_cuda_mark(fse_cuda_ctx* ctx);
fse_status fse_cuda_elapsed_ms(fse_cuda_ctx* ctx, double* ms);
/* number of kernels this library launched on the context since creation */
uint64_t fse_cuda_launch_count(const fse_cuda_ctx* ctx);
/* device time (ms) of the stages of the last total/fourier/real sum, CUDA events on the
 * launching streams: [0] source prep (support keys, sort, weights) [1] spectrum memset
 * [2] spread kernel [3] forward FFTs [4] k-space scale [5] inverse FFTs [6] target prep
 * [7] gather kernel [8] real-space binning [9] real-space pair kernel [10] whole call */
fse_status fse_cuda_kernel_ms(fse_cuda_ctx* ctx, double* out, int n);
/* fse::freespace_solve (greens.hpp:76, greens.cpp:115-139): rhs and out are
 * M~^3 host arrays [i][j][k] on the green's grid (M~ = green Mtilde); the free-space
 * convolution of rhs with the green's kernel (harmonic: 1/r, biharmonic: r),
 * unscaled by h^3 as in the reference. */
fse_status fse_cuda_freespace_solve(fse_cuda_ctx* ctx, const fse_green* green, const double* rhs,
                                    double* out);

/* ---- z-slab decomposition over several GPUs (no reference counterpart:
 * the reference is single-process).  Slab `rank` of `nslabs` owns the x-planes
 * [x_lo, x_lo + nx) of the M~ grid and the ky rows [ky_lo, ky_lo + nky) of the
 * k-space pass; every rank holds all points.  Per evaluation:
 *   fse_cuda_slab_forward  -> spectrum send buffer, nslabs blocks of block_complex
 *   all-to-all (block s -> rank s; received blocks in source-rank order)
 *   fse_cuda_slab_scale    (in place on the received buffer)
 *   all-to-all back        (block r -> rank r)
 *   fse_cuda_slab_inverse  -> this rank's partial velocities (NT x 3)
 *   sum of the partials over ranks = total_sum.
 * The exchanges are the caller's (bench.py / slabs.py use NCCL via torch.distributed).
 * nslabs = 1 reproduces fse_cuda_total_sum_dev. */
typedef struct {
    int x_lo, nx, nxs;      /* this slab's x-planes; nxs planes per slab */
    int ky_lo, nky, nkys;   /* this rank's ky rows; nkys rows per block */
    int64_t block_complex;  /* complex values per spectrum block (a * nxs * nkys * (D/2+1)) */
} fse_slab_info;
fse_status fse_cuda_slab_info(const fse_config* cfg, int kind, int rank, int nslabs,
                              fse_slab_info* out);
/* spread of all sources onto this slab's planes, z and y FFT passes (device pointers;
 * d_spec: nslabs * block_complex complex doubles) */
fse_status fse_cuda_slab_forward(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                 const double* d_pos, const double* d_str, int64_t n, int rank,
                                 int nslabs, double* d_spec);
/* x-FFT, k-space multiplier, inverse x-FFT for this rank's ky rows, in place on the
 * received spectrum (blocks in source-rank order) */
fse_status fse_cuda_slab_scale(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                               const fse_green* green, int rank, int nslabs, double* d_spec);
/* inverse y/z passes and this slab's share of the quadrature for all targets, plus the
 * real-space sum and self term of targets [nt*rank/nslabs, nt*(rank+1)/nslabs):
 * d_u (NT x 3, device) = this rank's partial velocities */
fse_status fse_cuda_slab_inverse(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                 const double* d_pos, const double* d_str, int64_t n,
                                 double* d_spec, int rank, int nslabs, const double* d_tgt,
                                 int64_t nt, int tas, double* d_u);
/* Peer-direct exchange (no all-to-all): every rank allocates two exchange buffers
 * A_s, B_s (nslabs * block_complex each) that all ranks map (CUDA IPC / symmetric
 * memory over NVLink); dst_bufs[s] is rank s's buffer as seen from this process.
 *   fse_cuda_slab_forward_peers(dst_bufs = {A_s}): the y pass stores block s of this
 *       rank's spectrum straight into A_s at block `rank` (what the all-to-all would
 *       have delivered);
 *   barrier;
 *   fse_cuda_slab_scale_peers(d_spec = A_rank, dst_bufs = {B_s}): the x pass reads its
 *       own A and stores x block r of the results into B_r at block `rank`;
 *   barrier;
 *   fse_cuda_slab_inverse(d_spec = B_rank), then the sum of the partials.
 * nslabs <= 16.  Both calls return after their kernels completed (the caller's
 * barrier then orders the phases across ranks). */
fse_status fse_cuda_slab_forward_peers(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                       const double* d_pos, const double* d_str, int64_t n,
                                       int rank, int nslabs, double* const* dst_bufs);
fse_status fse_cuda_slab_scale_peers(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                     const fse_green* green, int rank, int nslabs,
                                     double* d_spec, double* const* dst_bufs);

/* ---- partitioned multi-GPU evaluation (no reference counterpart).
 * Each rank (one GPU, one process or thread) holds only the points it OWNS: a point
 * at x belongs to the slab whose x-planes hold its support centre ceil((x - origin)/h)
 * (fse_dist_owner).  One call of fse_cuda_dist_total_sum on every rank exchanges, over
 * NCCL (grouped ncclSend / ncclRecv on the context's stream):
 *   the ghost sources each neighbour needs (supports crossing into its planes,
 *   real-space neighbours within rc of its owned targets) and the targets whose
 *   support crosses into its planes; the two spectrum transposes of the distributed
 *   FFT; and the ghost targets' partial quadrature sums back to their owners.
 * u receives the velocities of this rank's owned targets, in their input order
 * (n_total: the global source count, which fixes the cell-list geometry).
 * fse_cuda_nccl_unique_id fills the 128-byte ncclUniqueId that rank 0 creates and the
 * caller broadcasts (any channel) before fse_cuda_dist_create. */
typedef struct fse_dist fse_dist;
fse_status fse_cuda_nccl_unique_id(void* id128);
fse_status fse_cuda_dist_create(fse_cuda_ctx* ctx, int rank, int nranks, const void* id128,
                                fse_dist** out);
void fse_cuda_dist_destroy(fse_dist* d);
fse_status fse_cuda_dist_total_sum(fse_dist* d, const fse_config* cfg, int kind,
                                   const double* d_pos, const double* d_str, int64_t n_own,
                                   int64_t n_total, const double* d_tgt, int64_t nt_own, int tas,
                                   const fse_green* green, double* d_u);
/* one process, several GPUs: a multi-device context (one fse_cuda_ctx per device and
 * the NCCL communicators of ncclCommInitAll) and fse::total_sum over it with HOST
 * buffers: the points are partitioned by owner, every device runs its rank of the
 * partitioned evaluation in its own host thread, u comes back in caller order.  The
 * Green's table: green_full (the reference layout, (2 Mtilde)^3 host doubles, e.g.
 * fse::MollifiedGreen::fourier) uploaded to every device, or NULL to precompute it on
 * every device; cached by kind, geometry and table pointer.
 * tas: -1 detect by value (ewald.cpp:405-407), 0 no, 1 yes.  tm (optional) accumulates
 * only `total` (the call's wall clock, transfers included). */
typedef struct fse_multi fse_multi;
fse_status fse_cuda_multi_create(const int* devices, int ndev, fse_multi** out);
void fse_cuda_multi_destroy(fse_multi* m);
const char* fse_cuda_multi_last_error(const fse_multi* m);
fse_status fse_cuda_multi_total_sum(fse_multi* m, const fse_config* cfg, int kind,
                                    const double* pos, const double* str, int64_t n,
                                    double box_side, const double* tgt, int64_t nt, int tas,
                                    const double* green_full, double* u, fse_timings* tm);
/* owner rank of each of n host points (x = pos[3 i]) for nranks slabs (host, no GPU) */
fse_status fse_dist_owner(const fse_config* cfg, int nranks, const double* pos, int64_t n,
                          int32_t* owner);
/* bit masks of the ranks that need each host point as a source (ghost rule) or as a
 * target (quadrature share); the owner's bit is always set (host, no GPU) */
fse_status fse_dist_masks(const fse_config* cfg, int nranks, const double* pos, int64_t n,
                          int targets, uint32_t* mask);
/* the whole partitioned algorithm with nranks VIRTUAL ranks on this context's device
 * (exchanges as device copies): partitions all n points by the ownership rule, runs
 * every step of every rank, returns u for all targets in caller order (tests).  prof
 * (optional, nranks x 6 x 2 doubles): per rank and step (classify, pack, forward, scale,
 * inverse, finish) the step's time with the rank alone on the device (ms) and the bytes
 * it sends to other ranks -- the per-rank work of a multi-GPU run, measured on one GPU */
fse_status fse_cuda_dist_virtual_total_sum(fse_cuda_ctx* ctx, int nranks, const fse_config* cfg,
                                           int kind, const double* d_pos, const double* d_str,
                                           int64_t n, const double* d_tgt, int64_t nt, int tas,
                                           const fse_green* green, double* d_u, double* prof);

/* measured FP64 DFMA throughput of this device (TFLOP/s): roofline denominator */
fse_status fse_cuda_fp64_peak(fse_cuda_ctx* ctx, double* tflops);
/* overlap the real-space sum (second stream) with the Fourier part of total sums
 * (default 1; 0 serialises them so fse_cuda_kernel_ms reports isolated stage times;
 * env FSE_SERIAL sets the default to 0).  Results are identical either way. */
fse_status fse_cuda_set_overlap(fse_cuda_ctx* ctx, int on);
/* work of the last real-space pair kernel: (target, source) candidates tested and
 * accepted pairs (0 < r^2 <= rc^2) -- the real-space roofline numerator */
fse_status fse_cuda_realspace_counts(fse_cuda_ctx* ctx, uint64_t* candidates, uint64_t* pairs);

/* ---- config: replaces fse::make_config (ewald.cpp:103-134) -------------- */
fse_status fse_make_config(double L, double xi, double rc, int M, int P, double sf,
                           fse_config* out, char* err, size_t errlen);

/* ---- Green's function: replaces fse::precompute_mollified_green
 *      (greens.cpp:48-113), computed on the GPU ---------------------------- */
fse_status fse_cuda_green_precompute(fse_cuda_ctx* ctx, int green_kind, double Ltilde,
                                     int Mtilde, double sf, fse_green** out);
/* upload a host table in the reference layout: (2 Mtilde)^3 doubles, standard FFT order */
fse_status fse_cuda_green_upload(fse_cuda_ctx* ctx, int green_kind, double Ltilde,
                                 int Mtilde, double h, double R, const double* fourier_full,
                                 fse_green** out);
/* download the full (2 Mtilde)^3 table (reference layout) */
fse_status fse_cuda_green_download(fse_cuda_ctx* ctx, const fse_green* g, double* fourier_full);
/* kind, Ltilde, h, R, Mtilde */
fse_status fse_cuda_green_info(const fse_green* g, int* green_kind, double* Ltilde, double* h,
                               double* R, int* Mtilde);
void fse_cuda_green_free(fse_green* g);
/* FSEG binary cache (greens.cpp:141-203): same on-disk format */
fse_status fse_cuda_green_save(fse_cuda_ctx* ctx, const fse_green* g, const char* path);
fse_status fse_cuda_green_load(fse_cuda_ctx* ctx, const char* path, fse_green** out);

/* ---- hot path ----------------------------------------------------------- */
/* replaces fse::total_sum (ewald.cpp:394-415).  targets_are_sources: -1 detect
 * by value (std::equal, ewald.cpp:405-407), 0 no, 1 yes. */
fse_status fse_cuda_total_sum(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                              const double* pos, const double* str, int64_t n,
                              double box_side, const double* targets, int64_t nt,
                              int targets_are_sources, const fse_green* green, double* u,
                              fse_timings* timings);
fse_status fse_cuda_total_sum_dev(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                  const double* d_pos, const double* d_str, int64_t n,
                                  double box_side, const double* d_targets, int64_t nt,
                                  int targets_are_sources, const fse_green* green, double* d_u,
                                  fse_timings* timings);
/* replaces fse::fourier_sum (ewald.cpp:295-392) */
fse_status fse_cuda_fourier_sum(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                const double* pos, const double* str, int64_t n,
                                double box_side, const double* targets, int64_t nt,
                                const fse_green* green, double* u, fse_timings* timings);
/* replaces fse::real_space_sum (realspace.cpp:86-149) */
fse_status fse_cuda_real_space_sum(fse_cuda_ctx* ctx, int kind, const double* pos,
                                   const double* str, int64_t n, double box_side, double xi,
                                   double rc, const double* targets, int64_t nt, double* u);
/* replaces fse::spread (ewald.cpp:136-214): grid = a planes of Mtilde^3 */
fse_status fse_cuda_spread(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                           const double* pos, const double* str, int64_t n, double box_side,
                           double* grid);
/* spread(..., use_fgg) (ewald.hpp:45-46): use_fgg = 0 builds the per-axis weights with
 * one exp per node (axis_weights_naive, ewald.cpp:53-66) instead of the FGG
 * recurrence (ewald.cpp:33-51) */
fse_status fse_cuda_spread_ex(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                              const double* pos, const double* str, int64_t n, double box_side,
                              int use_fgg, double* grid);
/* replaces fse::kspace_scale (ewald.cpp:216-293) on full D^3 interleaved complex
 * planes: ghat a planes in, 3 planes out (D = 2 Mtilde) */
fse_status fse_cuda_kspace_scale(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                 const fse_green* green, const double* ghat, double* out);
/* replaces fse::build_cell_list (realspace.cpp:65-84) plus the bucket-contiguous
 * order of realspace.cpp:95-109.  Call with bstart == NULL to get dims first;
 * bstart has dims^3 + 1 entries, perm n entries (source indices, ascending per bucket). */
fse_status fse_cuda_build_cell_list(fse_cuda_ctx* ctx, const double* pos, int64_t n,
                                    double box_side, double rc, double domain_pad, int* dims,
                                    double* cell_side, double* origin, int64_t* bstart,
                                    int64_t* perm);
/* per-point support start indices i0 (ewald.cpp:33-51), n x 3 ints; FSE_EINVAL
 * if a support leaves the grid (ewald.cpp:87-91) */
fse_status fse_cuda_support_index(fse_cuda_ctx* ctx, const fse_config* cfg, const double* pos,
                                  int64_t n, int32_t* i0);
/* replaces fse::direct_sum (kernels.cpp:59-82), O(N NT) on the GPU */
fse_status fse_cuda_direct_sum(fse_cuda_ctx* ctx, int kind, const double* pos,
                               const double* str, int64_t n, const double* targets, int64_t nt,
                               int exclude_self, double* u);
/* the FFT seam (fft.hpp:11,14): in-place 3D C2C on interleaved complex host data;
 * inverse scales by 1/(n0 n1 n2) */
fse_status fse_cuda_fft3d(fse_cuda_ctx* ctx, double* data, int n0, int n1, int n2, int inverse);
/* diagnostics: the fused x pass of the hot path (forward x-FFT, k-space multiplier
 * with the Nyquist-exact Hermitian average and 1/D^3, inverse x-FFT, window x < Mtilde;
 * the kspace_scale of ewald.cpp:216-293 on the pruned layout) applied to a pseudo-random
 * spectrum C[c][x][ky][kz] = splitmix64-derived values (seed), with the Green's table of
 * `green`, or (green == NULL) a pseudo-random half table.  Returns out = nprobe x 3 x
 * Mtilde complex (interleaved) results at the columns (ky[p], kz[p]) and gcol = nprobe x D
 * the table values G[kx][ky[p]][kz[p]] used there. */
fse_status fse_cuda_xscale_probe(fse_cuda_ctx* ctx, const fse_config* cfg, int kind,
                                 const fse_green* green, uint64_t seed, int nprobe,
                                 const int* ky, const int* kz, double* out, double* gcol);
/* diagnostics: the hand-written fp64 FFT engine of the hot path on `ncols` contiguous
 * interleaved-complex columns of length D, in place, unnormalised (sign -1 / +1) */
fse_status fse_cuda_fft_columns(fse_cuda_ctx* ctx, int D, int ncols, double* data, int inverse);

#ifdef __cplusplus
}
#endif

#endif /* FSE_CUDA_H */
