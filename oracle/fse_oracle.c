/*
 * fse_oracle.c -- TEST INFRASTRUCTURE: plain-C restatement of the reference's
 * free-space Spectral Ewald hot path.  The CHECKER for the CUDA product; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Pinned against the reference compiled from its own sources (oracle/_ref)
 * in tests/test_oracle_pin.py, and against the reference's known-answer
 * tests restated in tests/test_oracle_known_answers.py.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  Arithmetic is written in the reference's
 * operation order; it is built without FMA contraction (x86-64 -O2), like
 * the reference.
 *
 * Deliberate difference: spreading is deterministic (per-node summation in
 * a stable spatial order; the reference merges per-thread grids in an
 * unspecified order, SPEC.md:327 documents that 1e-13-level nondeterminism).
 */
#include "fse_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "fftw_shim/fft_core.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { K_STOKESLET = 0, K_STRESSLET = 1, K_ROTLET = 2 };

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* or_last_error(void) { return g_err; }

static int arity_of(int kind) { return kind == K_STRESSLET ? 9 : 3; }

/* ewald.cpp:103-134 */
int or_make_config(double L, double xi, double rc, int M, int P, double sf, or_cfg* c) {
    if (!(L > 0) || !(xi > 0) || !(rc > 0) || M < 1 || P < 2)
        return fail(1, "make_config: all parameters must be positive");
    if (P % 2 != 0) return fail(1, "make_config: P must be even");
    memset(c, 0, sizeof *c);
    c->L = L;
    c->xi = xi;
    c->rc = rc;
    c->M = M;
    c->P = P;
    c->h = L / M;
    c->d = c->h * P;
    c->m = 0.976 * sqrt(M_PI * P);
    c->eta = (xi * c->d / c->m) * (xi * c->d / c->m);
    double raw = c->d;
    if (c->eta < 1.0) {
        double alt = sqrt(2.0 * (1.0 - c->eta)) * c->m / xi;
        raw = c->d > alt ? c->d : alt;
    }
    const int pad = (int)ceil(raw / c->h - 1e-12);
    c->deltaL = pad * c->h;
    c->Mtilde = M + pad;
    c->Ltilde = c->Mtilde * c->h;
    c->kinf = M_PI * c->Mtilde / c->Ltilde;
    c->R = sqrt(3.0) * c->Ltilde;
    c->sf = sf > 0 ? sf : 1.0 + sqrt(3.0);
    if (c->sf < 1.0 + sqrt(3.0) - 1e-12) return fail(1, "make_config: sf below 1 + sqrt(3)");
    if (P > c->Mtilde) return fail(1, "make_config: Gaussian support exceeds grid");
    return 0;
}

/* ---------------------------------------------------------------- cell list */

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* realspace.cpp:60-63 */
static int cell_of(double coord, double origin, double side, int dim) {
    int c = (int)floor((coord - origin) / side);
    return clampi(c, 0, dim - 1);
}

/* realspace.cpp:65-84; buckets listed contiguously in ascending source index
 * (the bucket-contiguous copy of realspace.cpp:95-109). */
int or_build_cell_list(const double* pos, int64_t n, double L, double rc, double pad,
                       int* dims, double* cell_side, double* origin, int64_t* bstart,
                       int64_t* perm) {
    if (!(rc > 0)) return fail(1, "build_cell_list: rc must be positive");
    *origin = -pad;
    const double extent = L + 2.0 * pad;
    const int cap = 1 + (int)cbrt(8.0 * (double)(n > 1 ? n : 1));
    int want = (int)floor(extent / rc);
    if (want < 1) want = 1;
    const int d = want < cap ? want : cap;
    dims[0] = dims[1] = dims[2] = d;
    *cell_side = extent / d;
    if (!bstart) return 0;
    const int64_t ncell = (int64_t)d * d * d;
    int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    memset(bstart, 0, sizeof(int64_t) * (ncell + 1));
    for (int64_t i = 0; i < n; ++i) {
        const int a = cell_of(pos[3 * i], *origin, *cell_side, d);
        const int b = cell_of(pos[3 * i + 1], *origin, *cell_side, d);
        const int e = cell_of(pos[3 * i + 2], *origin, *cell_side, d);
        key[i] = ((int64_t)a * d + b) * d + e;
        bstart[key[i] + 1]++;
    }
    for (int64_t c = 0; c < ncell; ++c) bstart[c + 1] += bstart[c];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (ncell > 0 ? ncell : 1));
    memcpy(fill, bstart, sizeof(int64_t) * ncell);
    for (int64_t i = 0; i < n; ++i) perm[fill[key[i]]++] = i;
    free(fill);
    free(key);
    return 0;
}

/* ------------------------------------------------------------ pair kernels */

static const double kInvSqrtPi = 0.5641895835477562869;

/* realspace.cpp:13-58 */
int or_eval_real_kernel(int kind, const double* r, double xi, const double* f, double* out) {
    const double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    if (r2 == 0) return fail(2, "eval_real_kernel: zero separation");
    if (!(xi > 0)) return fail(1, "eval_real_kernel: xi must be positive");
    const double rn = sqrt(r2);
    const double xr = xi * rn;
    const double gauss = exp(-xr * xr);
    const double erfc_xr = erfc(xr);
    const double inv = 1.0 / rn;
    const double rh[3] = {inv * r[0], inv * r[1], inv * r[2]};
    if (kind == K_STOKESLET) {
        const double a = 2.0 * (xi * gauss * kInvSqrtPi + erfc_xr / (2.0 * rn));
        const double b = 4.0 * xi * kInvSqrtPi * gauss;
        const double amb = a - b;
        const double s = a * (rh[0] * f[0] + rh[1] * f[1] + rh[2] * f[2]);
        for (int j = 0; j < 3; ++j) out[j] = amb * f[j] + s * rh[j];
    } else if (kind == K_STRESSLET) {
        const double c1 = -(2.0 / rn) *
            (3.0 * erfc_xr / rn + 2.0 * xi * kInvSqrtPi * (3.0 + 2.0 * xr * xr) * gauss);
        const double c2 = 4.0 * xi * xi * xi * kInvSqrtPi * gauss * rn;
        double rfr = 0, f_r[3] = {0, 0, 0}, r_f[3] = {0, 0, 0};
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) {
                rfr += rh[l] * f[3 * l + m] * rh[m];
                f_r[l] += f[3 * l + m] * rh[m];
                r_f[m] += rh[l] * f[3 * l + m];
            }
        const double trf = f[0] + f[4] + f[8];
        const double s = c1 * rfr + c2 * trf;
        for (int j = 0; j < 3; ++j) out[j] = s * rh[j] + c2 * (f_r[j] + r_f[j]);
    } else {
        const double c = erfc_xr / r2 + 2.0 * xi * kInvSqrtPi * gauss / rn;
        out[0] = c * (f[1] * rh[2] - f[2] * rh[1]);
        out[1] = c * (f[2] * rh[0] - f[0] * rh[2]);
        out[2] = c * (f[0] * rh[1] - f[1] * rh[0]);
    }
    return 0;
}

/* kernels.cpp:27-57 */
int or_eval_kernel(int kind, const double* r, const double* f, double* out) {
    const double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    if (r2 == 0) return fail(2, "eval_kernel: zero separation");
    const double rn = sqrt(r2);
    if (kind == K_STOKESLET) {
        const double rf = r[0] * f[0] + r[1] * f[1] + r[2] * f[2];
        const double a = 1.0 / rn, b = rf / (r2 * rn);
        for (int j = 0; j < 3; ++j) out[j] = a * f[j] + b * r[j];
    } else if (kind == K_STRESSLET) {
        double rfr = 0;
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) rfr += r[l] * f[3 * l + m] * r[m];
        const double c = -6.0 * rfr / (r2 * r2 * rn);
        for (int j = 0; j < 3; ++j) out[j] = c * r[j];
    } else {
        const double inv_r3 = 1.0 / (r2 * rn);
        out[0] = (f[1] * r[2] - f[2] * r[1]) * inv_r3;
        out[1] = (f[2] * r[0] - f[0] * r[2]) * inv_r3;
        out[2] = (f[0] * r[1] - f[1] * r[0]) * inv_r3;
    }
    return 0;
}

/* realspace.cpp:86-149: 27-cell neighbourhood in lexicographic (di,dj,dk)
 * order, sources in bucket order, closed ball 0 < d2 <= rc2. */
int or_real_space_sum(int kind, const double* pos, const double* str, int64_t n, double L,
                      double xi, double rc, const double* tgt, int64_t nt, double* u) {
    if (!(xi > 0) || !(rc > 0)) return fail(1, "real_space_sum: xi and rc must be positive");
    int dims[3];
    double side, origin;
    or_build_cell_list(pos, n, L, rc, 0.0, dims, &side, &origin, NULL, NULL);
    const int64_t ncell = (int64_t)dims[0] * dims[1] * dims[2];
    int64_t* bstart = (int64_t*)malloc(sizeof(int64_t) * (ncell + 1));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    or_build_cell_list(pos, n, L, rc, 0.0, dims, &side, &origin, bstart, perm);
    const int a = arity_of(kind);
    double* sp = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
    double* ss = (double*)malloc(sizeof(double) * a * (n > 0 ? n : 1));
    for (int64_t q = 0; q < n; ++q) {
        memcpy(sp + 3 * q, pos + 3 * perm[q], 3 * sizeof(double));
        memcpy(ss + a * q, str + a * perm[q], a * sizeof(double));
    }
    const double rc2 = rc * rc;
    const int d = dims[0];
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t m = 0; m < nt; ++m) {
        const double* x = tgt + 3 * m;
        const int ci = cell_of(x[0], origin, side, d);
        const int cj = cell_of(x[1], origin, side, d);
        const int ck = cell_of(x[2], origin, side, d);
        double acc[3] = {0, 0, 0};
        for (int di = -1; di <= 1; ++di) {
            const int i = ci + di;
            if (i < 0 || i >= d) continue;
            for (int dj = -1; dj <= 1; ++dj) {
                const int j = cj + dj;
                if (j < 0 || j >= d) continue;
                for (int dk = -1; dk <= 1; ++dk) {
                    const int k = ck + dk;
                    if (k < 0 || k >= d) continue;
                    const int64_t b = ((int64_t)i * d + j) * d + k;
                    for (int64_t q = bstart[b]; q < bstart[b + 1]; ++q) {
                        const double r[3] = {x[0] - sp[3 * q], x[1] - sp[3 * q + 1],
                                             x[2] - sp[3 * q + 2]};
                        const double d2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
                        if (d2 == 0 || d2 > rc2) continue;
                        double v[3];
                        or_eval_real_kernel(kind, r, xi, ss + a * q, v);
                        acc[0] += v[0];
                        acc[1] += v[1];
                        acc[2] += v[2];
                    }
                }
            }
        }
        u[3 * m] = acc[0];
        u[3 * m + 1] = acc[1];
        u[3 * m + 2] = acc[2];
    }
    free(sp);
    free(ss);
    free(bstart);
    free(perm);
    return 0;
}

/* ------------------------------------------------------------------ spread */

static double alpha_of(const or_cfg* c) { return 2.0 * c->xi * c->xi / c->eta; }
static double prefac_of(const or_cfg* c) {
    return pow(2.0 * c->xi * c->xi / (M_PI * c->eta), 1.5);
}

/* ewald.cpp:33-66 (FGG and naive axis weights); check_support :87-91 */
int or_support(const or_cfg* c, const double* x, int use_fgg, int* i0, double* w) {
    const int P = c->P;
    const double alpha = alpha_of(c);
    const double origin = -c->deltaL / 2;
    for (int axis = 0; axis < 3; ++axis) {
        const double s = (x[axis] - origin) / c->h;
        const int first = (int)ceil(s - 0.5 * P);
        i0[axis] = first;
        double* wa = w + axis * P;
        if (use_fgg) {
            const double x0 = (first - s) * c->h;
            const double e0 = exp(-alpha * x0 * x0);
            const double ratio = exp(-2.0 * alpha * x0 * c->h);
            double r = 1.0;
            for (int p = 0; p < P; ++p) {
                const double q = exp(-alpha * (p * c->h) * (p * c->h));
                wa[p] = e0 * r * q;
                r *= ratio;
            }
        } else {
            for (int p = 0; p < P; ++p) {
                const double dx = (first + p - s) * c->h;
                wa[p] = exp(-alpha * dx * dx);
            }
        }
    }
    for (int axis = 0; axis < 3; ++axis)
        if (i0[axis] < 0 || i0[axis] + P > c->Mtilde)
            return fail(1, "spread/quadrature: point support exceeds grid");
    return 0;
}

/* or_support over many points (test convenience, ewald.cpp:33-51 index rule) */
int64_t or_support_index(const or_cfg* c, const double* pts, int64_t n, int* i0) {
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t q = 0; q < n; ++q) {
        double w[3 * 64];
        double* wa = c->P <= 64 ? w : (double*)malloc(sizeof(double) * 3 * c->P);
        if (or_support(c, pts + 3 * q, 1, i0 + 3 * q, wa)) ++bad;
        if (wa != w) free(wa);
    }
    return bad;
}

/* ewald.cpp:70-85: block key, stable order within a block */
static int64_t* spatial_order(const double* pts, int64_t n, double block, double L) {
    int nb = (int)(L / block);
    if (nb < 1) nb = 1;
    const double inv = nb / L;
    const int64_t nk = (int64_t)nb * nb * nb;
    int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t* cnt = (int64_t*)calloc(nk + 1, sizeof(int64_t));
    for (int64_t q = 0; q < n; ++q) {
        const int i = clampi((int)(pts[3 * q] * inv), 0, nb - 1);
        const int j = clampi((int)(pts[3 * q + 1] * inv), 0, nb - 1);
        const int k = clampi((int)(pts[3 * q + 2] * inv), 0, nb - 1);
        key[q] = ((int64_t)i * nb + j) * nb + k;
        cnt[key[q] + 1]++;
    }
    for (int64_t b = 0; b < nk; ++b) cnt[b + 1] += cnt[b];
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    for (int64_t q = 0; q < n; ++q) order[cnt[key[q]]++] = q;
    free(cnt);
    free(key);
    return order;
}

/* ewald.cpp:136-214.  Parallel over x-planes of the grid: each thread owns a
 * range of planes and applies, in the spatial order, every point whose
 * support meets its planes -- per-node summation order is the sequential
 * one, so the result is deterministic. */
int or_spread(const or_cfg* c, int kind, const double* pos, const double* str, int64_t n,
              double box_side, int use_fgg, double* grid) {
    if (fabs(box_side - c->L) > 1e-12 * c->L)
        return fail(1, "spread: config box does not match system");
    const int Mt = c->Mtilde, P = c->P, a = arity_of(kind);
    const size_t vol = (size_t)Mt * Mt * Mt;
    memset(grid, 0, sizeof(double) * vol * a);
    const double prefac = prefac_of(c);
    int* i0s = (int*)malloc(sizeof(int) * 3 * (n > 0 ? n : 1));
    double* ws = (double*)malloc(sizeof(double) * 3 * P * (n > 0 ? n : 1));
    int bad = 0;
    for (int64_t q = 0; q < n; ++q)
        if (or_support(c, pos + 3 * q, use_fgg, i0s + 3 * q, ws + 3 * P * q)) bad = 1;
    if (bad) {
        free(i0s);
        free(ws);
        return 1;
    }
    int64_t* order = spatial_order(pos, n, c->d, c->L);
#pragma omp parallel
    {
#ifdef _OPENMP
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
#else
        const int t = 0, nt = 1;
#endif
        const int lo = (int)((int64_t)Mt * t / nt), hi = (int)((int64_t)Mt * (t + 1) / nt);
        for (int64_t s = 0; s < n; ++s) {
            const int64_t q = order[s];
            const int* i0 = i0s + 3 * q;
            const double* w = ws + 3 * P * q;
            const double* f = str + a * q;
            for (int i = 0; i < P; ++i) {
                const int gi = i0[0] + i;
                if (gi < lo || gi >= hi) continue;
                const double wx = w[i];
                for (int j = 0; j < P; ++j) {
                    const double wxy = wx * w[P + j];
                    const size_t base = ((size_t)gi * Mt + (i0[1] + j)) * Mt + i0[2];
                    for (int k = 0; k < P; ++k) {
                        const double wt = prefac * wxy * w[2 * P + k];
                        for (int cc = 0; cc < a; ++cc) grid[cc * vol + base + k] += wt * f[cc];
                    }
                }
            }
        }
    }
    free(order);
    free(i0s);
    free(ws);
    return 0;
}

/* ------------------------------------------------------------- k-space */

/* ewald.cpp:216-293 on the full D^3 C2C spectrum (interleaved complex). */
int or_kspace_scale(const or_cfg* c, int kind, const double* green, const double* ghat,
                    double* out) {
    const int D = 2 * c->Mtilde;
    const size_t tot = (size_t)D * D * D;
    const double dk = M_PI / c->Ltilde;
    const double inv4xi2 = 1.0 / (4.0 * c->xi * c->xi);
    double* kax = (double*)malloc(sizeof(double) * D);
    for (int q = 0; q < D; ++q) kax[q] = dk * (q < D / 2 ? q : q - D);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            for (int l = 0; l < D; ++l) {
                const size_t idx = ((size_t)i * D + j) * D + l;
                const double k[3] = {kax[i], kax[j], kax[l]};
                const double k2 = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
                const double rem = exp(-(1.0 - c->eta) * k2 * inv4xi2);
                const double gval = green[idx];
                if (kind == K_STOKESLET) {
                    const double b = -gval * (1.0 + k2 * inv4xi2) * rem;
                    const double* g0 = ghat + 2 * idx;
                    const double* g1 = ghat + 2 * (tot + idx);
                    const double* g2 = ghat + 2 * (2 * tot + idx);
                    const double kgr = k[0] * g0[0] + k[1] * g1[0] + k[2] * g2[0];
                    const double kgi = k[0] * g0[1] + k[1] * g1[1] + k[2] * g2[1];
                    const double* g[3] = {g0, g1, g2};
                    for (int p = 0; p < 3; ++p) {
                        out[2 * (p * tot + idx)] = b * (k2 * g[p][0] - k[p] * kgr);
                        out[2 * (p * tot + idx) + 1] = b * (k2 * g[p][1] - k[p] * kgi);
                    }
                } else if (kind == K_STRESSLET) {
                    const double b = gval * (1.0 + k2 * inv4xi2) * rem;
                    double ar[3] = {0, 0, 0}, ai[3] = {0, 0, 0};
                    double br[3] = {0, 0, 0}, bi[3] = {0, 0, 0};
                    double trr = 0, tri = 0, kgkr = 0, kgki = 0;
                    for (int p = 0; p < 3; ++p) {
                        trr += ghat[2 * ((3 * p + p) * tot + idx)];
                        tri += ghat[2 * ((3 * p + p) * tot + idx) + 1];
                        for (int q = 0; q < 3; ++q) {
                            const double gr = ghat[2 * ((3 * p + q) * tot + idx)];
                            const double gi = ghat[2 * ((3 * p + q) * tot + idx) + 1];
                            ar[p] += gr * k[q];
                            ai[p] += gi * k[q];
                            br[q] += k[p] * gr;
                            bi[q] += k[p] * gi;
                        }
                    }
                    for (int p = 0; p < 3; ++p) {
                        kgkr += k[p] * ar[p];
                        kgki += k[p] * ai[p];
                    }
                    for (int p = 0; p < 3; ++p) {
                        const double vr = k2 * (ar[p] + br[p] + k[p] * trr) - 2.0 * k[p] * kgkr;
                        const double vi = k2 * (ai[p] + bi[p] + k[p] * tri) - 2.0 * k[p] * kgki;
                        /* (0, -b) * (vr + i vi) = b vi - i b vr */
                        out[2 * (p * tot + idx)] = b * vi;
                        out[2 * (p * tot + idx) + 1] = -b * vr;
                    }
                } else {
                    const double cm = -gval * rem; /* c = (0, cm) */
                    const double* g0 = ghat + 2 * idx;
                    const double* g1 = ghat + 2 * (tot + idx);
                    const double* g2 = ghat + 2 * (2 * tot + idx);
                    const double vr[3] = {g1[0] * k[2] - g2[0] * k[1], g2[0] * k[0] - g0[0] * k[2],
                                          g0[0] * k[1] - g1[0] * k[0]};
                    const double vi[3] = {g1[1] * k[2] - g2[1] * k[1], g2[1] * k[0] - g0[1] * k[2],
                                          g0[1] * k[1] - g1[1] * k[0]};
                    for (int p = 0; p < 3; ++p) {
                        out[2 * (p * tot + idx)] = -cm * vi[p];
                        out[2 * (p * tot + idx) + 1] = cm * vr[p];
                    }
                }
            }
    free(kax);
    return 0;
}

void or_fft3d(double* data, int n0, int n1, int n2, int inverse) {
    /* fft.cpp:28-37: inverse is scaled by 1/(n0 n1 n2) in a separate pass */
    fc_fft3d(data, n0, n1, n2, inverse ? +1 : -1);
    if (inverse) {
        const double scale = 1.0 / ((double)n0 * n1 * n2);
        const size_t tot = (size_t)n0 * n1 * n2;
        for (size_t q = 0; q < 2 * tot; ++q) data[q] *= scale;
    }
}

/* ewald.cpp:295-392 */
int or_fourier_sum(const or_cfg* c, int kind, const double* pos, const double* str,
                   int64_t n, double box_side, const double* tgt, int64_t nt,
                   const double* green, double* u, double* w_out) {
    for (int64_t m = 0; m < nt; ++m)
        for (int d = 0; d < 3; ++d)
            if (!(tgt[3 * m + d] >= 0 && tgt[3 * m + d] <= c->L))
                return fail(1, "fourier_sum: target outside [0,L]^3");
    const int Mt = c->Mtilde, D = 2 * Mt, a = arity_of(kind), P = c->P;
    const size_t vol = (size_t)Mt * Mt * Mt, tot = (size_t)D * D * D;
    double* grid = (double*)malloc(sizeof(double) * vol * a);
    int rc = or_spread(c, kind, pos, str, n, box_side, 1, grid);
    if (rc) {
        free(grid);
        return rc;
    }
    double* ghat = (double*)calloc(2 * tot * a, sizeof(double));
    for (int cc = 0; cc < a; ++cc) {
        double* gh = ghat + 2 * tot * cc;
        for (int i = 0; i < Mt; ++i)
            for (int j = 0; j < Mt; ++j)
                for (int l = 0; l < Mt; ++l)
                    gh[2 * (((size_t)i * D + j) * D + l)] =
                        grid[cc * vol + ((size_t)i * Mt + j) * Mt + l];
        fc_fft3d(gh, D, D, D, -1);
    }
    free(grid);
    double* what = (double*)malloc(sizeof(double) * 2 * tot * 3);
    or_kspace_scale(c, kind, green, ghat, what);
    free(ghat);
    double* w = (double*)malloc(sizeof(double) * vol * 3);
    for (int cc = 0; cc < 3; ++cc) {
        double* wh = what + 2 * tot * cc;
        or_fft3d(wh, D, D, D, 1);
        for (int i = 0; i < Mt; ++i)
            for (int j = 0; j < Mt; ++j)
                for (int l = 0; l < Mt; ++l)
                    w[cc * vol + ((size_t)i * Mt + j) * Mt + l] =
                        wh[2 * (((size_t)i * D + j) * D + l)];
    }
    free(what);
    if (w_out) memcpy(w_out, w, sizeof(double) * vol * 3);
    const double prefac = prefac_of(c);
    const double h3 = c->h * c->h * c->h;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t m = 0; m < nt; ++m) {
        int i0[3];
        double wt[3 * 64];
        double* wa = P <= 64 ? wt : (double*)malloc(sizeof(double) * 3 * P);
        if (or_support(c, tgt + 3 * m, 1, i0, wa)) {
            bad = 1;
        } else {
            double acc[3] = {0, 0, 0};
            for (int i = 0; i < P; ++i) {
                const double wx = wa[i];
                for (int j = 0; j < P; ++j) {
                    const double wxy = wx * wa[P + j];
                    const size_t base = ((size_t)(i0[0] + i) * Mt + (i0[1] + j)) * Mt + i0[2];
                    for (int l = 0; l < P; ++l) {
                        const double ww = wxy * wa[2 * P + l];
                        acc[0] += ww * w[base + l];
                        acc[1] += ww * w[vol + base + l];
                        acc[2] += ww * w[2 * vol + base + l];
                    }
                }
            }
            const double s = h3 * prefac;
            u[3 * m] = s * acc[0];
            u[3 * m + 1] = s * acc[1];
            u[3 * m + 2] = s * acc[2];
        }
        if (wa != wt) free(wa);
    }
    free(w);
    if (bad) return fail(1, "spread/quadrature: point support exceeds grid");
    return 0;
}

/* ewald.cpp:394-415 + kernels.cpp:84-89 */
int or_total_sum(const or_cfg* c, int kind, const double* pos, const double* str,
                 int64_t n, double box_side, const double* tgt, int64_t nt,
                 const double* green, double* u) {
    int rc = or_fourier_sum(c, kind, pos, str, n, box_side, tgt, nt, green, u, NULL);
    if (rc) return rc;
    double* ur = (double*)malloc(sizeof(double) * 3 * (nt > 0 ? nt : 1));
    rc = or_real_space_sum(kind, pos, str, n, box_side, c->xi, c->rc, tgt, nt, ur);
    if (rc) {
        free(ur);
        return rc;
    }
    for (int64_t q = 0; q < 3 * nt; ++q) u[q] += ur[q];
    free(ur);
    int same = (nt == n);
    for (int64_t q = 0; same && q < 3 * n; ++q)
        if (!(tgt[q] == pos[q])) same = 0;
    if (same && kind == K_STOKESLET) {
        const double cs = -4.0 * c->xi / sqrt(M_PI);
        for (int64_t q = 0; q < n; ++q)
            for (int d = 0; d < 3; ++d) u[3 * q + d] += cs * str[3 * q + d];
    }
    return 0;
}

/* --------------------------------------------------------- Green's fns */

static double sinc(double x) {
    if (fabs(x) < 1e-8) return 1.0 - x * x / 6.0;
    return sin(x) / x;
}

/* greens.cpp:22-26 */
double or_hhat(double k, double R) {
    const double s = sinc(0.5 * R * k);
    return 2.0 * M_PI * R * R * s * s;
}

/* greens.cpp:28-46 (long double branch as in the reference) */
double or_bhat(double k, double R) {
    const double t = R * k;
    const double piR4 = M_PI * R * R * R * R;
    if (t < 0.5) {
        const double t2 = t * t;
        return piR4 * (1.0 + t2 * (-1.0 / 9.0 + t2 * (1.0 / 240.0 +
                       t2 * (-1.0 / 12600.0 + t2 * (1.0 / 1088640.0 +
                       t2 * (-1.0 / 139708800.0 + t2 / 24908083200.0))))));
    }
    const long double tl = (long double)R * k;
    const long double num = (2.0L - tl * tl) * cosl(tl) + 2.0L * tl * sinl(tl) - 2.0L;
    return (double)(4.0L * (long double)M_PI * num / (tl * tl * tl * tl) *
                    ((long double)R * R * R * R));
}

/* greens.cpp:48-113 */
int or_precompute_green(int gkind, double Ltilde, int Mtilde, double sf, double* out) {
    const double sf_min = 1.0 + sqrt(3.0);
    if (!(Ltilde > 0) || Mtilde < 1) return fail(1, "precompute_mollified_green: bad domain");
    if (sf < sf_min - 1e-12) return fail(1, "precompute_mollified_green: sf below 1 + sqrt(3)");
    const double h = Ltilde / Mtilde;
    const double R = sqrt(3.0) * Ltilde;
    int sM = (int)ceil(sf * Mtilde);
    if (sM % 2 != 0) ++sM;
    const double dk = 2.0 * M_PI / (sM * h);
    const size_t sM3 = (size_t)sM * sM * sM;
    double* grid = (double*)malloc(sizeof(double) * 2 * sM3);
    double* k2a = (double*)malloc(sizeof(double) * sM);
    for (int q = 0; q < sM; ++q) {
        const int na = q < sM / 2 ? q : q - sM;
        k2a[q] = (dk * na) * (dk * na);
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < sM; ++i)
        for (int j = 0; j < sM; ++j) {
            const double k2ij = k2a[i] + k2a[j];
            double* row = grid + 2 * (((size_t)i * sM + j) * sM);
            for (int l = 0; l < sM; ++l) {
                const double k = sqrt(k2ij + k2a[l]);
                row[2 * l] = gkind == 0 ? or_hhat(k, R) : or_bhat(k, R);
                row[2 * l + 1] = 0;
            }
        }
    free(k2a);
    or_fft3d(grid, sM, sM, sM, 1);
    const int D = 2 * Mtilde;
    const size_t tot = (size_t)D * D * D;
    double* trunc = (double*)malloc(sizeof(double) * 2 * tot);
    int* src = (int*)malloc(sizeof(int) * D);
    for (int p = 0; p < D; ++p) {
        const int off = p < Mtilde ? p : p - D;
        src[p] = off >= 0 ? off : off + sM;
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j)
            for (int l = 0; l < D; ++l) {
                const size_t o = ((size_t)i * D + j) * D + l;
                trunc[2 * o] = grid[2 * (((size_t)src[i] * sM + src[j]) * sM + src[l])];
                trunc[2 * o + 1] = 0;
            }
    free(src);
    free(grid);
    fc_fft3d(trunc, D, D, D, -1);
    for (size_t o = 0; o < tot; ++o) out[o] = trunc[2 * o];
    free(trunc);
    return 0;
}

/* kernels.cpp:59-82 */
int or_direct_sum(int kind, const double* pos, const double* str, int64_t n,
                  const double* tgt, int64_t nt, int exclude_self, double* u) {
    const int a = arity_of(kind);
    int coincident = 0;
#pragma omp parallel for schedule(static) reduction(| : coincident)
    for (int64_t m = 0; m < nt; ++m) {
        double acc[3] = {0, 0, 0};
        for (int64_t q = 0; q < n; ++q) {
            if (exclude_self && m == q) continue;
            const double r[3] = {tgt[3 * m] - pos[3 * q], tgt[3 * m + 1] - pos[3 * q + 1],
                                 tgt[3 * m + 2] - pos[3 * q + 2]};
            if (r[0] == 0 && r[1] == 0 && r[2] == 0) {
                coincident = 1;
                continue;
            }
            double v[3];
            or_eval_kernel(kind, r, str + a * q, v);
            acc[0] += v[0];
            acc[1] += v[1];
            acc[2] += v[2];
        }
        u[3 * m] = acc[0];
        u[3 * m + 1] = acc[1];
        u[3 * m + 2] = acc[2];
    }
    if (coincident) return fail(2, "direct_sum: coincident target/source point");
    return 0;
}
