/*
 * fse_oracle.h -- TEST INFRASTRUCTURE: plain-C restatement of the reference's
 * free-space Spectral Ewald hot path (fse::total_sum and everything under it).
 *
 * This is the CHECKER for the CUDA product, never part of it.  It is pinned
 * against the reference itself (oracle/_ref, the reference compiled from its
 * own sources) and against the reference's known-answer tests restated in
 * tests/test_oracle_*.py.
 *
 * Conventions: positions are N x 3 AoS doubles; strengths N x a doubles
 * (a = 3, or 9 for the stresslet, f_lm at 3l+m); velocities NT x 3.
 * Kinds: 0 stokeslet, 1 stresslet, 2 rotlet.  Green kinds: 0 harmonic,
 * 1 biharmonic.  Return codes: 0 ok, 1 invalid_argument, 2 domain_error.
 */
#ifndef FSE_ORACLE_H
#define FSE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double L, xi, rc;
    int M, P;
    double h, d, m, eta, deltaL, Ltilde;
    int Mtilde;
    double kinf, R, sf;
    int deterministic;
} or_cfg;

const char* or_last_error(void);

int or_make_config(double L, double xi, double rc, int M, int P, double sf, or_cfg* out);

int or_build_cell_list(const double* pos, int64_t n, double L, double rc, double pad,
                       int* dims, double* cell_side, double* origin, int64_t* bstart,
                       int64_t* perm);

int or_eval_real_kernel(int kind, const double* r, double xi, const double* f, double* out);
int or_eval_kernel(int kind, const double* r, const double* f, double* out);

int or_real_space_sum(int kind, const double* pos, const double* str, int64_t n, double L,
                      double xi, double rc, const double* tgt, int64_t nt, double* u);

/* per-point support: first index per axis and the 3P FGG axis weights */
int or_support(const or_cfg* cfg, const double* x, int use_fgg, int* i0, double* w);
/* i0 of n points (n x 3 ints), or_support's index rule; returns #points out of the grid */
int64_t or_support_index(const or_cfg* cfg, const double* pts, int64_t n, int* i0);

int or_spread(const or_cfg* cfg, int kind, const double* pos, const double* str, int64_t n,
              double box_side, int use_fgg, double* grid);

int or_kspace_scale(const or_cfg* cfg, int kind, const double* green, const double* ghat,
                    double* out);

/* w_out (optional): the 3 windowed real grids Mtilde^3 before quadrature */
int or_fourier_sum(const or_cfg* cfg, int kind, const double* pos, const double* str,
                   int64_t n, double box_side, const double* tgt, int64_t nt,
                   const double* green, double* u, double* w_out);

int or_total_sum(const or_cfg* cfg, int kind, const double* pos, const double* str,
                 int64_t n, double box_side, const double* tgt, int64_t nt,
                 const double* green, double* u);

double or_hhat(double k, double R);
double or_bhat(double k, double R);
int or_precompute_green(int gkind, double Ltilde, int Mtilde, double sf, double* out);

int or_direct_sum(int kind, const double* pos, const double* str, int64_t n,
                  const double* tgt, int64_t nt, int exclude_self, double* u);

void or_fft3d(double* data, int n0, int n1, int n2, int inverse);

#ifdef __cplusplus
}
#endif

#endif
