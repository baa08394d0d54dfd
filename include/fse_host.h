/*
 * fse_host.h -- host-only helpers exported by libfse_b200.so (not on the GPU
 * hot path): deterministic input generators.
 */
#ifndef FSE_HOST_H
#define FSE_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Replaces fse::generate_system (harness.cpp:47-66): std::mt19937_64(seed),
 * u = (rng() >> 11) 2^-53; all positions L*u first, then strengths 2u-1.
 * kind 1 (stresslet) draws 9 components per point, else 3.  Returns 0 on success. */
int fse_generate_system(int kind, int64_t n, double L, uint64_t seed, double* pos, double* str);

/* SURVEY.md 8(d) workload generators, unit box, std::mt19937_64(seed),
 * normals by Box-Muller (u1 = ((rng()>>11)+1) 2^-53):
 *   FSE_WL_UNIFORM          positions U[0,1)^3, then N(0,1) 3-vector strengths (cfg1, cfg2)
 *   FSE_WL_SPHERE           sphere radius 0.5 about the box centre, f = n q^T, q ~ N(0,1)^3 (cfg3)
 *   FSE_WL_CLUSTERED        32 blobs, sigma 0.03, clamped to [0, 1) (cfg4)
 *   FSE_WL_UNIFORM_TARGETS  as UNIFORM plus n distinct U[0,1)^3 targets (cfg5) */
enum {
    FSE_WL_UNIFORM = 1,
    FSE_WL_SPHERE = 3,
    FSE_WL_CLUSTERED = 4,
    FSE_WL_UNIFORM_TARGETS = 5
};
int fse_generate_workload(int which, int64_t n, uint64_t seed, double* pos, double* str,
                          double* tgt);

/* ---- closed-form truncation-error estimates and parameter selection (host scalar
 * math).  Replace fse::fourier_error_estimate, real_error_estimate,
 * error_budget, reference_velocity_rms and select_parameters
 * (/root/reference/proj/include/fse/estimates.hpp:11-40, estimates.cpp:13-126).
 * Status codes as in fse_cuda.h (FSE_EINVAL = std::invalid_argument). */
#include "fse_cuda.h"

typedef struct {
    int kind;
    double xi, rc, k_inf, L, R;
    double Q;                      /* sum of squared strength components */
    double predicted_real_rms;
    double predicted_fourier_rms;
} fse_error_budget_t;

fse_status fse_fourier_error_estimate(int kind, double Q, double xi, double k_inf, double L,
                                      double R, double* out);
fse_status fse_real_error_estimate(int kind, double Q, double xi, double rc, double L,
                                   double* out);
fse_status fse_error_budget(int kind, const fse_config* cfg, double Q, fse_error_budget_t* out);
fse_status fse_reference_velocity_rms(int kind, double Q, double L, uint64_t N, double* out);
/* smallest rc and even M meeting the relative RMS tolerance; *feasible = 0 when the
 * real-space budget needs rc > L sqrt(3) (direct summation recommended) */
fse_status fse_select_parameters(int kind, uint64_t N, double L, double Q, double xi, double tol,
                                 fse_config* out, int* feasible);

/* Host-only planner query (no GPU needed): can the FFT passes of a grid of D = 2 Mtilde
 * points run for this kernel kind?  FSE_OK, or FSE_EINVAL when D exceeds the engines
 * (total_sum / fourier_sum then fail the same way before allocating anything).
 * *engine: 0 Stockham (generic_stage = 1: with a generic O(p^2) first stage),
 * 1-4 register engines 624 / 1200 / 704 / 242, 5-7 Bluestein on 400 / 624 / 1024. */
fse_status fse_fft_plan_query(int D, int kind, int* engine, int* generic_stage);

#ifdef __cplusplus
}
#endif

#endif
