// fse_estimates.cpp -- closed-form truncation-error estimates and automatic
// parameter selection (host scalar math), restating
// /root/reference/proj/src/estimates.cpp:13-126 behind the C-ABI of
// include/fse_host.h.  The estimators are the statistical (Kolafa-Perram
// style) RMS bounds of the SE papers:
//   Fourier: sqrt(Q) R k^3 / (xi^2 pi L) e^{-k^2/4xi^2}        (stokeslet)
//            sqrt(7Q/6) R k^4 / (xi^2 pi L) e^{-k^2/4xi^2}     (stresslet)
//            sqrt(8 xi^2 Q / (3 pi L^3 k)) e^{-k^2/4xi^2}      (rotlet)
//   real:    sqrt(4 Q rc / L^3) e^{-xi^2 rc^2}                 (stokeslet)
//            sqrt(112 Q xi^4 rc^3 / (9 L^3)) e^{-xi^2 rc^2}   (stresslet)
//            sqrt(8 Q / (3 L^3 rc)) e^{-xi^2 rc^2}             (rotlet)
// and the selection splits a relative RMS tolerance evenly between the two
// with a calibration factor of 2, bisects rc on the monotone real-space
// tail and takes the smallest even M meeting the Fourier budget.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "fse_cuda.h"
#include "fse_host.h"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kCalibration = 2.0;  // estimates.cpp:11

bool bad_kind(int k) { return k != FSE_STOKESLET && k != FSE_STRESSLET && k != FSE_ROTLET; }

// estimates.cpp:14-29
bool fourier_est(int kind, double Q, double xi, double kinf, double L, double R, double* out) {
    if (!(Q >= 0) || !(xi > 0) || !(kinf > 0) || !(L > 0) || !(R > 0) || bad_kind(kind))
        return false;
    const double decay = std::exp(-kinf * kinf / (4.0 * xi * xi));
    // left-to-right products, as the reference rounds them
    switch (kind) {
        case FSE_STOKESLET:
            *out = std::sqrt(Q) * R * kinf * kinf * kinf / (xi * xi * kPi * L) * decay;
            break;
        case FSE_STRESSLET:
            *out = std::sqrt(7.0 * Q / 6.0) * R * kinf * kinf * kinf * kinf / (xi * xi * kPi * L) *
                   decay;
            break;
        default: *out = std::sqrt(8.0 * xi * xi * Q / (3.0 * kPi * L * L * L * kinf)) * decay;
    }
    return true;
}

// estimates.cpp:31-47
bool real_est(int kind, double Q, double xi, double rc, double L, double* out) {
    if (!(Q >= 0) || !(xi > 0) || !(rc > 0) || !(L > 0) || bad_kind(kind)) return false;
    const double L3 = L * L * L;
    const double decay = std::exp(-xi * xi * rc * rc);
    switch (kind) {
        case FSE_STOKESLET: *out = std::sqrt(4.0 * Q * rc / L3) * decay; break;
        case FSE_STRESSLET:
            *out = std::sqrt(112.0 * Q * xi * xi * xi * xi * rc * rc * rc / (9.0 * L3)) * decay;
            break;
        default: *out = std::sqrt(8.0 * Q / (3.0 * L3 * rc)) * decay;
    }
    return true;
}

// estimates.cpp:64-79
double velocity_rms(int kind, double Q, double L, uint64_t N) {
    const double a = 0.5 * L / std::cbrt(static_cast<double>(N < 8 ? 8 : N));
    const double L3 = L * L * L;
    switch (kind) {
        case FSE_STOKESLET: return std::sqrt(Q * 4.0 * kPi / (L * L));
        case FSE_STRESSLET: return std::sqrt(Q * 16.0 * kPi * (1.0 / a - 2.0 / L) / L3);
        default: return std::sqrt(Q * (8.0 * kPi / 3.0) * (1.0 / a - 2.0 / L) / L3);
    }
}

}  // namespace

extern "C" {

fse_status fse_fourier_error_estimate(int kind, double Q, double xi, double k_inf, double L,
                                      double R, double* out) {
    if (!out) return FSE_EINVAL;
    return fourier_est(kind, Q, xi, k_inf, L, R, out) ? FSE_OK : FSE_EINVAL;
}

fse_status fse_real_error_estimate(int kind, double Q, double xi, double rc, double L,
                                   double* out) {
    if (!out) return FSE_EINVAL;
    return real_est(kind, Q, xi, rc, L, out) ? FSE_OK : FSE_EINVAL;
}

fse_status fse_error_budget(int kind, const fse_config* cfg, double Q, fse_error_budget_t* out) {
    if (!cfg || !out || bad_kind(kind)) return FSE_EINVAL;
    fse_error_budget_t b;
    std::memset(&b, 0, sizeof b);
    b.kind = kind;
    b.xi = cfg->xi;
    b.rc = cfg->rc;
    b.k_inf = cfg->kinf;
    b.L = cfg->L;
    b.R = cfg->R;
    b.Q = Q;
    if (!real_est(kind, Q, cfg->xi, cfg->rc, cfg->L, &b.predicted_real_rms) ||
        !fourier_est(kind, Q, cfg->xi, cfg->kinf, cfg->L, cfg->R, &b.predicted_fourier_rms))
        return FSE_EINVAL;
    *out = b;
    return FSE_OK;
}

fse_status fse_reference_velocity_rms(int kind, double Q, double L, uint64_t N, double* out) {
    if (!out || bad_kind(kind)) return FSE_EINVAL;
    *out = velocity_rms(kind, Q, L, N);
    return FSE_OK;
}

fse_status fse_select_parameters(int kind, uint64_t N, double L, double Q, double xi, double tol,
                                 fse_config* out, int* feasible) {
    if (!out || !feasible || bad_kind(kind)) return FSE_EINVAL;
    if (!(tol > 0) || !(xi > 0) || !(L > 0) || N < 1) return FSE_EINVAL;
    // P from the accuracy lookup: 16 ~ 8 digits, 24 ~ 12, 32 at round-off
    const int P = tol >= 5e-9 ? 16 : (tol >= 1e-12 ? 24 : 32);
    const double budget = 0.5 * tol * velocity_rms(kind, Q, L, N) / kCalibration;
    const double rc_hi = std::sqrt(3.0) * L, rc_lo = 1.0 / xi;
    double e = 0;
    int ok = 1;
    double rc;
    real_est(kind, Q, xi, rc_hi, L, &e);
    if (e > budget) {
        ok = 0;  // the real-space sum alone cannot meet tol: direct summation
        rc = rc_hi;
    } else if (real_est(kind, Q, xi, rc_lo, L, &e), e <= budget) {
        rc = rc_lo;
    } else {
        double lo = rc_lo, hi = rc_hi;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            real_est(kind, Q, xi, mid, L, &e);
            (e <= budget ? hi : lo) = mid;
        }
        rc = hi;
    }
    fse_config cfg;
    char err[128];
    int M = 2;
    for (;; ++M) {
        if (fse_make_config(L, xi, rc, M, P, 0.0, &cfg, err, sizeof err) == FSE_OK) {
            fourier_est(kind, Q, xi, cfg.kinf, L, cfg.R, &e);
            if (e <= budget) break;
        }
        if (M > 8192) return FSE_EINVAL;  // no feasible grid size
    }
    if (M % 2 != 0 && fse_make_config(L, xi, rc, ++M, P, 0.0, &cfg, err, sizeof err) != FSE_OK)
        return FSE_EINVAL;
    *out = cfg;
    *feasible = ok;
    return FSE_OK;
}

}  // extern "C"
