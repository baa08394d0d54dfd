// ref_capi.cpp -- TEST INFRASTRUCTURE (oracle), not product code.
//
// A flat extern "C" surface over the UNMODIFIED reference library, compiled
// from its own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libfse_ref.so.  Python (oracle/refimpl.py) binds it with ctypes
// to generate golden vectors, to pin the C restatement (oracle/fse_oracle.c)
// and to time the reference CPU path for bench.py's cpu_baseline / --impl
// reference legs.  Every entry point is a thin marshalling shim: the work is
// done by the reference's own fse:: functions, cited per function.
//
// Status codes (shared with the product C-ABI, include/fse_cuda.h):
//   0 ok, 1 std::invalid_argument, 2 std::domain_error, 3 std::runtime_error,
//   4 anything else.

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <random>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "fse/estimates.hpp"
#include "fse/ewald.hpp"
#include "fse/fft.hpp"
#include "fse/greens.hpp"
#include "fse/harness.hpp"
#include "fse/kernels.hpp"
#include "fse/realspace.hpp"

using namespace fse;

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_msg = e.what();
        return 2;
    } catch (const std::runtime_error& e) {
        g_msg = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 4;
    }
}

KernelKind kind_of(int k) { return static_cast<KernelKind>(k); }

SourceSystem system_of(int kind, const double* pos, const double* str, int64_t n, double L) {
    const int a = strength_arity(kind_of(kind));
    SourceSystem s;
    s.box_side = L;
    s.positions.resize(n);
    s.strengths.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        s.positions[i] = Vec3{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        s.strengths[i].arity = a;
        for (int c = 0; c < a; ++c) s.strengths[i].c[c] = str[a * i + c];
    }
    return s;
}

std::vector<Vec3> points_of(const double* p, int64_t n) {
    std::vector<Vec3> v(n);
    for (int64_t i = 0; i < n; ++i) v[i] = Vec3{p[3 * i], p[3 * i + 1], p[3 * i + 2]};
    return v;
}

void store(const Velocities& u, double* out) {
    for (size_t i = 0; i < u.size(); ++i) {
        out[3 * i] = u[i].x;
        out[3 * i + 1] = u[i].y;
        out[3 * i + 2] = u[i].z;
    }
}

// cfg fields in EwaldConfig declaration order (ewald.hpp:16-35)
void pack_cfg(const EwaldConfig& c, double* o) {
    const double v[16] = {c.L, c.xi, c.rc, double(c.M), double(c.P), c.h, c.d, c.m,
                          c.eta, c.deltaL, c.Ltilde, double(c.Mtilde), c.kinf, c.R, c.sf,
                          c.deterministic ? 1.0 : 0.0};
    std::memcpy(o, v, sizeof v);
}

MollifiedGreen green_of(int gkind, double Ltilde, int Mtilde, double h, double R,
                        const double* fourier) {
    MollifiedGreen g;
    g.kind = static_cast<GreenKind>(gkind);
    g.Ltilde = Ltilde;
    g.Mtilde = Mtilde;
    g.h = h;
    g.R = R;
    const size_t D = 2 * static_cast<size_t>(Mtilde);
    g.fourier.assign(fourier, fourier + D * D * D);
    return g;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

void ref_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int ref_max_threads() { return omp_get_max_threads(); }

// ewald.cpp:103-134
int ref_make_config(double L, double xi, double rc, int M, int P, double sf, double* out16) {
    return guarded([&] { pack_cfg(make_config(L, xi, rc, M, P, sf), out16); });
}

// realspace.cpp:65-84 (+ the bucket-contiguous layout of :95-109).  With
// bstart == nullptr only dims / cell_side / origin are filled.
int ref_build_cell_list(const double* pos, int64_t n, double L, double rc, double pad,
                        int* dims, double* cell_side, double* origin, int64_t* bstart,
                        int64_t* perm) {
    return guarded([&] {
        SourceSystem s;
        s.box_side = L;
        s.positions = points_of(pos, n);
        s.strengths.resize(n);
        CellList cl = build_cell_list(s, rc, pad);
        for (int d = 0; d < 3; ++d) dims[d] = cl.dims[d];
        *cell_side = cl.cell_side;
        *origin = cl.origin;
        if (!bstart) return;
        int64_t at = 0;
        for (size_t b = 0; b < cl.buckets.size(); ++b) {
            bstart[b] = at;
            for (size_t idx : cl.buckets[b]) perm[at++] = static_cast<int64_t>(idx);
        }
        bstart[cl.buckets.size()] = at;
    });
}

// realspace.cpp:86-149
int ref_real_space_sum(int kind, const double* pos, const double* str, int64_t n, double L,
                       double xi, double rc, const double* tgt, int64_t nt, double* u) {
    return guarded([&] {
        store(real_space_sum(system_of(kind, pos, str, n, L), kind_of(kind), xi, rc,
                             points_of(tgt, nt)),
              u);
    });
}

// realspace.cpp:13-58
int ref_eval_real_kernel(int kind, const double* r, double xi, const double* f, double* out) {
    return guarded([&] {
        Strength s;
        s.arity = strength_arity(kind_of(kind));
        for (int c = 0; c < s.arity; ++c) s.c[c] = f[c];
        Vec3 v = eval_real_kernel(kind_of(kind), Vec3{r[0], r[1], r[2]}, xi, s);
        out[0] = v.x; out[1] = v.y; out[2] = v.z;
    });
}

// kernels.cpp:27-57
int ref_eval_kernel(int kind, const double* r, const double* f, double* out) {
    return guarded([&] {
        Strength s;
        s.arity = strength_arity(kind_of(kind));
        for (int c = 0; c < s.arity; ++c) s.c[c] = f[c];
        Vec3 v = eval_kernel(kind_of(kind), Vec3{r[0], r[1], r[2]}, s);
        out[0] = v.x; out[1] = v.y; out[2] = v.z;
    });
}

// ewald.cpp:136-214
int ref_spread(double L, double xi, double rc, int M, int P, double sf, int deterministic,
               int kind, const double* pos, const double* str, int64_t n, int use_fgg,
               double* grid) {
    return guarded([&] {
        EwaldConfig cfg = make_config(L, xi, rc, M, P, sf);
        cfg.deterministic = deterministic != 0;
        GriddedSources g = spread(system_of(kind, pos, str, n, L), cfg, kind_of(kind),
                                  use_fgg != 0);
        const size_t vol = static_cast<size_t>(cfg.Mtilde) * cfg.Mtilde * cfg.Mtilde;
        for (size_t c = 0; c < g.components.size(); ++c)
            std::memcpy(grid + c * vol, g.components[c].data(), vol * sizeof(double));
    });
}

// ewald.cpp:216-293.  ghat: arity planes of D^3 interleaved complex; out: 3 planes.
int ref_kspace_scale(double L, double xi, double rc, int M, int P, double sf, int kind,
                     const double* green_fourier, const double* ghat, double* out) {
    return guarded([&] {
        EwaldConfig cfg = make_config(L, xi, rc, M, P, sf);
        MollifiedGreen g = green_of(static_cast<int>(green_kind_for(kind_of(kind))),
                                    cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, green_fourier);
        const size_t D = 2 * static_cast<size_t>(cfg.Mtilde), tot = D * D * D;
        const int a = strength_arity(kind_of(kind));
        std::vector<std::vector<std::complex<double>>> gh(a);
        const auto* src = reinterpret_cast<const std::complex<double>*>(ghat);
        for (int c = 0; c < a; ++c) gh[c].assign(src + c * tot, src + (c + 1) * tot);
        auto res = kspace_scale(gh, cfg, kind_of(kind), g);
        auto* dst = reinterpret_cast<std::complex<double>*>(out);
        for (int c = 0; c < 3; ++c) std::memcpy(dst + c * tot, res[c].data(), tot * 16);
    });
}

// ewald.cpp:295-392 / 394-415.  timings7: precompute, spread, fft, scale,
// quadrature, realspace, total (StageTimings order, ewald.hpp:56-64).
int ref_fourier_sum(double L, double xi, double rc, int M, int P, double sf, int kind,
                    const double* pos, const double* str, int64_t n, const double* tgt,
                    int64_t nt, const double* green_fourier, double* u, double* timings7) {
    return guarded([&] {
        EwaldConfig cfg = make_config(L, xi, rc, M, P, sf);
        MollifiedGreen g = green_of(static_cast<int>(green_kind_for(kind_of(kind))),
                                    cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, green_fourier);
        StageTimings t;
        store(fourier_sum(system_of(kind, pos, str, n, L), cfg, kind_of(kind),
                          points_of(tgt, nt), g, &t),
              u);
        if (timings7) {
            const double v[7] = {t.precompute, t.spread, t.fft, t.scale, t.quadrature,
                                 t.realspace, t.total};
            std::memcpy(timings7, v, sizeof v);
        }
    });
}

int ref_total_sum(double L, double xi, double rc, int M, int P, double sf, int kind,
                  const double* pos, const double* str, int64_t n, const double* tgt,
                  int64_t nt, const double* green_fourier, double* u, double* timings7) {
    return guarded([&] {
        EwaldConfig cfg = make_config(L, xi, rc, M, P, sf);
        MollifiedGreen g = green_of(static_cast<int>(green_kind_for(kind_of(kind))),
                                    cfg.Ltilde, cfg.Mtilde, cfg.h, cfg.R, green_fourier);
        StageTimings t;
        store(total_sum(system_of(kind, pos, str, n, L), kind_of(kind), cfg,
                        points_of(tgt, nt), g, &t),
              u);
        if (timings7) {
            const double v[7] = {t.precompute, t.spread, t.fft, t.scale, t.quadrature,
                                 t.realspace, t.total};
            std::memcpy(timings7, v, sizeof v);
        }
    });
}

// greens.cpp:48-113.  out: (2 Mtilde)^3 doubles.
int ref_precompute_green(int gkind, double Ltilde, int Mtilde, double sf, double* out) {
    return guarded([&] {
        MollifiedGreen g =
            precompute_mollified_green(static_cast<GreenKind>(gkind), Ltilde, Mtilde, sf);
        std::memcpy(out, g.fourier.data(), g.fourier.size() * sizeof(double));
    });
}

// greens.cpp:22-46
int ref_hhat(double k, double R, double* out) {
    return guarded([&] { *out = hhat_R(k, R); });
}
int ref_bhat(double k, double R, double* out) {
    return guarded([&] { *out = bhat_R(k, R); });
}

// greens.cpp:155-203 (FSEG cache)
int ref_save_green(int gkind, double Ltilde, int Mtilde, double sf, const char* path) {
    return guarded([&] {
        save_mollified_green(
            precompute_mollified_green(static_cast<GreenKind>(gkind), Ltilde, Mtilde, sf),
            path);
    });
}
int ref_load_green(const char* path, int* gkind, double* Ltilde, double* h, double* R,
                   int* Mtilde, double* out) {
    return guarded([&] {
        MollifiedGreen g = load_mollified_green(path);
        *gkind = static_cast<int>(g.kind);
        *Ltilde = g.Ltilde;
        *h = g.h;
        *R = g.R;
        *Mtilde = g.Mtilde;
        if (out) std::memcpy(out, g.fourier.data(), g.fourier.size() * sizeof(double));
    });
}

// kernels.cpp:59-82
int ref_direct_sum(int kind, const double* pos, const double* str, int64_t n, double L,
                   const double* tgt, int64_t nt, int exclude_self, double* u) {
    return guarded([&] {
        store(direct_sum(system_of(kind, pos, str, n, L), kind_of(kind), points_of(tgt, nt),
                         exclude_self != 0),
              u);
    });
}

// estimates.cpp:49-62, 81-126
int ref_error_budget(int kind, double L, double xi, double rc, int M, int P, double Q,
                     double* real_rms, double* fourier_rms) {
    return guarded([&] {
        ErrorBudget b = error_budget(kind_of(kind), make_config(L, xi, rc, M, P), Q);
        *real_rms = b.predicted_real_rms;
        *fourier_rms = b.predicted_fourier_rms;
    });
}
int ref_select_parameters(int kind, int64_t n, double L, double Q, double xi, double tol,
                          double* out16, int* feasible) {
    return guarded([&] {
        SelectedParameters s = select_parameters(kind_of(kind), n, L, Q, xi, tol);
        pack_cfg(s.config, out16);
        *feasible = s.feasible ? 1 : 0;
    });
}

// harness.cpp:47-66
int ref_generate_system(int kind, int64_t n, double L, uint64_t seed, double* pos,
                        double* str) {
    return guarded([&] {
        SourceSystem s = generate_system(kind_of(kind), n, L, seed);
        const int a = strength_arity(kind_of(kind));
        for (int64_t i = 0; i < n; ++i) {
            for (int d = 0; d < 3; ++d) pos[3 * i + d] = s.positions[i][d];
            for (int c = 0; c < a; ++c) str[a * i + c] = s.strengths[i].c[c];
        }
    });
}

// SURVEY.md 8(d) workload generators (BASELINE.json configs), restated here so
// that bench.py's reference arm and the golden-vector script build their inputs
// without loading the product library.  The stream conventions follow the
// reference harness (harness.cpp:32-34: u = (rng() >> 11) * 2^-53 from
// std::mt19937_64) plus SURVEY 8(d)'s Box-Muller normal (u1 = ((rng() >> 11) + 1)
// * 2^-53, one normal per pair).  Draw order: positions, strengths, targets.
// which: 1 uniform (cfg1/2), 3 sphere (cfg3), 4 clustered (cfg4), 5 uniform +
// distinct targets (cfg5).  tests/test_oracle_generators.py checks the product's
// fse_generate_workload reproduces these streams bit for bit.
namespace {
struct Stream {
    std::mt19937_64 g;
    explicit Stream(uint64_t seed) : g(seed) {}
    double u() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    double z() {
        const double u1 = (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = u();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
};
}  // namespace

int ref_generate_workload(int which, int64_t n, uint64_t seed, double* pos, double* str,
                          double* tgt) {
    return guarded([&] {
        Stream s(seed);
        if (which == 1 || which == 5) {
            for (int64_t i = 0; i < 3 * n; ++i) pos[i] = s.u();
            for (int64_t i = 0; i < 3 * n; ++i) str[i] = s.z();
            if (which == 5)
                for (int64_t i = 0; i < 3 * n; ++i) tgt[i] = s.u();
        } else if (which == 3) {
            std::vector<double> nrm(3 * n);
            for (int64_t i = 0; i < n; ++i) {
                double d0, d1, d2, r2;
                do {
                    d0 = s.z();
                    d1 = s.z();
                    d2 = s.z();
                    r2 = d0 * d0 + d1 * d1 + d2 * d2;
                } while (r2 == 0);
                const double inv = 1.0 / std::sqrt(r2);
                const double d[3] = {d0 * inv, d1 * inv, d2 * inv};
                for (int c = 0; c < 3; ++c) {
                    nrm[3 * i + c] = d[c];
                    pos[3 * i + c] = std::min(1.0, std::max(0.0, 0.5 + 0.5 * d[c]));
                }
            }
            for (int64_t i = 0; i < n; ++i) {
                const double q[3] = {s.z(), s.z(), s.z()};
                // Strength::pair(q, n): f_lm = n_l q_m (kernels.hpp:39-45)
                for (int l = 0; l < 3; ++l)
                    for (int m = 0; m < 3; ++m) str[9 * i + 3 * l + m] = nrm[3 * i + l] * q[m];
            }
        } else if (which == 4) {
            double ctr[32][3];
            for (int b = 0; b < 32; ++b)
                for (int c = 0; c < 3; ++c) ctr[b][c] = 0.2 + 0.6 * s.u();
            const double hi = std::nextafter(1.0, 0.0);
            for (int64_t i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c)
                    pos[3 * i + c] = std::min(hi, std::max(0.0, ctr[i % 32][c] + 0.03 * s.z()));
            for (int64_t i = 0; i < 3 * n; ++i) str[i] = s.z();
        } else {
            throw std::invalid_argument("ref_generate_workload: unknown workload");
        }
    });
}

// fft.cpp:28-37 (through the FFTW shim)
int ref_fft3d(double* data, int n0, int n1, int n2, int inverse) {
    return guarded([&] {
        auto* p = reinterpret_cast<std::complex<double>*>(data);
        if (inverse)
            fft3d_inverse(p, n0, n1, n2);
        else
            fft3d_forward(p, n0, n1, n2);
    });
}

}  // extern "C"
