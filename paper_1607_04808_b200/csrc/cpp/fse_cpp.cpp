// fse_cpp.cpp -- the reference's C++ hot-path API (namespace fse, headers in
// cpp/include/fse) implemented over the C-ABI of libfse_b200.so.  A C++
// program written against the reference library (/root/reference/proj) links
// this instead of libfse.a; the sums, spreading, k-space scaling, cell list,
// Green's precompute, direct sum and the FFT seam run on the GPU.  Scalar
// helpers (single-pair kernels, hhat/bhat, rms_error) are host code.
//
// Errors: fse_status -> the reference's exception types (std::invalid_argument,
// std::domain_error, std::runtime_error).  One process-wide GPU context on
// device $FSE_CUDA_DEVICE (default 0), created on first use; the C-ABI
// serialises calls on it, matching the reference's reentrancy.
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "fse/estimates.hpp"
#include "fse/ewald.hpp"
#include "fse/fft.hpp"
#include "fse/greens.hpp"
#include "fse/kernels.hpp"
#include "fse/realspace.hpp"
#include "fse_cuda.h"
#include "fse_host.h"

static_assert(sizeof(fse::EwaldConfig) == sizeof(fse_config), "EwaldConfig <-> fse_config");
static_assert(offsetof(fse::EwaldConfig, Mtilde) == offsetof(fse_config, Mtilde), "layout");
static_assert(offsetof(fse::EwaldConfig, kinf) == offsetof(fse_config, kinf), "layout");
static_assert(offsetof(fse::EwaldConfig, deterministic) == offsetof(fse_config, deterministic),
              "layout");
static_assert(sizeof(fse::StageTimings) == sizeof(fse_timings), "StageTimings <-> fse_timings");

namespace fse {

namespace detail {

struct DeviceGreen {
    fse_green* h = nullptr;
    ~DeviceGreen() { fse_cuda_green_free(h); }
};

fse_cuda_ctx* ctx() {
    static std::once_flag once;
    static fse_cuda_ctx* c = nullptr;
    static fse_status st = FSE_OK;
    std::call_once(once, [] {
        const char* dev = std::getenv("FSE_CUDA_DEVICE");
        st = fse_cuda_create(dev ? std::atoi(dev) : 0, &c);
    });
    if (st != FSE_OK || !c) throw std::runtime_error("fse: no CUDA device / context creation failed");
    return c;
}

[[noreturn]] void raise(fse_status st, const char* msg) {
    const std::string m = msg ? msg : "fse error";
    if (st == FSE_EINVAL) throw std::invalid_argument(m);
    if (st == FSE_EDOMAIN) throw std::domain_error(m);
    throw std::runtime_error(m);
}

void check(fse_status st) {
    if (st != FSE_OK) raise(st, fse_cuda_last_error(ctx()));
}

std::vector<double> pack_strengths(const SourceSystem& s, KernelKind kind) {
    const int a = strength_arity(kind);
    std::vector<double> out(static_cast<size_t>(a) * s.size());
    for (size_t i = 0; i < s.size() && i < s.strengths.size(); ++i)
        for (int c = 0; c < a; ++c) out[a * i + c] = s.strengths[i].c[c];
    return out;
}

const double* pts(const std::vector<Vec3>& v) { return reinterpret_cast<const double*>(v.data()); }

fse_green* device_green(const MollifiedGreen& g) {
    if (g.device && g.device->h) {
        int k = 0, mt = 0;
        double lt = 0;
        fse_cuda_green_info(g.device->h, &k, &lt, nullptr, nullptr, &mt);
        if (k == static_cast<int>(g.kind) && mt == g.Mtilde && lt == g.Ltilde) return g.device->h;
    }
    const size_t D = static_cast<size_t>(g.doubled());
    if (g.fourier.size() != D * D * D)
        throw std::invalid_argument("MollifiedGreen: fourier table has the wrong size");
    auto dg = std::make_shared<DeviceGreen>();
    check(fse_cuda_green_upload(ctx(), static_cast<int>(g.kind), g.Ltilde, g.Mtilde, g.h, g.R,
                                g.fourier.data(), &dg->h));
    g.device = dg;
    return dg->h;
}

const fse_config* cfg_of(const EwaldConfig& c) { return reinterpret_cast<const fse_config*>(&c); }

// $FSE_CUDA_DEVICES = "0,1,2,3": total_sum runs partitioned over those GPUs
// (fse_cuda_multi_*, one process, NCCL inside the library); unset: one GPU
fse_multi* multi() {
    static std::once_flag once;
    static fse_multi* m = nullptr;
    std::call_once(once, [] {
        const char* env = std::getenv("FSE_CUDA_DEVICES");
        if (!env || !*env) return;
        std::vector<int> devs;
        for (const char* p = env; *p;) {
            char* end = nullptr;
            const long v = std::strtol(p, &end, 10);
            if (end == p) break;
            devs.push_back(static_cast<int>(v));
            p = *end == ',' ? end + 1 : end;
        }
        if (devs.empty() || fse_cuda_multi_create(devs.data(), static_cast<int>(devs.size()), &m) != FSE_OK)
            throw std::runtime_error("fse: FSE_CUDA_DEVICES multi-GPU context creation failed");
    });
    return m;
}

}  // namespace detail

using detail::check;
using detail::ctx;

// ------------------------------------------------------------------ config
EwaldConfig make_config(double L, double xi, double rc, int M, int P, double sf) {
    EwaldConfig c;
    char err[256] = {0};
    const fse_status st =
        fse_make_config(L, xi, rc, M, P, sf, reinterpret_cast<fse_config*>(&c), err, sizeof err);
    if (st != FSE_OK) detail::raise(st, err);
    return c;
}

// ------------------------------------------------------------------ estimates.hpp
double fourier_error_estimate(KernelKind kind, double Q, double xi, double k_inf, double L,
                              double R) {
    double v = 0;
    const fse_status st = fse_fourier_error_estimate(static_cast<int>(kind), Q, xi, k_inf, L, R, &v);
    if (st != FSE_OK) detail::raise(st, "fourier_error_estimate: bad arguments");
    return v;
}

double real_error_estimate(KernelKind kind, double Q, double xi, double rc, double L) {
    double v = 0;
    const fse_status st = fse_real_error_estimate(static_cast<int>(kind), Q, xi, rc, L, &v);
    if (st != FSE_OK) detail::raise(st, "real_error_estimate: bad arguments");
    return v;
}

ErrorBudget error_budget(KernelKind kind, const EwaldConfig& cfg, double Q) {
    fse_error_budget_t b;
    const fse_status st = fse_error_budget(static_cast<int>(kind), detail::cfg_of(cfg), Q, &b);
    if (st != FSE_OK) detail::raise(st, "error_budget: bad arguments");
    ErrorBudget out;
    out.kind = kind;
    out.xi = b.xi;
    out.rc = b.rc;
    out.k_inf = b.k_inf;
    out.L = b.L;
    out.R = b.R;
    out.Q = b.Q;
    out.predicted_real_rms = b.predicted_real_rms;
    out.predicted_fourier_rms = b.predicted_fourier_rms;
    return out;
}

double reference_velocity_rms(KernelKind kind, double Q, double L, std::size_t N) {
    double v = 0;
    const fse_status st = fse_reference_velocity_rms(static_cast<int>(kind), Q, L, N, &v);
    if (st != FSE_OK) detail::raise(st, "reference_velocity_rms: bad arguments");
    return v;
}

SelectedParameters select_parameters(KernelKind kind, std::size_t N, double L, double Q,
                                     double xi, double tol) {
    SelectedParameters sel;
    int feasible = 1;
    const fse_status st = fse_select_parameters(static_cast<int>(kind), N, L, Q, xi, tol,
                                                reinterpret_cast<fse_config*>(&sel.config),
                                                &feasible);
    if (st != FSE_OK) detail::raise(st, "select_parameters: bad arguments");
    sel.feasible = feasible != 0;
    return sel;
}

// ------------------------------------------------------------------ kernels.hpp
void SourceSystem::validate(KernelKind kind) const {  // kernels.cpp:8-25
    if (positions.empty()) throw std::invalid_argument("SourceSystem: N must be >= 1");
    if (positions.size() != strengths.size())
        throw std::invalid_argument("SourceSystem: positions/strengths length mismatch");
    if (!(box_side > 0)) throw std::invalid_argument("SourceSystem: box side must be positive");
    for (size_t n = 0; n < positions.size(); ++n) {
        for (int d = 0; d < 3; ++d)
            if (!(positions[n][d] >= 0 && positions[n][d] <= box_side))
                throw std::invalid_argument("SourceSystem: position outside [0,L]^3");
        if (strengths[n].arity != strength_arity(kind))
            throw std::invalid_argument("SourceSystem: strength arity does not match kernel");
        for (double v : strengths[n].c)
            if (!std::isfinite(v)) throw std::invalid_argument("SourceSystem: non-finite strength");
    }
}

Vec3 eval_kernel(KernelKind kind, const Vec3& r, const Strength& f) {  // kernels.cpp:27-57
    const double r2 = norm2(r);
    if (r2 == 0) throw std::domain_error("eval_kernel: zero separation");
    const double rn = std::sqrt(r2);
    if (kind == KernelKind::Stokeslet) {
        const Vec3 fv{f.c[0], f.c[1], f.c[2]};
        return (1.0 / rn) * fv + (dot(r, fv) / (r2 * rn)) * r;
    }
    if (kind == KernelKind::Stresslet) {
        double rfr = 0;
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) rfr += r[l] * f(l, m) * r[m];
        return (-6.0 * rfr / (r2 * r2 * rn)) * r;
    }
    const Vec3 fv{f.c[0], f.c[1], f.c[2]};
    return Vec3{fv.y * r.z - fv.z * r.y, fv.z * r.x - fv.x * r.z, fv.x * r.y - fv.y * r.x} *
           (1.0 / (r2 * rn));
}

Velocities direct_sum(const SourceSystem& system, KernelKind kind,
                      const std::vector<Vec3>& targets, bool exclude_self) {
    const auto str = detail::pack_strengths(system, kind);
    Velocities u(targets.size());
    check(fse_cuda_direct_sum(ctx(), static_cast<int>(kind), detail::pts(system.positions),
                              str.data(), static_cast<int64_t>(system.size()), detail::pts(targets),
                              static_cast<int64_t>(targets.size()), exclude_self ? 1 : 0,
                              reinterpret_cast<double*>(u.data())));
    return u;
}

Vec3 self_interaction(double xi, const Strength& f, KernelKind kind) {  // kernels.cpp:84-89
    if (!(xi > 0)) throw std::invalid_argument("self_interaction: xi must be positive");
    if (kind != KernelKind::Stokeslet) return {};
    return (-4.0 * xi / std::sqrt(M_PI)) * Vec3{f.c[0], f.c[1], f.c[2]};
}

double rms_error(const Velocities& u, const Velocities& u_ref, bool relative) {
    if (u.size() != u_ref.size()) throw std::invalid_argument("rms_error: length mismatch");
    double num = 0, den = 0;
    for (size_t i = 0; i < u.size(); ++i) {
        num += norm2(u[i] - u_ref[i]);
        den += norm2(u_ref[i]);
    }
    const double n = static_cast<double>(u.size());
    const double abs_rms = std::sqrt(num / n);
    if (!relative) return abs_rms;
    if (den == 0) throw std::domain_error("rms_error: relative error of zero reference");
    return abs_rms / std::sqrt(den / n);
}

double strength_quadratic_sum(const SourceSystem& system) {
    double q = 0;
    for (const Strength& s : system.strengths)
        for (double v : s.c) q += v * v;
    return q;
}

// ------------------------------------------------------------------ greens.hpp
double hhat_R(double k, double R) {  // greens.cpp:22-26
    if (!(R > 0) || k < 0) throw std::invalid_argument("hhat_R: need k >= 0, R > 0");
    const double x = 0.5 * R * k;
    const double s = std::abs(x) < 1e-8 ? 1.0 - x * x / 6.0 : std::sin(x) / x;
    return 2.0 * M_PI * R * R * s * s;
}

double bhat_R(double k, double R) {  // greens.cpp:28-46
    if (!(R > 0) || k < 0) throw std::invalid_argument("bhat_R: need k >= 0, R > 0");
    const double t = R * k;
    const double piR4 = M_PI * R * R * R * R;
    if (t < 0.5) {
        const double t2 = t * t;
        return piR4 * (1.0 + t2 * (-1.0 / 9.0 + t2 * (1.0 / 240.0 + t2 * (-1.0 / 12600.0 +
                       t2 * (1.0 / 1088640.0 + t2 * (-1.0 / 139708800.0 + t2 / 24908083200.0))))));
    }
    const long double tl = static_cast<long double>(R) * k;
    const long double num = (2.0L - tl * tl) * std::cos(tl) + 2.0L * tl * std::sin(tl) - 2.0L;
    return static_cast<double>(4.0L * static_cast<long double>(M_PI) * num / (tl * tl * tl * tl) *
                               (static_cast<long double>(R) * R * R * R));
}

MollifiedGreen precompute_mollified_green(GreenKind kind, double Ltilde, int Mtilde, double sf) {
    auto dg = std::make_shared<detail::DeviceGreen>();
    check(fse_cuda_green_precompute(ctx(), static_cast<int>(kind), Ltilde, Mtilde, sf, &dg->h));
    MollifiedGreen g;
    int k = 0;
    fse_cuda_green_info(dg->h, &k, &g.Ltilde, &g.h, &g.R, &g.Mtilde);
    g.kind = static_cast<GreenKind>(k);
    const size_t D = static_cast<size_t>(g.doubled());
    g.fourier.resize(D * D * D);
    check(fse_cuda_green_download(ctx(), dg->h, g.fourier.data()));
    g.device = dg;
    return g;
}

ScalarGrid freespace_solve(const MollifiedGreen& green, const ScalarGrid& rhs) {  // greens.cpp:115-139
    const int M = green.Mtilde;
    if (rhs.extents[0] != M || rhs.extents[1] != M || rhs.extents[2] != M ||
        rhs.values.size() != rhs.size())
        throw std::invalid_argument("freespace_solve: rhs extents must match green");
    ScalarGrid out;
    out.extents[0] = out.extents[1] = out.extents[2] = M;
    out.h = green.h;
    out.origin = rhs.origin;
    out.values.resize(rhs.size());
    check(fse_cuda_freespace_solve(ctx(), detail::device_green(green), rhs.values.data(),
                                   out.values.data()));
    return out;
}

void save_mollified_green(const MollifiedGreen& green, const std::string& path) {
    check(fse_cuda_green_save(ctx(), detail::device_green(green), path.c_str()));
}

MollifiedGreen load_mollified_green(const std::string& path) {
    auto dg = std::make_shared<detail::DeviceGreen>();
    check(fse_cuda_green_load(ctx(), path.c_str(), &dg->h));
    MollifiedGreen g;
    int k = 0;
    fse_cuda_green_info(dg->h, &k, &g.Ltilde, &g.h, &g.R, &g.Mtilde);
    g.kind = static_cast<GreenKind>(k);
    const size_t D = static_cast<size_t>(g.doubled());
    g.fourier.resize(D * D * D);
    check(fse_cuda_green_download(ctx(), dg->h, g.fourier.data()));
    g.device = dg;
    return g;
}

// ------------------------------------------------------------------ ewald.hpp
GriddedSources spread(const SourceSystem& system, const EwaldConfig& cfg, KernelKind kind,
                      bool use_fgg) {
    const int a = strength_arity(kind);
    const size_t vol = static_cast<size_t>(cfg.Mtilde) * cfg.Mtilde * cfg.Mtilde;
    std::vector<double> flat(vol * a);
    const auto str = detail::pack_strengths(system, kind);
    check(fse_cuda_spread_ex(ctx(), detail::cfg_of(cfg), static_cast<int>(kind),
                             detail::pts(system.positions), str.data(),
                             static_cast<int64_t>(system.size()), system.box_side,
                             use_fgg ? 1 : 0, flat.data()));
    GriddedSources g;
    g.extents[0] = g.extents[1] = g.extents[2] = cfg.Mtilde;
    g.h = cfg.h;
    g.origin = Vec3{-cfg.deltaL / 2, -cfg.deltaL / 2, -cfg.deltaL / 2};
    g.arity = a;
    g.components.resize(a);
    for (int c = 0; c < a; ++c)
        g.components[c].assign(flat.begin() + c * vol, flat.begin() + (c + 1) * vol);
    return g;
}

std::vector<std::vector<std::complex<double>>> kspace_scale(
    const std::vector<std::vector<std::complex<double>>>& ghat, const EwaldConfig& cfg,
    KernelKind kind, const MollifiedGreen& green) {
    const int a = strength_arity(kind);
    if (static_cast<int>(ghat.size()) != a)
        throw std::invalid_argument("kspace_scale: component count does not match kernel");
    const size_t D = static_cast<size_t>(2 * cfg.Mtilde), tot = D * D * D;
    std::vector<std::complex<double>> in(tot * a), out(tot * 3);
    for (int c = 0; c < a; ++c) {
        if (ghat[c].size() != tot)
            throw std::invalid_argument("kspace_scale: plane size does not match grid");
        std::memcpy(in.data() + c * tot, ghat[c].data(), tot * sizeof(std::complex<double>));
    }
    check(fse_cuda_kspace_scale(ctx(), detail::cfg_of(cfg), static_cast<int>(kind),
                                detail::device_green(green),
                                reinterpret_cast<const double*>(in.data()),
                                reinterpret_cast<double*>(out.data())));
    std::vector<std::vector<std::complex<double>>> r(3);
    for (int c = 0; c < 3; ++c) r[c].assign(out.begin() + c * tot, out.begin() + (c + 1) * tot);
    return r;
}

Velocities fourier_sum(const SourceSystem& system, const EwaldConfig& cfg, KernelKind kind,
                       const std::vector<Vec3>& targets, const MollifiedGreen& green,
                       StageTimings* timings) {
    const auto str = detail::pack_strengths(system, kind);
    Velocities u(targets.size());
    check(fse_cuda_fourier_sum(ctx(), detail::cfg_of(cfg), static_cast<int>(kind),
                               detail::pts(system.positions), str.data(),
                               static_cast<int64_t>(system.size()), system.box_side,
                               detail::pts(targets), static_cast<int64_t>(targets.size()),
                               detail::device_green(green), reinterpret_cast<double*>(u.data()),
                               reinterpret_cast<fse_timings*>(timings)));
    return u;
}

Velocities total_sum(const SourceSystem& system, KernelKind kind, const EwaldConfig& cfg,
                     const std::vector<Vec3>& targets, const MollifiedGreen& green,
                     StageTimings* timings) {
    const auto str = detail::pack_strengths(system, kind);
    Velocities u(targets.size());
    if (fse_multi* m = detail::multi()) {
        // the partitioned multi-GPU evaluation (timings: only `total`, the call's wall clock)
        const fse_status st = fse_cuda_multi_total_sum(
            m, detail::cfg_of(cfg), static_cast<int>(kind), detail::pts(system.positions),
            str.data(), static_cast<int64_t>(system.size()), system.box_side,
            detail::pts(targets), static_cast<int64_t>(targets.size()), -1,
            green.fourier.empty() ? nullptr : green.fourier.data(),
            reinterpret_cast<double*>(u.data()), reinterpret_cast<fse_timings*>(timings));
        if (st != FSE_OK) detail::raise(st, fse_cuda_multi_last_error(m));
        return u;
    }
    check(fse_cuda_total_sum(ctx(), detail::cfg_of(cfg), static_cast<int>(kind),
                             detail::pts(system.positions), str.data(),
                             static_cast<int64_t>(system.size()), system.box_side,
                             detail::pts(targets), static_cast<int64_t>(targets.size()), -1,
                             detail::device_green(green), reinterpret_cast<double*>(u.data()),
                             reinterpret_cast<fse_timings*>(timings)));
    return u;
}

// ------------------------------------------------------------------ realspace.hpp
int CellList::cell_of(double coord, int axis) const {  // realspace.cpp:60-63
    const int c = static_cast<int>(std::floor((coord - origin) / cell_side));
    return c < 0 ? 0 : (c > dims[axis] - 1 ? dims[axis] - 1 : c);
}

Vec3 eval_real_kernel(KernelKind kind, const Vec3& r, double xi, const Strength& f) {
    const double r2 = norm2(r);  // realspace.cpp:13-58
    if (r2 == 0) throw std::domain_error("eval_real_kernel: zero separation");
    if (!(xi > 0)) throw std::invalid_argument("eval_real_kernel: xi must be positive");
    const double rn = std::sqrt(r2), xr = xi * rn;
    const double gauss = std::exp(-xr * xr), erfc_xr = std::erfc(xr);
    const double isp = 0.5641895835477562869;
    const Vec3 rh = (1.0 / rn) * r;
    if (kind == KernelKind::Stokeslet) {
        const Vec3 fv{f.c[0], f.c[1], f.c[2]};
        const double a = 2.0 * (xi * gauss * isp + erfc_xr / (2.0 * rn));
        const double b = 4.0 * xi * isp * gauss;
        return (a - b) * fv + (a * dot(rh, fv)) * rh;
    }
    if (kind == KernelKind::Stresslet) {
        const double c1 = -(2.0 / rn) * (3.0 * erfc_xr / rn + 2.0 * xi * isp * (3.0 + 2.0 * xr * xr) * gauss);
        const double c2 = 4.0 * xi * xi * xi * isp * gauss * rn;
        double rfr = 0;
        Vec3 f_r{}, r_f{};
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) {
                rfr += rh[l] * f(l, m) * rh[m];
                f_r[l] += f(l, m) * rh[m];
                r_f[m] += rh[l] * f(l, m);
            }
        const double trf = f(0, 0) + f(1, 1) + f(2, 2);
        return (c1 * rfr + c2 * trf) * rh + c2 * (f_r + r_f);
    }
    const Vec3 fv{f.c[0], f.c[1], f.c[2]};
    const double c = erfc_xr / r2 + 2.0 * xi * isp * gauss / rn;
    return c * Vec3{fv.y * rh.z - fv.z * rh.y, fv.z * rh.x - fv.x * rh.z, fv.x * rh.y - fv.y * rh.x};
}

CellList build_cell_list(const SourceSystem& system, double rc, double domain_pad) {
    CellList cl;
    const int64_t n = static_cast<int64_t>(system.size());
    check(fse_cuda_build_cell_list(ctx(), detail::pts(system.positions), n, system.box_side, rc,
                                   domain_pad, cl.dims, &cl.cell_side, &cl.origin, nullptr, nullptr));
    const size_t ncell = static_cast<size_t>(cl.dims[0]) * cl.dims[1] * cl.dims[2];
    std::vector<int64_t> bstart(ncell + 1), perm(n > 0 ? n : 1);
    check(fse_cuda_build_cell_list(ctx(), detail::pts(system.positions), n, system.box_side, rc,
                                   domain_pad, cl.dims, &cl.cell_side, &cl.origin, bstart.data(),
                                   perm.data()));
    cl.buckets.resize(ncell);
    for (size_t b = 0; b < ncell; ++b)
        cl.buckets[b].assign(perm.begin() + bstart[b], perm.begin() + bstart[b + 1]);
    return cl;
}

Velocities real_space_sum(const SourceSystem& system, KernelKind kind, double xi, double rc,
                          const std::vector<Vec3>& targets) {
    const auto str = detail::pack_strengths(system, kind);
    Velocities u(targets.size());
    check(fse_cuda_real_space_sum(ctx(), static_cast<int>(kind), detail::pts(system.positions),
                                  str.data(), static_cast<int64_t>(system.size()), system.box_side,
                                  xi, rc, detail::pts(targets),
                                  static_cast<int64_t>(targets.size()),
                                  reinterpret_cast<double*>(u.data())));
    return u;
}

// ------------------------------------------------------------------ fft.hpp
void fft3d_forward(std::complex<double>* data, int n0, int n1, int n2) {
    check(fse_cuda_fft3d(ctx(), reinterpret_cast<double*>(data), n0, n1, n2, 0));
}

void fft3d_inverse(std::complex<double>* data, int n0, int n1, int n2) {
    check(fse_cuda_fft3d(ctx(), reinterpret_cast<double*>(data), n0, n1, n2, 1));
}

}  // namespace fse
