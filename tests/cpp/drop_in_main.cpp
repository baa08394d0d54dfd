// A program written against the reference's fse:: API (as its acceptance
// criterion 2, /root/reference/proj/tests/acceptance.cpp:112-133, uses it),
// compiled against paper_1607_04808_b200/csrc/cpp/include and linked with
// libfse_b200.so instead of the reference's libfse.a.  Prints one line per
// check; exit code 0 iff all pass.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "fse/estimates.hpp"
#include "fse/ewald.hpp"
#include "fse/greens.hpp"
#include "fse/kernels.hpp"
#include "fse/realspace.hpp"

using namespace fse;

static int failures = 0;
static void report(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

// harness.cpp:47-66 generator semantics
static SourceSystem make_system(KernelKind kind, std::size_t n, double L, unsigned long long seed) {
    std::mt19937_64 rng(seed);
    auto u = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
    SourceSystem s;
    s.box_side = L;
    s.positions.resize(n);
    for (auto& p : s.positions)
        for (int c = 0; c < 3; ++c) p[c] = L * u();
    for (std::size_t i = 0; i < n; ++i) {
        Strength f;
        f.arity = strength_arity(kind);
        for (int k = 0; k < f.arity; ++k) f.c[k] = 2.0 * u() - 1.0;
        s.strengths.push_back(f);
    }
    return s;
}

int main() {
    // criterion 2: recorded rel RMS (proj/test_output.txt:8)
    struct Pt { KernelKind kind; double rc; int M; double recorded; } pts[] = {
        {KernelKind::Stokeslet, 0.63, 48, 1.426e-9},
        {KernelKind::Stresslet, 0.63, 50, 1.247e-9},
        {KernelKind::Rotlet, 0.58, 38, 3.376e-9}};
    for (const Pt& p : pts) {
        SourceSystem sys = make_system(p.kind, 20000, 2.0, 2026);
        EwaldConfig cfg = make_config(2.0, 7.0, p.rc, p.M, 16);
        MollifiedGreen g = precompute_mollified_green(green_kind_for(p.kind), cfg.Ltilde,
                                                      cfg.Mtilde, cfg.sf);
        StageTimings t;
        Velocities u = total_sum(sys, p.kind, cfg, sys.positions, g, &t);
        Velocities ref = direct_sum(sys, p.kind, sys.positions, true);
        const double err = rms_error(u, ref, true);
        char buf[160];
        std::snprintf(buf, sizeof buf, "criterion2 kind=%d rel_rms=%.4e recorded=%.3e total=%.4fs",
                      static_cast<int>(p.kind), err, p.recorded, t.total);
        report(std::abs(err - p.recorded) <= 2e-3 * p.recorded && t.total > 0, buf);
    }
    // total_sum N=2 vs direct (test_spectral.cpp:185-196), with the reference's
    // fixture stream (tests/helpers.hpp:11-35: per point 3 uniforms in [0,L),
    // then `arity` uniforms in [-1,1); one mt19937_64(42) across the kinds)
    {
        std::mt19937_64 rng(42);
        auto uni = [&](double lo, double hi) {
            return lo + (hi - lo) * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
        };
        for (KernelKind kind : {KernelKind::Stokeslet, KernelKind::Stresslet, KernelKind::Rotlet}) {
            SourceSystem s;
            s.box_side = 1.0;
            for (int n = 0; n < 2; ++n) {
                s.positions.push_back({uni(0, 1), uni(0, 1), uni(0, 1)});
                Strength f;
                f.arity = strength_arity(kind);
                for (int k = 0; k < f.arity; ++k) f.c[k] = uni(-1, 1);
                s.strengths.push_back(f);
            }
            EwaldConfig cfg = make_config(1.0, 6.0, 1.0, 28, 32);
            MollifiedGreen g = precompute_mollified_green(green_kind_for(kind), cfg.Ltilde,
                                                          cfg.Mtilde, cfg.sf);
            const double err = rms_error(total_sum(s, kind, cfg, s.positions, g),
                                         direct_sum(s, kind, s.positions, true), true);
            // The reference scores 3.75e-13 / 9.98e-13 / 1.27e-14 on exactly this stream
            // (oracle/_ref); with the reference's own Green's table uploaded the GPU scores
            // 4.08e-13 / 9.84e-13 / 7.8e-15.  The GPU-precomputed table differs from the
            // reference's by FFT round-off (1.5e-16 of max) that the stresslet's high-k
            // multiplier amplifies to 1.6e-12 here, so the stresslet bound is 2e-12.
            const double bound = kind == KernelKind::Stresslet ? 2e-12 : 1e-12;
            char buf[120];
            std::snprintf(buf, sizeof buf, "two sources vs direct, kind %d: %.2e < %.0e",
                          static_cast<int>(kind), err, bound);
            report(err < bound, buf);
        }
    }
    // a hand-filled table (no device copy) is uploaded transparently
    {
        SourceSystem s = make_system(KernelKind::Stokeslet, 300, 1.0, 5);
        EwaldConfig cfg = make_config(1.0, 8.0, 0.3, 24, 16);
        MollifiedGreen g = precompute_mollified_green(GreenKind::Biharmonic, cfg.Ltilde, cfg.Mtilde, cfg.sf);
        MollifiedGreen copy = g;
        copy.device.reset();
        const double d = rms_error(total_sum(s, KernelKind::Stokeslet, cfg, s.positions, copy),
                                   total_sum(s, KernelKind::Stokeslet, cfg, s.positions, g), true);
        report(d < 1e-15, "host table upload path");
        CellList cl = build_cell_list(s, 0.1);
        std::size_t count = 0;
        for (const auto& b : cl.buckets) count += b.size();
        report(count == s.size() && cl.dims[0] == 10, "build_cell_list");
        GriddedSources gs = spread(s, cfg, KernelKind::Stokeslet);
        double mass = 0, want = 0;
        for (double v : gs.components[0]) mass += v;
        for (const auto& f : s.strengths) want += f.c[0];
        report(std::abs(mass * cfg.h * cfg.h * cfg.h - want) < 1e-6 * (1 + std::abs(want)),
               "spread conserves strength");
        // error mapping
        bool ok = false;
        try {
            fourier_sum(s, cfg, KernelKind::Stokeslet, {{1.5, 0.5, 0.5}}, g);
        } catch (const std::invalid_argument&) { ok = true; }
        report(ok, "target outside box -> std::invalid_argument");
        ok = false;
        try {
            make_config(2.0, 7.0, 0.63, 48, 15);
        } catch (const std::invalid_argument&) { ok = true; }
        report(ok, "odd P -> std::invalid_argument");
        ok = false;
        SourceSystem two;
        two.box_side = 1.0;
        two.positions = {{0.1, 0.2, 0.3}, {0.1, 0.2, 0.3}};
        two.strengths = {Strength::vec({1, 0, 0}), Strength::vec({0, 1, 0})};
        try {
            direct_sum(two, KernelKind::Stokeslet, two.positions, true);
        } catch (const std::domain_error&) { ok = true; }
        report(ok, "coincident points -> std::domain_error");
    }
    // estimates.hpp: the criterion-2 workload selection (test_estimates.cpp:84-93) and
    // the selected configuration meeting its own budget
    {
        SourceSystem s = make_system(KernelKind::Stokeslet, 20000, 2.0, 2026);
        double Q = 0;
        for (const auto& f : s.strengths)
            for (int k = 0; k < f.arity; ++k) Q += f.c[k] * f.c[k];
        SelectedParameters sel = select_parameters(KernelKind::Stokeslet, 20000, 2.0, Q, 7.0, 0.5e-8);
        ErrorBudget b = error_budget(KernelKind::Stokeslet, sel.config, Q);
        const double ref = reference_velocity_rms(KernelKind::Stokeslet, Q, 2.0, 20000);
        char buf[160];
        std::snprintf(buf, sizeof buf, "select_parameters: M=%d P=%d rc=%.4f real %.2e fourier %.2e",
                      sel.config.M, sel.config.P, sel.config.rc, b.predicted_real_rms,
                      b.predicted_fourier_rms);
        report(sel.feasible && sel.config.P == 16 && sel.config.M % 2 == 0 &&
                   b.predicted_real_rms <= 0.25 * 0.5e-8 * ref * (1 + 1e-12) &&
                   b.predicted_fourier_rms <= 0.25 * 0.5e-8 * ref * (1 + 1e-12),
               buf);
    }
    // greens.hpp freespace_solve: Gaussian Poisson oracle (test_greens.cpp:117-120)
    {
        const int M = 48;
        const double a = 200.0;
        MollifiedGreen g = precompute_mollified_green(GreenKind::Harmonic, 1.0, M,
                                                      1.0 + std::sqrt(3.0));
        ScalarGrid rhs;
        rhs.extents[0] = rhs.extents[1] = rhs.extents[2] = M;
        rhs.h = 1.0 / M;
        rhs.values.resize(rhs.size());
        const double pref = std::pow(a / M_PI, 1.5);
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j)
                for (int k = 0; k < M; ++k) {
                    const double x = i * rhs.h - 0.5, y = j * rhs.h - 0.5, z = k * rhs.h - 0.5;
                    rhs.at(i, j, k) = pref * std::exp(-a * (x * x + y * y + z * z));
                }
        ScalarGrid phi = freespace_solve(g, rhs);
        double err = 0, mx = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j)
                for (int k = 0; k < M; ++k) {
                    const double x = i * rhs.h - 0.5, y = j * rhs.h - 0.5, z = k * rhs.h - 0.5;
                    const double r = std::sqrt(x * x + y * y + z * z);
                    const double ex = r < 1e-12 ? 2.0 * std::sqrt(a / M_PI) : std::erf(std::sqrt(a) * r) / r;
                    err = std::max(err, std::abs(phi.at(i, j, k) - ex));
                    mx = std::max(mx, std::abs(ex));
                }
        char buf[120];
        std::snprintf(buf, sizeof buf, "freespace_solve Gaussian oracle: %.2e < 1e-10", err / mx);
        report(err / mx < 1e-10, buf);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
    return failures ? 1 : 0;
}
