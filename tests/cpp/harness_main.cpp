// A program written against the reference's harness API (harness.hpp), linked
// with libfse_b200.so: one timed run with the O(N^2) oracle, an xi sweep, the
// FSEG cache directory, and the fse-report-v1 CSV/JSON files.
//   harness_main <out_dir>
#include <cstdio>
#include <string>

#include "fse/harness.hpp"

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    fse::RunSpec spec;
    spec.kind = fse::KernelKind::Stokeslet;
    spec.N = 3000;
    spec.L = 1.0;
    spec.seed = 2026;
    spec.xi = 10.0;
    spec.rc = 0.3;
    spec.M = 32;
    spec.P = 16;
    spec.cache_dir = dir + "/greens";
    fse::RunReport rep = fse::run(spec);
    fse::RunReport again = fse::run(spec);  // second run hits the FSEG cache
    rep.records.push_back(again.records.front());
    fse::RunSpec tol = spec;
    tol.rc = 0;
    tol.M = 0;
    tol.P = 0;
    tol.tol = 1e-6;
    tol.kind = fse::KernelKind::Rotlet;
    rep.records.push_back(fse::run(tol).records.front());
    fse::RunReport sw = fse::sweep_xi(spec, {10.0, 12.0});
    for (const auto& r : sw.records) rep.records.push_back(r);
    fse::write_csv(rep, dir + "/report.csv");
    fse::write_json(rep, dir + "/report.json");
    for (const auto& r : rep.records)
        std::printf("%s N=%zu M=%d rel_rms=%.3e pre=%.3f total=%.4f e2e=%.4f\n",
                    fse::kernel_name(r.kind), r.N, r.M, r.rel_rms_error, r.times.precompute,
                    r.times.total, r.gpu.t_e2e);
    return 0;
}
