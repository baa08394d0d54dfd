// fse_host.cpp -- host-side (non-hot-path) pieces of the library:
// deterministic system generators (the reference harness's generate_system,
// harness.cpp:32-34,47-66, and the SURVEY 8(d) workload generators used by
// bench.py), plus small scalar helpers.  Plain C++; exported through the
// C-ABI in include/fse_host.h.
#include "fse_host.h"
#include "fse_cuda.h"
#include "../fse_dist_rules.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>

namespace {

// harness.cpp:32-34: fixed 53-bit mapping
inline double unit_double(std::mt19937_64& rng) {
    return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}

// Box-Muller, u1 in (0,1], one normal per pair of uniforms
inline double normal(std::mt19937_64& rng) {
    const double u1 = (static_cast<double>(rng() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = unit_double(rng);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

}  // namespace

extern "C" {

int fse_generate_system(int kind, int64_t n, double L, uint64_t seed, double* pos, double* str) {
    if (n < 1 || !(L > 0) || !pos || !str) return 1;
    const int a = kind == 1 ? 9 : 3;
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) pos[3 * i + c] = L * unit_double(rng);
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < a; ++c) str[a * i + c] = 2.0 * unit_double(rng) - 1.0;
    return 0;
}

int fse_generate_workload(int which, int64_t n, uint64_t seed, double* pos, double* str,
                          double* tgt) {
    if (n < 0 || (n > 0 && (!pos || !str))) return 1;
    std::mt19937_64 rng(seed);
    const double top = std::nextafter(1.0, 0.0);
    switch (which) {
        case FSE_WL_UNIFORM:
        case FSE_WL_UNIFORM_TARGETS: {
            for (int64_t i = 0; i < 3 * n; ++i) pos[i] = unit_double(rng);
            for (int64_t i = 0; i < 3 * n; ++i) str[i] = normal(rng);
            if (which == FSE_WL_UNIFORM_TARGETS) {
                if (!tgt) return 1;
                for (int64_t i = 0; i < 3 * n; ++i) tgt[i] = unit_double(rng);
            }
            return 0;
        }
        case FSE_WL_SPHERE: {
            // radius 0.5 about (0.5,0.5,0.5); n = outward radial; f_lm = n_l q_m
            double* nrm = new double[3 * n];
            for (int64_t i = 0; i < n; ++i) {
                double d[3], r2 = 0;
                do {
                    r2 = 0;
                    for (int c = 0; c < 3; ++c) {
                        d[c] = normal(rng);
                        r2 += d[c] * d[c];
                    }
                } while (r2 == 0);
                const double inv = 1.0 / std::sqrt(r2);
                for (int c = 0; c < 3; ++c) {
                    nrm[3 * i + c] = d[c] * inv;
                    pos[3 * i + c] = std::clamp(0.5 + 0.5 * d[c] * inv, 0.0, 1.0);
                }
            }
            for (int64_t i = 0; i < n; ++i) {
                double q[3];
                for (int c = 0; c < 3; ++c) q[c] = normal(rng);
                for (int l = 0; l < 3; ++l)
                    for (int m = 0; m < 3; ++m) str[9 * i + 3 * l + m] = nrm[3 * i + l] * q[m];
            }
            delete[] nrm;
            return 0;
        }
        case FSE_WL_CLUSTERED: {
            double centre[32][3];
            for (auto& cc : centre)
                for (double& v : cc) v = 0.2 + 0.6 * unit_double(rng);
            for (int64_t i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c)
                    pos[3 * i + c] = std::clamp(centre[i % 32][c] + 0.03 * normal(rng), 0.0, top);
            for (int64_t i = 0; i < 3 * n; ++i) str[i] = normal(rng);
            return 0;
        }
    }
    return 1;
}

// z-slab ownership and halo masks (fse_dist_rules.h), host side: the same
// arithmetic the device engine (fse_dist.cuh) uses, so a caller can partition
// its input before fse_cuda_dist_total_sum
static bool dist_geom(const fse_config* cfg, int nranks, fsedist::Geom* q) {
    if (!cfg || nranks < 1 || nranks > 16 || cfg->Mtilde < 1 || !(cfg->h > 0)) return false;
    const int Mt = cfg->Mtilde;
    const int nxs = nranks > 1 ? ((Mt + nranks - 1) / nranks + 7) / 8 * 8 : Mt;
    *q = fsedist::Geom{nranks, nxs, Mt, cfg->P, -cfg->deltaL / 2, cfg->h, cfg->rc / cfg->h};
    return true;
}

fse_status fse_dist_owner(const fse_config* cfg, int nranks, const double* pos, int64_t n,
                          int32_t* owner) {
    fsedist::Geom q;
    if (!dist_geom(cfg, nranks, &q) || n < 0 || (n > 0 && (!pos || !owner))) return FSE_EINVAL;
    for (int64_t i = 0; i < n; ++i) owner[i] = fsedist::owner_of(pos[3 * i], q);
    return FSE_OK;
}

fse_status fse_dist_masks(const fse_config* cfg, int nranks, const double* pos, int64_t n,
                          int targets, uint32_t* mask) {
    fsedist::Geom q;
    if (!dist_geom(cfg, nranks, &q) || n < 0 || (n > 0 && (!pos || !mask))) return FSE_EINVAL;
    for (int64_t i = 0; i < n; ++i)
        mask[i] = targets ? fsedist::target_mask(pos[3 * i], q) : fsedist::source_mask(pos[3 * i], q);
    return FSE_OK;
}

}  // extern "C"
