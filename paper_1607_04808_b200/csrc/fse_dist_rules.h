// fse_dist_rules.h -- particle ownership and halo rules of the z-slab (x-plane)
// decomposition, shared by the device engine (fse_dist.cuh),
// the host-side input partition (fse_host.cpp, fse_dist_classify) and the
// tests.  Plain arithmetic, identical on host and device.
//
// Slab r of G owns the Mtilde-grid x-planes [x_lo(r), x_lo(r) + nx(r)),
// x_lo = min(r nxs, Mt), nx = min(nxs, Mt - x_lo) (fsecu::set_slab).  A point
// at x has s = (x - origin) / h and support start f = ceil(s - P/2)
// (ewald.cpp:38-39, the product's support_start); its "plane" is c = f + P/2
// (= ceil(s)) and its owner is min(max(c, 0) / nxs, G - 1).
//
// A source is needed by rank d when
//   (spread)     its support [f, f + P) meets d's planes, or
//   (real space) it lies within rc of the x-range of d's owned targets,
//                s in (d nxs - 1, (d + 1) nxs - 1] (unbounded at the ends),
//                widened by one plane for rounding;
// a target by rank d when its support meets d's planes (d adds that part of
// its quadrature and returns it to the owner).  Both sets are intervals of
// ranks that contain the owner.
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define FSE_HD __host__ __device__ __forceinline__
#else
#define FSE_HD inline
#endif

namespace fsedist {

struct Geom {
    int G;         // ranks
    int nxs;       // x-planes per slab (whole spread tiles)
    int Mt;        // Mtilde
    int P;         // support
    double origin; // -deltaL / 2
    double h;      // grid spacing
    double rh;     // rc / h (real-space reach in planes)
};

FSE_HD double plane_coord(double x, const Geom& q) { return (x - q.origin) / q.h; }
FSE_HD int support_first(double s, const Geom& q) {
    return static_cast<int>(ceil(s - 0.5 * q.P));
}
FSE_HD int owner_of(double x, const Geom& q) {
    int c = support_first(plane_coord(x, q), q) + q.P / 2;
    if (c < 0) c = 0;
    const int o = c / q.nxs;
    return o < q.G - 1 ? o : q.G - 1;
}
FSE_HD int slab_lo(int d, const Geom& q) { return d * q.nxs < q.Mt ? d * q.nxs : q.Mt; }
FSE_HD int slab_n(int d, const Geom& q) {
    const int lo = slab_lo(d, q);
    return q.nxs < q.Mt - lo ? q.nxs : q.Mt - lo;
}
// ranks (bit d) whose planes meet the support [f, f + P)
FSE_HD uint32_t support_mask(int f, const Geom& q) {
    uint32_t m = 0;
    for (int d = 0; d < q.G; ++d) {
        const int lo = slab_lo(d, q), n = slab_n(d, q);
        if (n > 0 && f < lo + n && f + q.P > lo) m |= 1u << d;
    }
    return m;
}
// ranks (bit d) that need source x: support overlap or real-space reach
FSE_HD uint32_t source_mask(double x, const Geom& q) {
    const double s = plane_coord(x, q);
    uint32_t m = support_mask(support_first(s, q), q);
    for (int d = 0; d < q.G; ++d) {
        const bool lo_ok = d == 0 || s > d * static_cast<double>(q.nxs) - 2.0 - q.rh;
        const bool hi_ok = d == q.G - 1 || s <= (d + 1) * static_cast<double>(q.nxs) + q.rh;
        if (lo_ok && hi_ok) m |= 1u << d;
    }
    return m;
}
// ranks (bit d) that add part of target x's quadrature
FSE_HD uint32_t target_mask(double x, const Geom& q) {
    return support_mask(support_first(plane_coord(x, q), q), q);
}

}  // namespace fsedist
