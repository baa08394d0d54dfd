// k_realspace.cu -- screened real-space pair sum (realspace.cpp:86-149) with
// the screened kernels of realspace.cpp:13-58.
//
// Sources and targets are sorted by (cell, sub-cell): 64 sub-cells per cell in
// Morton order (octant bits, then quarter bits; 8 or none when the cell grid is
// large next to the point count) -- the kernels' own order; the reference's
// CellList order is kept for build_cell_list only.  The 32 targets of an item are
// then neighbours, so on clustered input their lanes accept similar numbers of
// pairs (cfg4 real space 91.4 -> 80.2 ms from the ordering alone).
// Work item = (target cell, up to 32 of its targets) = one warp, one lane
// per target; a CTA runs 8 independent items (no CTA barrier in the loop).
// Dense cells (>= 640 targets) are cut into octant items, whose neighbourhood is
// 125 of the 216 (cell, octant) sub-buckets.
// The 27 neighbour buckets (lexicographic (di,dj,dk)) are concatenated
// virtually and sampled with a coprime stride (so every chunk mixes all
// buckets and the lanes accept similar numbers of pairs), then streamed
// through the warp's shared memory in chunks of 64 sources.  Each lane first
// tests its target against the whole chunk (closed ball 0 < d2 <= rc2, d2 =
// (x*x + y*y) + z*z rounded like the reference, realspace.cpp:140) into a
// 64-bit mask, then evaluates only the accepted pairs.  The accepted set is
// the reference's; the summation order differs (fixed, deterministic).
//
// Pair math: with x = xi r and inv = 1/r, every screened kernel is a power
// of inv times smooth functions of x alone (s = 2/sqrt(pi)):
//   stokeslet: a - b = inv Ahat(x), a = inv Chat(x),
//              Ahat = erfc x - s x e^{-x^2},  Chat = erfc x + s x e^{-x^2}
//   rotlet:    c = inv^2 Chat(x)
//   stresslet: c1 = -2 inv^2 Dhat(x), c2 = xi^2 Ehat(x),
//              Dhat = 3 erfc x + s x (3 + 2x^2) e^{-x^2},  Ehat = 2 s x e^{-x^2}
// With erfc x = e^{-x^2} erfcx(x) they all are e^{-x^2} times polynomials in
// x and erfcx(x).  erfcx is tabulated on [0, 6.5) as 128 piecewise degree-7
// Chebyshev fits (monomials in the local t, built in long double from
// erfcl/expl; max abs error 1.6e-16) and e^{-x^2} is computed (bounded-range
// exp, constants in constant memory): one 8-byte table load per coefficient per
// pair.  (Tabulating the two functions directly removes the exp but doubles
// the shared-memory bytes per pair, and the table loads -- random intervals per
// lane, bank conflicts -- then bound the loop: 6.2 vs 5.2 ms at cfg2.)
// 1/r: fp32 seed + two fp64 Newton steps.  x >= 6.5 (only for xi rc > 6.5)
// uses the erfc/exp formulas directly.
//
// Candidate test: the closed-ball test is decided in fp32 on coordinates
// relative to the item's cell centre (FP32 pipe, off the FP64 pipe that
// the pair math saturates).  With |relative coordinate| <= Rm the fp32
// squared distance is within B of the exact one (bound derived in
// fp32_bounds()), so d2f <= rc2 - B is certainly inside, d2f > rc2 + B
// certainly outside, and only the rare band in between, near-coincident
// pairs and points farther than Rm from the centre (NaN sentinels: points
// outside the box clamped into edge cells) take the exact fp64 test of
// realspace.cpp:140.  The accepted set is therefore exactly the reference's.
//
// Roofline: FP64 (pair work).
#include <cmath>
#include <cstdlib>

#include "fse_internal.cuh"

namespace fsecu {

namespace {

// 64-source chunks: a smaller per-warp chunk buffer buys occupancy (the
// pair loop is latency-bound), which beats the better lane balance of
// 128-source chunks (cfg2 5.84 -> 5.22 ms, cfg4 105 -> 98 ms on B200).
// Three 256-thread CTAs per SM (78 registers): with the branch-free candidate
// test the pair loop no longer rematerialises constants at the 64-register
// cap (cfg2 5.55 -> 5.27 ms, cfg4 98.5 -> 91.6 ms; 2 CTAs at 107 registers,
// 128-thread CTAs at 93 or 78 registers and 128-source chunks all measured slower)
#ifndef FSE_RS_TPB
#define FSE_RS_TPB 256
#endif
#ifndef FSE_RS_CH
#define FSE_RS_CH 64
#endif
#ifndef FSE_RS_MINB
#define FSE_RS_MINB 3
#endif
constexpr int TPB = FSE_RS_TPB, CH = FSE_RS_CH, NW = CH / 32;
static_assert(CH % 32 == 0 && NW >= 1 && NW <= 4, "chunk of 1..4 mask words");
constexpr double kInvSqrtPi = 0.5641895835477562869;

constexpr int kNI = 128, kDeg = 7;
constexpr double kXMax = 6.5;
// erfcx(x) = e^{x^2} erfc(x), piecewise degree-7 on kNI intervals of [0, kXMax):
// [j][iv] = monomial coefficient j in the local t (coefficient-major: the lanes
// of a warp read different intervals iv of one coefficient, 8-byte words)
__constant__ double c_erfcx[kDeg + 1][kNI];
// e^{-x^2}: Cody-Waite constants and the degree-13 Taylor coefficients, in
// constant memory so the FMAs take them as c[] operands (immediates would be
// rematerialised into uniform registers inside the pair loop)
__constant__ double c_exp[18] = {
    1.4426950408889634074, 6.93147180559945286227e-01, 2.31904681384629955842e-17,
    6755399441055744.0,
    1.0, 1.0 / 6.0, 0.5, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 5040.0, 1.0 / 720.0,
    1.0 / 362880.0, 1.0 / 40320.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.1283791670955126};


struct FastTest {
    double rm;        // max |relative coordinate| of the fast path
    float lo, hi, z0; // certainly inside: z0 < d2f <= lo; certainly outside: d2f > hi
};

// Error bound of the fp32 squared distance.  Relative coordinates are
// computed in fp64 (error <= 2^-53 Rm) and rounded to fp32 (<= 2^-24 Rm);
// the fp32 difference adds <= 2^-24 |dx| <= 2^-23 Rm, so per component
// |dxf - dx| <= delta = 2^-21 Rm (generous).  Then
//   |d2f - d2| <= 2 sqrt(3) d delta + 3 delta^2 + 2^-22 d2f,
// evaluated at d <= 1.01 rc and doubled for the band; near zero
// d2f <= 3 delta^2 (1 + 2^-22) when d2 = 0, doubled for z0.
FastTest fp32_bounds(double rc, double side) {
    FastTest f;
    f.rm = 1.6 * side;
    const double delta = std::ldexp(f.rm, -21);
    const double d = 1.01 * rc;
    const double B = 2.0 * (2.0 * std::sqrt(3.0) * d * delta + 3.0 * delta * delta +
                            std::ldexp(d * d, -22));
    const double rc2 = rc * rc;
    f.lo = std::nextafter(static_cast<float>(rc2 - B), 0.0f);
    f.hi = std::nextafter(static_cast<float>(rc2 + B), 1e30f);
    f.z0 = std::nextafter(static_cast<float>(6.0 * delta * delta), 1e30f);
    if (!(rc2 - B > 0.0)) f.lo = -1.0f;  // degenerate: everything takes the exact test
    return f;
}

// exact functions (fallback beyond the table)
__device__ __forceinline__ void fn_exact(int which, double x, double* out) {
    const double e = exp(-x * x), ec = erfc(x), s = 2.0 * kInvSqrtPi;
    switch (which) {
        case 0: *out = ec - s * x * e; break;
        case 1: *out = ec + s * x * e; break;
        case 2: *out = 3.0 * ec + s * x * (3.0 + 2.0 * x * x) * e; break;
        default: *out = 2.0 * s * x * e; break;
    }
}

__device__ __forceinline__ double exact_d2(double rx, double ry, double rz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz));
}

// e^y for y in [-kXMax^2, 0]: y = j ln2 + r (|r| <= ln2 / 2, Cody-Waite with
// FMA), degree-13 Taylor polynomial in Estrin form (remainder < 5e-18
// relative), 2^j added to the exponent field (j >= -61: no overflow,
// underflow or subnormal cases).  Max error ~2 ulp (host-checked against expl).
__device__ __forceinline__ double exp_neg_bounded(double y) {
    const double k = fma(y, c_exp[0], c_exp[3]);  // round(y log2 e) in the low word
    const double jd = k - c_exp[3];
    const int j = __double2loint(k);
    double r = fma(jd, -c_exp[1], y);
    r = fma(jd, -c_exp[2], r);
    const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    const double a0 = r + c_exp[4], a1 = fma(r, c_exp[5], c_exp[6]);
    const double a2 = fma(r, c_exp[7], c_exp[8]), a3 = fma(r, c_exp[9], c_exp[10]);
    const double a4 = fma(r, c_exp[11], c_exp[12]);
    const double a5 = fma(r, c_exp[13], c_exp[14]);
    const double a6 = fma(r, c_exp[15], c_exp[16]);
    const double b0 = fma(a1, r2, a0), b1 = fma(a3, r2, a2), b2 = fma(a5, r2, a4);
    const double d0 = fma(b1, r4, b0), d1 = fma(a6, r4, b2);
    const double p = fma(d1, r8, d0);
    return __hiloint2double(__double2hiint(p) + j * (1 << 20), __double2loint(p));
}

// 1/sqrt(r2): the FP64 MUFU seed (rsqrt.approx.f64, ~2^-22 relative, the
// whole double range: no conversions and no special-case branch) and two
// Newton steps in fp64 (22 -> 44 -> full bits, ~1 ulp)
__device__ __forceinline__ double rsqrt_nr(double r2) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double h = 0.5 * r2;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    return y;
}

// tab: erfcx coefficients [j][iv] (shared memory); F0, F1 = the two functions
// this kernel needs (stokeslet: Ahat, Chat; rotlet: Chat, -; stresslet: Dhat,
// Ehat) as e^{-x^2} times polynomials in x and erfcx(x): one 8-byte table load
// per coefficient per pair, e^{-x^2} computed.  TAIL: x = xi r can reach the
// end of the table (xi rc >= 6.5), so the exact formulas take over there.
template <int KIND, bool TAIL>
__device__ __forceinline__ void pair(double rx, double ry, double rz, double r2, double xi,
                                     const double* f, const double (*tab)[kNI], double acc[3]) {
    const double inv = rsqrt_nr(r2);
    const double rn = r2 * inv;
    const double xr = xi * rn;
    double F0, F1 = 0.0;
    if (!TAIL || xr < kXMax) {
        // interval iv = floor(uu) by the round-to-nearest magic constant (no
        // F2I/I2F conversions): round(uu - 1/2); at an integer uu this may give
        // uu - 1 and t = 1, the fitted interval's closed end
        // (uu < kNI: xr < kXMax, clamped against the product's rounding)
        const double uu = fmin(xr * (kNI / kXMax), kNI - 1e-9);
        const double kk = (uu - 0.5) + c_exp[3];
        const int iv = __double2loint(kk);
        const double t = 2.0 * (uu - (kk - c_exp[3])) - 1.0;
#ifdef FSE_RS_HORNER
        double ex = tab[kDeg][iv];
#pragma unroll
        for (int j = kDeg - 1; j >= 0; --j) ex = fma(ex, t, tab[j][iv]);
#else
        // Estrin (degree 7): dependency depth 4 instead of Horner's 7
        static_assert(kDeg == 7, "Estrin scheme written for degree 7");
        const double t2 = t * t, t4 = t2 * t2;
        const double a0 = fma(tab[1][iv], t, tab[0][iv]), a1 = fma(tab[3][iv], t, tab[2][iv]);
        const double a2 = fma(tab[5][iv], t, tab[4][iv]), a3 = fma(tab[7][iv], t, tab[6][iv]);
        const double ex = fma(fma(a3, t2, a2), t4, fma(a1, t2, a0));
#endif
        const double E = exp_neg_bounded(-xr * xr);
        const double sx = c_exp[17] * xr;  // 2 x / sqrt(pi)
        if (KIND == FSE_STOKESLET) {
            F0 = E * (ex - sx);
            F1 = E * (ex + sx);
        } else if (KIND == FSE_ROTLET) {
            F0 = E * (ex + sx);
        } else {
            F0 = E * (3.0 * ex + sx * (3.0 + 2.0 * xr * xr));
            F1 = 2.0 * sx * E;
        }
    } else {
        fn_exact(KIND == FSE_STOKESLET ? 0 : (KIND == FSE_ROTLET ? 1 : 2), xr, &F0);
        if (KIND != FSE_ROTLET) fn_exact(KIND == FSE_STOKESLET ? 1 : 3, xr, &F1);
    }
    if (KIND == FSE_STOKESLET) {
        // (a - b) f + a (rhat . f) rhat = inv F0 f + inv^3 F1 (r . f) r
        const double amb = inv * F0;
        const double s = inv * inv * inv * F1 * (rx * f[0] + ry * f[1] + rz * f[2]);
        acc[0] += amb * f[0] + s * rx;
        acc[1] += amb * f[1] + s * ry;
        acc[2] += amb * f[2] + s * rz;
    } else if (KIND == FSE_STRESSLET) {
        const double rh[3] = {inv * rx, inv * ry, inv * rz};
        const double c1 = -2.0 * inv * inv * F0;
        const double c2 = xi * xi * F1;
        double rfr = 0, f_r[3] = {0, 0, 0}, r_f[3] = {0, 0, 0};
#pragma unroll
        for (int l = 0; l < 3; ++l)
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                rfr += rh[l] * f[3 * l + m] * rh[m];
                f_r[l] += f[3 * l + m] * rh[m];
                r_f[m] += rh[l] * f[3 * l + m];
            }
        const double trf = f[0] + f[4] + f[8];
        const double s = c1 * rfr + c2 * trf;
#pragma unroll
        for (int j = 0; j < 3; ++j) acc[j] += s * rh[j] + c2 * (f_r[j] + r_f[j]);
    } else {
        // inv^2 Chat (f x rhat) = inv^3 Chat (f x r)
        const double c = inv * inv * inv * F0;
        acc[0] += c * (f[1] * rz - f[2] * ry);
        acc[1] += c * (f[2] * rx - f[0] * rz);
        acc[2] += c * (f[0] * ry - f[1] * rx);
    }
}

__device__ __forceinline__ int gcd_int(int a, int b) {
    while (b) {
        const int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// fp32 relative coordinate, NaN beyond Rm (forces the exact test)
__device__ __forceinline__ float rel32(double v, double rm) {
    return fabs(v) <= rm ? static_cast<float>(v) : __int_as_float(0x7fffffff);
}

// Neighbour list entries per item: the 27 buckets of a cell item, or the <= 125
// (cell, octant) sub-buckets an octant item can reach (see k_realspace below)
constexpr int kNB = 128;

template <int A>
struct WarpChunk {
    float sxf[CH], syf[CH], szf[CH];  // SoA: two candidates per packed fp32 op
    double sx[CH], sy[CH], sz[CH];
    double sf[CH][A];
    int nb_start[kNB], nb_pref[kNB + 1];
};

template <int KIND, bool TAIL>
__global__ void __launch_bounds__(TPB, FSE_RS_MINB) k_realspace(
    int dim, int nsub, const double* __restrict__ spx, const double* __restrict__ spy,
    const double* __restrict__ spz, const double* __restrict__ sfs,
    const int32_t* __restrict__ bstart, const double* __restrict__ tpx,
    const double* __restrict__ tpy, const double* __restrict__ tpz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ items,
    const uint32_t* __restrict__ tperm, const int32_t* __restrict__ nitems_dev, double xi,
    double rc2, double origin, double side, FastTest ft, unsigned long long* __restrict__ counts,
    double* __restrict__ u) {
    constexpr int A = KIND == FSE_STRESSLET ? 9 : 3;
    constexpr int W = TPB / 32;
    // per-warp source chunk (each warp is an independent work item), in
    // dynamic shared memory: WarpChunk<A>[W]
    extern __shared__ __align__(16) unsigned char rs_smem[];
    WarpChunk<A>& wc = reinterpret_cast<WarpChunk<A>*>(rs_smem)[threadIdx.x >> 5];
    auto& sx = wc.sx;
    auto& sy = wc.sy;
    auto& sz = wc.sz;
    auto& sxf = wc.sxf;  // fp32 coordinates relative to the cell centre
    auto& syf = wc.syf;
    auto& szf = wc.szf;
    auto& sf = wc.sf;
    auto& nb_start = wc.nb_start;
    auto& nb_pref = wc.nb_pref;
    __shared__ double tab[kDeg + 1][kNI];
    // the grid is an upper bound on the item count: surplus CTAs leave at once
    if (static_cast<int>(blockIdx.x) * W >= *nitems_dev) return;
    {
        const double* src = &c_erfcx[0][0];
        double* dst = &tab[0][0];
        for (int e = threadIdx.x; e < (kDeg + 1) * kNI; e += blockDim.x) dst[e] = src[e];
    }
    __syncthreads();  // the only CTA-wide barrier

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int item = blockIdx.x * W + warp;
    if (item >= *nitems_dev) return;  // grid is an upper bound
    const int cell = items[2 * item];
    const int sub = items[2 * item + 1] & 0xffffff;
    const int oct = (items[2 * item + 1] >> 24) - 1;  // -1: the whole cell; else its octant
    const int ost = nsub >> 3;  // sub-buckets per octant (sub = 8 or 64 buckets per cell)
    const int ck = cell % dim, cj = (cell / dim) % dim, ci = cell / (dim * dim);
    // Neighbour list, prefix-summed.  bstart / tstart hold (cell, octant) bucket
    // starts: cell b is [bstart[nsub b], bstart[nsub b + nsub]).  A cell item takes the 27
    // neighbour cells.  An octant item (targets of octant (a_x, a_y, a_z) of a dense
    // cell) takes per axis both halves of its own cell, and of a neighbour cell only
    // the near half when the neighbour lies on the far side of the target's half:
    // a target with x < cx_i and a source with x >= cx_{i+1} are more than one cell
    // side > rc apart (bits are comparisons against the same centres, k_cell_ids), so
    // no accepted pair is dropped: 125 of the 216 sub-buckets remain.
    {
        int n_nb = 0;  // entries so far (warp-uniform)
        const int ne = oct < 0 ? 27 : 216;
        for (int e0 = 0; e0 < ne; e0 += 32) {
            const int e = e0 + lane;
            int st = 0, len = 0;
            bool use = false;
            if (e < ne) {
                const int nc = oct < 0 ? e : e >> 3, so = e & 7;
                const int di = nc / 9 - 1, dj = (nc / 3) % 3 - 1, dk = nc % 3 - 1;
                const int i = ci + di, j = cj + dj, k = ck + dk;
                if (i >= 0 && i < dim && j >= 0 && j < dim && k >= 0 && k < dim) {
                    const int b = (i * dim + j) * dim + k;
                    if (oct < 0) {
                        st = bstart[nsub * b];
                        len = bstart[nsub * b + nsub] - st;
                        use = len > 0;
                    } else {
                        // keep (d, source bit s) unless the neighbour is on the far side:
                        // d = -1 needs s = 1 when the target bit is 1; d = +1 needs s = 0
                        // when the target bit is 0
                        const int ax = (oct >> 2) & 1, ay = (oct >> 1) & 1, az = oct & 1;
                        const int sx = (so >> 2) & 1, sy = (so >> 1) & 1, sz = so & 1;
                        const bool kx = di == 0 || (di < 0 ? (ax == 0 || sx == 1) : (ax == 1 || sx == 0));
                        const bool ky = dj == 0 || (dj < 0 ? (ay == 0 || sy == 1) : (ay == 1 || sy == 0));
                        const bool kz = dk == 0 || (dk < 0 ? (az == 0 || sz == 1) : (az == 1 || sz == 0));
                        if (kx && ky && kz) {
                            st = bstart[nsub * b + ost * so];
                            len = bstart[nsub * b + ost * (so + 1)] - st;
                            use = len > 0;
                        }
                    }
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, use);
            if (use) {
                const int o = n_nb + __popc(m & ((1u << lane) - 1u));
                nb_start[o] = st;
                nb_pref[o] = len;  // lengths first, scanned below
            }
            n_nb += __popc(m);
        }
        __syncwarp();
        // exclusive scan of the lengths, four entries per lane
        int v[4], tot = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int o = 4 * lane + i;
            v[i] = o < n_nb ? nb_pref[o] : 0;
            tot += v[i];
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total_all = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        int run = incl - tot;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            nb_pref[4 * lane + i] = run;  // entries past n_nb hold the total
            run += v[i];
        }
        if (lane == 0) nb_pref[kNB] = total_all;
    }
    const int tb = oct < 0 ? tstart[nsub * cell] : tstart[nsub * cell + ost * oct];
    const int te = oct < 0 ? tstart[nsub * cell + nsub] : tstart[nsub * cell + ost * (oct + 1)];
    const int q = tb + sub * 32 + lane;
    const bool valid = q < te;
    double x = 0, y = 0, z = 0;
    if (valid) {
        x = tpx[q];
        y = tpy[q];
        z = tpz[q];
    }
    const double cxc = origin + (ci + 0.5) * side, cyc = origin + (cj + 0.5) * side,
                 czc = origin + (ck + 0.5) * side;
    // idle lanes sit at infinity: every candidate is certainly outside
    const float xf = valid ? rel32(x - cxc, ft.rm) : 3e38f;
    const float yf = valid ? rel32(y - cyc, ft.rm) : 3e38f;
    const float zf = valid ? rel32(z - czc, ft.rm) : 3e38f;
    double acc[3] = {0.0, 0.0, 0.0};
    __syncwarp();
    const int total = nb_pref[kNB];
    unsigned long long ncand = 0, npair = 0;  // work counters (roofline)
    // Chunks sample the neighbourhood with a coprime stride S ~ 0.618 total,
    // so every chunk mixes sources from all 27 buckets and each lane accepts
    // about the same number of pairs per chunk (bucket-ordered chunks left
    // ~10 of 32 lanes busy in the pair loop: a chunk from one corner bucket
    // is accepted only by the targets near that corner).
    int S = 1;
    if (total > 2) {
        S = static_cast<int>(0.6180339887 * total) | 1;
        while (gcd_int(S, total) != 1) S += 2;
    }
    for (int base = 0; base < total; base += CH) {
#pragma unroll
        for (int k = 0; k < CH / 32; ++k) {
            const int slot = k * 32 + lane;
            const int v = base + slot;
            if (v < total) {
                const int pos = static_cast<int>((static_cast<int64_t>(v) * S) % total);
                int r = 0;  // entry of pos: largest r with nb_pref[r] <= pos (none is empty)
#pragma unroll
                for (int stp = kNB / 2; stp > 0; stp >>= 1)
                    if (nb_pref[r + stp] <= pos) r += stp;
                const int sidx = nb_start[r] + (pos - nb_pref[r]);
                const double vx = spx[sidx], vy = spy[sidx], vz = spz[sidx];
                sx[slot] = vx;
                sy[slot] = vy;
                sz[slot] = vz;
                sxf[slot] = rel32(vx - cxc, ft.rm);
                syf[slot] = rel32(vy - cyc, ft.rm);
                szf[slot] = rel32(vz - czc, ft.rm);
#pragma unroll
                for (int c = 0; c < A; ++c)
                    sf[slot][c] = sfs[static_cast<int64_t>(sidx) * A + c];
            } else {  // past the last source: never accepted
                sxf[slot] = syf[slot] = szf[slot] = 3e38f;
            }
        }
        __syncwarp();
        const int cnt = min(CH, total - base);
        uint32_t mask[CH / 32];
        // two candidates per step with packed fp32 (FFMA2/FMUL2); slots past
        // cnt hold +3e38 sentinels, so the trip count is fixed
        const float2 xf2 = make_float2(xf, xf), yf2 = make_float2(yf, yf),
                     zf2 = make_float2(zf, zf), neg1 = make_float2(-1.0f, -1.0f);
#pragma unroll
        for (int wd = 0; wd < CH / 32; ++wd) {
            uint32_t m = 0, mx = 0;
#pragma unroll 4
            for (int b = 0; b < 32; b += 2) {
                const int j = wd * 32 + b;
                const float2 dx = __ffma2_rn(*reinterpret_cast<const float2*>(&sxf[j]), neg1, xf2);
                const float2 dy = __ffma2_rn(*reinterpret_cast<const float2*>(&syf[j]), neg1, yf2);
                const float2 dz = __ffma2_rn(*reinterpret_cast<const float2*>(&szf[j]), neg1, zf2);
                const float2 d2f = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float d = h ? d2f.y : d2f.x;
                    const bool in = d <= ft.lo && d > ft.z0;
                    // band, near-coincident or NaN: decided by the exact test below
                    const bool ex = !in && !(d > ft.hi);
                    m |= static_cast<uint32_t>(in) << (b + h);
                    mx |= static_cast<uint32_t>(ex) << (b + h);
                }
            }
            // the rare undecided candidates: the exact fp64 test of realspace.cpp:140
            // (out of the per-candidate loop, so that loop has no branch)
            while (mx) {
                const int b = __ffs(mx) - 1;
                mx &= mx - 1u;
                const int j = wd * 32 + b;
                const double d2 = exact_d2(x - sx[j], y - sy[j], z - sz[j]);
                if ((d2 != 0.0) && !(d2 > rc2)) m |= 1u << b;
            }
            mask[wd] = m;
        }
        // accepted pairs in ascending source order, one CH-bit mask per lane
        // (a single loop over all words balances the lanes better than a
        // loop per word)
        if (valid) {
            ncand += cnt;
#pragma unroll
            for (int i = 0; i < NW; ++i) npair += __popc(mask[i]);
        }
        if constexpr (NW <= 2) {
            // one 64-bit mask: a single loop over the accepted sources, ascending
            uint64_t mm = mask[0];
            if (NW == 2) mm |= static_cast<uint64_t>(mask[NW - 1]) << 32;
            while (mm) {
                const int j = __ffsll(static_cast<long long>(mm)) - 1;
                mm &= mm - 1;
                const double rx = x - sx[j], ry = y - sy[j], rz = z - sz[j];
                pair<KIND, TAIL>(rx, ry, rz, exact_d2(rx, ry, rz), xi, sf[j], tab, acc);
            }
        } else {
            // the mask words as a shift register: m[0] is the current word
            uint32_t m[NW];
#pragma unroll
            for (int i = 0; i < NW; ++i) m[i] = mask[i];
            int wbase = 0;
            while (true) {
                while (true) {
                    uint32_t rest = 0u;
#pragma unroll
                    for (int i = 1; i < NW; ++i) rest |= m[i];
                    if (m[0] != 0u || rest == 0u) break;
#pragma unroll
                    for (int i = 0; i + 1 < NW; ++i) m[i] = m[i + 1];
                    m[NW - 1] = 0u;
                    wbase += 32;
                }
                if (m[0] == 0u) break;
                const int j = wbase + __ffs(m[0]) - 1;
                m[0] &= m[0] - 1u;
                const double rx = x - sx[j], ry = y - sy[j], rz = z - sz[j];
                pair<KIND, TAIL>(rx, ry, rz, exact_d2(rx, ry, rz), xi, sf[j], tab, acc);
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ncand += __shfl_xor_sync(0xffffffffu, ncand, o);
        npair += __shfl_xor_sync(0xffffffffu, npair, o);
    }
    if (lane == 0) {
        atomicAdd(counts, ncand);
        atomicAdd(counts + 1, npair);
    }
    if (valid) {
        const int64_t m = tperm[q];
        u[3 * m] = acc[0];
        u[3 * m + 1] = acc[1];
        u[3 * m + 2] = acc[2];
    }
}

// ---------------------------------------------------------------------------
// CTA-shared variant (small inputs, see realspace_item_size; FSE_RS_WARP=0 forces it).
//
// Work item = (target cell, an even share of <= kTB of its targets) = one CTA.
// The concatenated 27 neighbour buckets are staged ONCE per CTA, in chunks of
// CAP sources, and shared by all its warps (the warp-item kernel stages them
// per 32 targets).  A warp takes one target at a time (dynamic counter) and
// sweeps the chunk, four candidates per lane and round, with the fp32 test of
// certainly-outside only (d2f > hi); survivors are compacted into a per-warp
// queue (ballot + popc), and whenever the queue holds 32 entries all 32 lanes
// evaluate one pair each, so the pair math runs with every lane busy (the
// warp-item kernel's per-lane mask loop keeps ~20 of 32 busy).  The exact
// closed-ball test of realspace.cpp:140 is applied to every queued pair, so
// the accepted set is the reference's.  Each target's sum is split over the
// lanes in queue order and reduced by a fixed xor tree: deterministic.
// 384 threads, two CTAs per SM, chunks of 1536 (768 for the stresslet's nine
// strengths) sources: ~108 KB of shared memory per CTA.  Build parameters for A/B.
#ifndef FSE_RSC_T
#define FSE_RSC_T 384
#endif
#ifndef FSE_RSC_MINB
#define FSE_RSC_MINB 2
#endif
#ifndef FSE_RSC_CAP3
#define FSE_RSC_CAP3 1536
#endif
#ifndef FSE_RSC_CAP9
#define FSE_RSC_CAP9 768
#endif
constexpr int kRT = FSE_RSC_T, kRW = kRT / 32, kTB = 128, kQ = 160;
template <int A>
constexpr int cta_cap() {
    return A == 3 ? FSE_RSC_CAP3 : FSE_RSC_CAP9;  // sources per chunk (whole 128-slot rounds)
}

template <int A>
struct CtaChunk {
    static constexpr int CAP = cta_cap<A>();
    double tab[kDeg + 1][kNI];
    double sx[CAP], sy[CAP], sz[CAP];
    double sf[CAP][A];
    double tx[kTB], ty[kTB], tz[kTB];
    double tacc[kTB][3];
    float sxf[CAP], syf[CAP], szf[CAP];  // relative to the cell centre; pads = 3e38
    int nb_start[27], nb_pref[28];
    int next_t;
    unsigned short q[kRW][kQ];
};

template <int KIND, bool TAIL>
__global__ void __launch_bounds__(kRT, FSE_RSC_MINB) k_realspace_cta(
    int dim, int nbk, const double* __restrict__ spx, const double* __restrict__ spy,
    const double* __restrict__ spz, const double* __restrict__ sfs,
    const int32_t* __restrict__ bstart, const double* __restrict__ tpx,
    const double* __restrict__ tpy, const double* __restrict__ tpz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ items,
    const uint32_t* __restrict__ tperm, const int32_t* __restrict__ nitems_dev, double xi,
    double rc2, double origin, double side, FastTest ft, unsigned long long* __restrict__ counts,
    double* __restrict__ u) {
    constexpr int A = KIND == FSE_STRESSLET ? 9 : 3;
    constexpr int CAP = cta_cap<A>();
    extern __shared__ __align__(16) unsigned char rs_smem[];
    CtaChunk<A>& S = *reinterpret_cast<CtaChunk<A>*>(rs_smem);
    const int item = blockIdx.x;
    if (item >= *nitems_dev) return;  // grid is an upper bound
    // lane from the special register through a volatile asm: the compiler otherwise
    // rematerialises it from %tid inside the test round (S2R latency, 4% of the stalls)
    int lane;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
    const int warp = threadIdx.x >> 5;
    const int cell = items[2 * item], sub = items[2 * item + 1];
    const int ck = cell % dim, cj = (cell / dim) % dim, ci = cell / (dim * dim);
    {
        const double* src = &c_erfcx[0][0];
        double* dst = &S.tab[0][0];
        for (int e = threadIdx.x; e < (kDeg + 1) * kNI; e += kRT) dst[e] = src[e];
    }
    if (warp == 0) {  // the 27 neighbour buckets, lexicographic (di, dj, dk), prefix-summed
        int len = 0, st = 0;
        if (lane < 27) {
            const int i = ci + lane / 9 - 1, j = cj + (lane / 3) % 3 - 1, k = ck + lane % 3 - 1;
            if (i >= 0 && i < dim && j >= 0 && j < dim && k >= 0 && k < dim) {
                const int b = (i * dim + j) * dim + k;
                st = bstart[nbk * b];  // (cell, sub-cell) bucket starts
                len = bstart[nbk * b + nbk] - st;
            }
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane < 27) {
            S.nb_start[lane] = st;
            S.nb_pref[lane] = incl - len;
        }
        if (lane == 26) S.nb_pref[27] = incl;
    }
    // this item's even share of the cell's targets
    const int t0c = tstart[nbk * cell], ntc = tstart[nbk * cell + nbk] - t0c;
    const int nsub = (ntc + kTB - 1) / kTB;
    const int lo = static_cast<int>(static_cast<int64_t>(sub) * ntc / nsub);
    const int ntb = static_cast<int>(static_cast<int64_t>(sub + 1) * ntc / nsub) - lo;
    const int q0 = t0c + lo;
    for (int t = threadIdx.x; t < ntb; t += kRT) {
        S.tx[t] = tpx[q0 + t];
        S.ty[t] = tpy[q0 + t];
        S.tz[t] = tpz[q0 + t];
        S.tacc[t][0] = S.tacc[t][1] = S.tacc[t][2] = 0.0;
    }
    const double cxc = origin + (ci + 0.5) * side, cyc = origin + (cj + 0.5) * side,
                 czc = origin + (ck + 0.5) * side;
    __syncthreads();
    const int total = S.nb_pref[27];
    unsigned long long npair = 0;
    unsigned short* q = S.q[warp];
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    static_assert(CAP % 128 == 0, "whole test rounds");
    for (int base = 0; base < total; base += CAP) {
        const int cnt = min(CAP, total - base);
        const int cnt_pad = (cnt + 127) & ~127;  // whole test rounds (CAP % 128 == 0)
        if (base > 0) __syncthreads();  // every warp is done with the previous chunk
        for (int e = threadIdx.x; e < cnt_pad; e += kRT) {
            if (e < cnt) {
                const int pos = base + e;
                int r = 0;  // bucket of pos: largest r with nb_pref[r] <= pos
#pragma unroll
                for (int stp = 16; stp > 0; stp >>= 1)
                    if (r + stp < 28 && S.nb_pref[r + stp] <= pos) r += stp;
                while (S.nb_pref[r + 1] <= pos) ++r;  // skip empty buckets
                const int sidx = S.nb_start[r] + (pos - S.nb_pref[r]);
                const double vx = spx[sidx], vy = spy[sidx], vz = spz[sidx];
                S.sx[e] = vx;
                S.sy[e] = vy;
                S.sz[e] = vz;
                S.sxf[e] = rel32(vx - cxc, ft.rm);
                S.syf[e] = rel32(vy - cyc, ft.rm);
                S.szf[e] = rel32(vz - czc, ft.rm);
#pragma unroll
                for (int c = 0; c < A; ++c) S.sf[e][c] = sfs[static_cast<int64_t>(sidx) * A + c];
            } else {  // pad: certainly outside in fp32 and in the exact test
                S.sxf[e] = S.syf[e] = S.szf[e] = 3e38f;
                S.sx[e] = S.sy[e] = S.sz[e] = 1e300;
#pragma unroll
                for (int c = 0; c < A; ++c) S.sf[e][c] = 0.0;
            }
        }
        if (threadIdx.x == 0) S.next_t = 0;
        __syncthreads();
        while (true) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&S.next_t, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= ntb) break;
            const double x = S.tx[t], y = S.ty[t], z = S.tz[t];
            // a target farther than Rm from its cell centre (outside the box, clamped
            // into an edge cell): NaN, so every candidate takes the exact test
            const float xf = rel32(x - cxc, ft.rm), yf = rel32(y - cyc, ft.rm),
                        zf = rel32(z - czc, ft.rm);
            const float2 xf2 = make_float2(xf, xf), yf2 = make_float2(yf, yf),
                         zf2 = make_float2(zf, zf), neg1 = make_float2(-1.0f, -1.0f);
            double acc[3] = {0.0, 0.0, 0.0};
            int qn = 0;
            auto eval = [&](int j) {
                const double rx = x - S.sx[j], ry = y - S.sy[j], rz = z - S.sz[j];
                const double d2 = exact_d2(rx, ry, rz);
                if ((d2 != 0.0) && !(d2 > rc2)) {  // realspace.cpp:140
                    pair<KIND, TAIL>(rx, ry, rz, d2, xi, S.sf[j], S.tab, acc);
                    ++npair;
                }
            };
            for (int r0 = 0; r0 < cnt_pad; r0 += 128) {
                const int e0 = r0 + 4 * lane;
                const float4 ax = *reinterpret_cast<const float4*>(&S.sxf[e0]);
                const float4 ay = *reinterpret_cast<const float4*>(&S.syf[e0]);
                const float4 az = *reinterpret_cast<const float4*>(&S.szf[e0]);
                const float2 dx0 = __ffma2_rn(make_float2(ax.x, ax.y), neg1, xf2);
                const float2 dx1 = __ffma2_rn(make_float2(ax.z, ax.w), neg1, xf2);
                const float2 dy0 = __ffma2_rn(make_float2(ay.x, ay.y), neg1, yf2);
                const float2 dy1 = __ffma2_rn(make_float2(ay.z, ay.w), neg1, yf2);
                const float2 dz0 = __ffma2_rn(make_float2(az.x, az.y), neg1, zf2);
                const float2 dz1 = __ffma2_rn(make_float2(az.z, az.w), neg1, zf2);
                const float2 d0 = __ffma2_rn(dx0, dx0, __ffma2_rn(dy0, dy0, __fmul2_rn(dz0, dz0)));
                const float2 d1 = __ffma2_rn(dx1, dx1, __ffma2_rn(dy1, dy1, __fmul2_rn(dz1, dz1)));
                // keep everything not certainly outside (NaN included)
                const bool p0 = !(d0.x > ft.hi), p1 = !(d0.y > ft.hi), p2 = !(d1.x > ft.hi),
                           p3 = !(d1.y > ft.hi);
                const unsigned b0 = __ballot_sync(0xffffffffu, p0), b1 = __ballot_sync(0xffffffffu, p1),
                               b2 = __ballot_sync(0xffffffffu, p2), b3 = __ballot_sync(0xffffffffu, p3);
                const int n0 = __popc(b0), n1 = __popc(b1), n2 = __popc(b2);
                const int o0 = qn + __popc(b0 & lt), o1 = qn + n0 + __popc(b1 & lt);
                const int o2 = qn + n0 + n1 + __popc(b2 & lt);
                const int o3 = qn + n0 + n1 + n2 + __popc(b3 & lt);
                if (p0) q[o0] = static_cast<unsigned short>(e0);
                if (p1) q[o1] = static_cast<unsigned short>(e0 + 1);
                if (p2) q[o2] = static_cast<unsigned short>(e0 + 2);
                if (p3) q[o3] = static_cast<unsigned short>(e0 + 3);
                qn += n0 + n1 + n2 + __popc(b3);
                __syncwarp();
                while (qn >= 32) {
                    qn -= 32;
                    eval(q[qn + lane]);
                }
                __syncwarp();  // the entries just read may be overwritten by the next round
            }
            if (lane < qn) eval(q[lane]);
            __syncwarp();
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
                acc[1] += __shfl_xor_sync(0xffffffffu, acc[1], o);
                acc[2] += __shfl_xor_sync(0xffffffffu, acc[2], o);
            }
            if (lane == 0) {
                S.tacc[t][0] += acc[0];
                S.tacc[t][1] += acc[1];
                S.tacc[t][2] += acc[2];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) npair += __shfl_xor_sync(0xffffffffu, npair, o);
    if (lane == 0 && npair) atomicAdd(counts + 1, npair);
    if (threadIdx.x == 0)
        atomicAdd(counts, static_cast<unsigned long long>(ntb) * static_cast<unsigned long long>(total));
    for (int e = threadIdx.x; e < 3 * ntb; e += kRT) {
        const int t = e / 3, c = e - 3 * t;
        u[3 * static_cast<int64_t>(tperm[q0 + t]) + c] = S.tacc[t][c];
    }
}

// Work items are scheduled heaviest cell first: the pair work of a cell is
// (its targets) x (sources in its 27 neighbour buckets), which varies by two
// orders of magnitude on clustered input (cfg4), and a heavy item dispatched
// last leaves the GPU waiting on a few warps.  Cells go to 32 buckets by
// log2(work) (bucket 0 heaviest); items are laid out bucket by bucket.  The
// order inside a bucket comes from atomics and only affects scheduling:
// every item computes the same targets' sums in the same order.
constexpr int kWorkBuckets = 32;

// sstart / tstart: (cell, octant) bucket starts (8 ncell + 1).  oct_min > 0: a cell
// with at least that many targets is cut into one item list per octant (item word 1 =
// sub | (octant + 1) << 24), whose neighbourhood is 125 of the 216 sub-buckets.
__device__ __forceinline__ int cell_items(const int32_t* __restrict__ tstart, int64_t c, int per,
                                          int oct_min, int sub) {
    const int nt = tstart[sub * c + sub] - tstart[sub * c];
    if (oct_min <= 0 || nt < oct_min) return (nt + per - 1) / per;
    const int ost = sub >> 3;
    int n = 0;
    for (int o = 0; o < 8; ++o)
        n += (tstart[sub * c + ost * (o + 1)] - tstart[sub * c + ost * o] + per - 1) / per;
    return n;
}

__global__ void k_cell_bucket(const int32_t* __restrict__ sstart, const int32_t* __restrict__ tstart,
                              int dim, int64_t ncell, int per, int64_t c_lo, int64_t c_hi,
                              int oct_min, int sub, uint8_t* __restrict__ bucket,
                              int32_t* __restrict__ bcount) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= ncell) return;
    const int nt = tstart[sub * c + sub] - tstart[sub * c];
    if (nt <= 0 || c < c_lo || c >= c_hi) return;
    const int ck = static_cast<int>(c % dim), cj = static_cast<int>((c / dim) % dim),
              ci = static_cast<int>(c / (static_cast<int64_t>(dim) * dim));
    int64_t cand = 0;
    for (int di = -1; di <= 1; ++di)
        for (int dj = -1; dj <= 1; ++dj)
            for (int dk = -1; dk <= 1; ++dk) {
                const int i = ci + di, j = cj + dj, k = ck + dk;
                if (i < 0 || i >= dim || j < 0 || j >= dim || k < 0 || k >= dim) continue;
                const int64_t b = (static_cast<int64_t>(i) * dim + j) * dim + k;
                cand += sstart[sub * b + sub] - sstart[sub * b];
            }
    const unsigned long long work = static_cast<unsigned long long>(nt) * (cand + 1);
    const int lg = 63 - __clzll(static_cast<long long>(work));  // floor(log2 work)
    const int bk = max(0, kWorkBuckets - 1 - lg);
    bucket[c] = static_cast<uint8_t>(bk);
    atomicAdd(bcount + bk, cell_items(tstart, c, per, oct_min, sub));
}

// one warp: bucket offsets (exclusive scan), item total for the pair kernel
__global__ void k_bucket_scan(const int32_t* __restrict__ bcount, int32_t* __restrict__ boff,
                              int32_t* __restrict__ nitems) {
    const int l = threadIdx.x;
    const int v = l < kWorkBuckets ? bcount[l] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += t;
    }
    if (l < kWorkBuckets) boff[l] = incl - v;
    if (l == 31) *nitems = incl;
}

__global__ void k_fill_items(const int32_t* __restrict__ tstart, const uint8_t* __restrict__ bucket,
                             int64_t ncell, int per, int64_t c_lo, int64_t c_hi, int oct_min,
                             int sub, const int32_t* __restrict__ boff,
                             int32_t* __restrict__ bcur, int32_t* __restrict__ items) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= ncell) return;
    const int nt = tstart[sub * c + sub] - tstart[sub * c];
    if (nt <= 0 || c < c_lo || c >= c_hi) return;
    const int n = cell_items(tstart, c, per, oct_min, sub), bk = bucket[c];
    const int ost = sub >> 3;
    int32_t at = boff[bk] + atomicAdd(bcur + bk, n);
    if (oct_min <= 0 || nt < oct_min) {
        for (int s = 0; s < n; ++s, ++at) {
            items[2 * at] = static_cast<int32_t>(c);
            items[2 * at + 1] = s;
        }
        return;
    }
    for (int o = 0; o < 8; ++o) {
        const int no = (tstart[sub * c + ost * (o + 1)] - tstart[sub * c + ost * o] + per - 1) / per;
        for (int s = 0; s < no; ++s, ++at) {
            items[2 * at] = static_cast<int32_t>(c);
            items[2 * at + 1] = s | ((o + 1) << 24);
        }
    }
}

// the tabulated functions in long double (s = 2/sqrt(pi), realspace.cpp:13-58
// rewritten as powers of 1/r times functions of x = xi r)
long double fn_ld(int which, long double x) {
    const long double sq = 1.128379167095512573896158903121545172L;  // 2/sqrt(pi)
    const long double e = expl(-x * x), ec = erfcl(x);
    switch (which) {
        case 0: return ec - sq * x * e;                           // Ahat
        case 1: return ec + sq * x * e;                           // Chat
        case 2: return 3.0L * ec + sq * x * (3.0L + 2.0L * x * x) * e;  // Dhat
        case 3: return 2.0L * sq * x * e;                         // Ehat
        case 4: return expl(x * x) * erfcl(x);                    // erfcx
        default: return 0.0L;
    }
}

// Chebyshev fit of function `which` on each interval, as monomials in t in [-1, 1]
void fit(int which, double out[kNI][kDeg + 1]) {
    const int n = kDeg + 1;
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int iv = 0; iv < kNI; ++iv) {
        const long double a = kXMax * iv / static_cast<long double>(kNI);
        const long double b = kXMax * (iv + 1) / static_cast<long double>(kNI);
        long double fv[n], cheb[n];
        for (int k = 0; k < n; ++k) {
            const long double t = cosl(PI * (k + 0.5L) / n);
            fv[k] = which < 0 ? 0.0L : fn_ld(which, 0.5L * (a + b) + 0.5L * (b - a) * t);
        }
        for (int j = 0; j < n; ++j) {
            long double sum = 0;
            for (int k = 0; k < n; ++k) sum += fv[k] * cosl(PI * j * (k + 0.5L) / n);
            cheb[j] = sum * 2.0L / n;
        }
        cheb[0] *= 0.5L;
        long double mono[n] = {}, Tprev[n] = {}, Tcur[n] = {}, Tnext[n];
        Tprev[0] = 1;
        Tcur[1] = 1;
        for (int j = 0; j < n; ++j) mono[j] += cheb[0] * Tprev[j] + cheb[1] * Tcur[j];
        for (int d = 2; d < n; ++d) {
            for (int j = 0; j < n; ++j) Tnext[j] = -Tprev[j] + (j > 0 ? 2 * Tcur[j - 1] : 0);
            for (int j = 0; j < n; ++j) mono[j] += cheb[d] * Tnext[j];
            for (int j = 0; j < n; ++j) {
                Tprev[j] = Tcur[j];
                Tcur[j] = Tnext[j];
            }
        }
        for (int j = 0; j < n; ++j) out[iv][j] = static_cast<double>(mono[j]);
    }
}

void ensure_tables() {
    static bool ready[64] = {};
    int dev = 0;
    FSE_CU(cudaGetDevice(&dev));
    if (dev < 64 && ready[dev]) return;
    static double tab[kDeg + 1][kNI];
    static bool built = false;
    if (!built) {
        static double f[kNI][kDeg + 1];
        fit(4, f);
        for (int iv = 0; iv < kNI; ++iv)
            for (int j = 0; j <= kDeg; ++j) tab[j][iv] = f[iv][j];
        built = true;
    }
    FSE_CU(cudaMemcpyToSymbol(c_erfcx, tab, sizeof tab));
    if (dev < 64) ready[dev] = true;
}

}  // namespace

// Which pair kernel: the warp-item kernel (32 targets per item) unless its items
// cannot fill the GPU -- fewer than ~2000 warps, e.g. cfg1's 216 cells of ~46
// targets -- where the CTA-shared kernel (kTB targets per item, 12 warps sharing
// one staged neighbourhood) is faster (cfg1 0.136 -> 0.048 ms).  On large inputs
// the warp-item kernel wins (cfg2 5.17 vs 5.25 ms, cfg3 2.33 vs 2.83, cfg4 91 vs
// 100: profiles/r02/cfg2_realspace_cta_kernel.md).  FSE_RS_WARP=1 / 0 forces one.
int realspace_item_size(int64_t nt, int64_t ncell) {
    static const int forced = [] {
        const char* e = std::getenv("FSE_RS_WARP");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    if (forced >= 0) return forced ? 32 : kTB;
    const int64_t warp_items = std::min<int64_t>(ncell, nt) + (nt + 31) / 32;
    return warp_items < 2000 ? kTB : 32;
}

void launch_realspace_items(const Launch& L, const int32_t* sstart, const int32_t* tstart,
                            int dim, int64_t ncell, int per, int64_t c_lo, int64_t c_hi,
                            uint8_t* bucket, int32_t* bwork, int32_t* items, int32_t* nitems,
                            int oct_min, int sub) {
    if (c_hi < 0) c_hi = ncell;
    if (sub < 8) oct_min = 0;
    int32_t* bcount = bwork;
    int32_t* boff = bwork + kWorkBuckets;
    int32_t* bcur = bwork + 2 * kWorkBuckets;
    FSE_CU(cudaMemsetAsync(bwork, 0, 3 * kWorkBuckets * sizeof(int32_t), L.s));
    const unsigned blocks = static_cast<unsigned>((ncell + 255) / 256);
    if (blocks > 0) {
        k_cell_bucket<<<blocks, 256, 0, L.s>>>(sstart, tstart, dim, ncell, per, c_lo, c_hi, oct_min,
                                               sub, bucket, bcount);
        FSE_LAUNCH_CHECK();
    }
    k_bucket_scan<<<1, 32, 0, L.s>>>(bcount, boff, nitems);
    FSE_LAUNCH_CHECK();
    if (blocks > 0) {
        k_fill_items<<<blocks, 256, 0, L.s>>>(tstart, bucket, ncell, per, c_lo, c_hi, oct_min, sub,
                                              boff, bcur, items);
        FSE_LAUNCH_CHECK();
    }
    *L.launches += blocks > 0 ? 3 : 1;
}

int realspace_work_buckets() { return kWorkBuckets; }

// Cells with at least this many targets are cut into octant items (42% fewer
// candidates each, at the price of up to eight partially filled items per cell).
// Measured on B200 with 8 sub-cells (real-space ms at thresholds off / 128 / 320 /
// 640): cfg4 85.0 / 82.9 / 82.6 / 82.3, cfg3 2.31 / 2.69 / 2.69 / 2.33, cfg2 (no cell
// that dense) 5.19; with 64 sub-cells off / 640: cfg4 80.2 / 77.5, cfg3 2.27 / 2.26.
// FSE_RS_OCT overrides (0: never).
int realspace_octant_threshold() {
    static const int t = [] {
        const char* e = std::getenv("FSE_RS_OCT");
        return e ? std::atoi(e) : 640;
    }();
    return t;
}

void launch_realspace(const Launch& L, int kind, const CellGrid& cg, const double* spx,
                      const double* spy, const double* spz, const double* sfs, int64_t ns,
                      const int32_t* bstart, const double* tpx, const double* tpy,
                      const double* tpz, const int32_t* tcell_start, const int32_t* items,
                      int64_t max_items, const int32_t* nitems_dev, const uint32_t* tperm,
                      double xi, double rc, unsigned long long* counts, double* uR, int per,
                      int sub) {
    (void)ns;
    if (max_items <= 0) return;
    ensure_tables();
    const double rc2 = rc * rc;
    const FastTest ft = fp32_bounds(rc, cg.side);
    // the table covers x = xi r < 6.5; past it (xi rc >= 6.5) the exact tail
    const bool tail = xi * rc >= kXMax * (1.0 - 1e-9);
    if (per == kTB) {  // CTA-shared kernel: the items were built with kTB targets each
        const unsigned b = static_cast<unsigned>(max_items);
        auto go = [&](auto kern, size_t sm) {
            FSE_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sm)));
            kern<<<b, kRT, sm, L.s>>>(cg.dim, sub, spx, spy, spz, sfs, bstart, tpx, tpy, tpz,
                                      tcell_start, items, tperm, nitems_dev, xi, rc2, cg.origin,
                                      cg.side, ft, counts, uR);
        };
        const size_t sm3 = sizeof(CtaChunk<3>), sm9 = sizeof(CtaChunk<9>);
        if (kind == FSE_STOKESLET)
            tail ? go(k_realspace_cta<FSE_STOKESLET, true>, sm3)
                 : go(k_realspace_cta<FSE_STOKESLET, false>, sm3);
        else if (kind == FSE_STRESSLET)
            tail ? go(k_realspace_cta<FSE_STRESSLET, true>, sm9)
                 : go(k_realspace_cta<FSE_STRESSLET, false>, sm9);
        else
            tail ? go(k_realspace_cta<FSE_ROTLET, true>, sm3)
                 : go(k_realspace_cta<FSE_ROTLET, false>, sm3);
        FSE_LAUNCH_CHECK();
        ++*L.launches;
        return;
    }
    const unsigned b = static_cast<unsigned>((max_items + TPB / 32 - 1) / (TPB / 32));
    const size_t sm3 = sizeof(WarpChunk<3>) * (TPB / 32), sm9 = sizeof(WarpChunk<9>) * (TPB / 32);
    auto go = [&](auto kern, size_t sm) {
        FSE_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sm)));
        kern<<<b, TPB, sm, L.s>>>(cg.dim, sub, spx, spy, spz, sfs, bstart, tpx, tpy, tpz, tcell_start,
                                  items, tperm, nitems_dev, xi, rc2, cg.origin, cg.side, ft, counts,
                                  uR);
    };
    if (kind == FSE_STOKESLET)
        tail ? go(k_realspace<FSE_STOKESLET, true>, sm3) : go(k_realspace<FSE_STOKESLET, false>, sm3);
    else if (kind == FSE_STRESSLET)
        tail ? go(k_realspace<FSE_STRESSLET, true>, sm9) : go(k_realspace<FSE_STRESSLET, false>, sm9);
    else
        tail ? go(k_realspace<FSE_ROTLET, true>, sm3) : go(k_realspace<FSE_ROTLET, false>, sm3);
    FSE_LAUNCH_CHECK();
    ++*L.launches;
}

}  // namespace fsecu
