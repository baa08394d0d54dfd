/*
 * fft_core.c -- TEST INFRASTRUCTURE (oracle), not product code.
 * See fft_core.h.  Plain DFT, any length, unnormalised, single-threaded.
 *
 * Stockham autosort (decimation in time): with Ns = product of the radices
 * already applied and p the current radix, element j in [0, n/p) of a stage
 *   loads   v[r] = in[j + r n/p]
 *   twists  v[r] *= exp(sign 2 pi i r (j mod Ns) / (Ns p))
 *   applies the length-p DFT
 *   stores  out[(j / Ns) Ns p + (j mod Ns) + r Ns] = v[r].
 * Lengths with a prime factor > 64 go through Bluestein's chirp-z identity
 *   jk = (j^2 + k^2 - (k-j)^2) / 2 with a power-of-two convolution.
 */
#include "fft_core.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FC_MAX_STAGES 64
#define FC_GENERIC_MAX 64

typedef struct {
    int p;          /* radix */
    int Ns;         /* product of earlier radices */
    double* tw;     /* Ns * (p-1) complex twiddles, [k][r-1] */
    double* w;      /* p complex roots exp(sign 2 pi i t / p) (generic radix) */
} fc_stage;

struct fc_plan1d {
    int n;
    int sign;
    int nstages;
    fc_stage st[FC_MAX_STAGES];
    double* work;   /* 2n doubles */
    /* Bluestein */
    int blue;
    int m;
    double* chirp;  /* n complex: exp(sign pi i t^2 / n) */
    double* bhat;   /* m complex: FFT_m of conj chirp, circularly embedded */
    double* abuf;   /* m complex */
    fc_plan1d* fwd_m;
    fc_plan1d* inv_m;
};

static const double FC_PI = 3.14159265358979323846264338327950288;

static int largest_prime_factor(int n) {
    int lp = 1;
    for (int f = 2; (long long)f * f <= n; ++f)
        while (n % f == 0) { lp = f > lp ? f : lp; n /= f; }
    if (n > 1 && n > lp) lp = n;
    return lp;
}

static void cexp_angle(double a, double* re, double* im) {
    *re = cos(a);
    *im = sin(a);
}

static void build_stages(fc_plan1d* p) {
    int n = p->n, rem = n, Ns = 1, k = 0;
    int radices[FC_MAX_STAGES];
    while (rem % 4 == 0) { radices[k++] = 4; rem /= 4; }
    while (rem % 2 == 0) { radices[k++] = 2; rem /= 2; }
    for (int f = 3; rem > 1; f += 2)
        while (rem % f == 0) { radices[k++] = f; rem /= f; }
    p->nstages = k;
    for (int s = 0; s < k; ++s) {
        fc_stage* st = &p->st[s];
        st->p = radices[s];
        st->Ns = Ns;
        st->tw = (double*)malloc(sizeof(double) * 2 * (size_t)Ns * (st->p - 1 > 0 ? st->p - 1 : 1));
        for (int kk = 0; kk < Ns; ++kk)
            for (int r = 1; r < st->p; ++r) {
                /* reduce r*kk modulo Ns*p before forming the angle */
                long long num = ((long long)r * kk) % ((long long)Ns * st->p);
                double a = p->sign * 2.0 * FC_PI * (double)num / ((double)Ns * st->p);
                double* t = &st->tw[2 * ((size_t)kk * (st->p - 1) + (r - 1))];
                cexp_angle(a, &t[0], &t[1]);
            }
        st->w = NULL;
        if (st->p > 4) {
            st->w = (double*)malloc(sizeof(double) * 2 * st->p);
            for (int t = 0; t < st->p; ++t)
                cexp_angle(p->sign * 2.0 * FC_PI * t / st->p, &st->w[2 * t], &st->w[2 * t + 1]);
        }
        Ns *= st->p;
    }
}

static void run_stage(const fc_stage* st, int n, int sign, const double* in, double* out) {
    const int p = st->p, Ns = st->Ns, stride = n / p;
    double v[2 * FC_GENERIC_MAX], y[2 * FC_GENERIC_MAX];
    for (int j = 0; j < stride; ++j) {
        const int k = j % Ns;
        for (int r = 0; r < p; ++r) {
            v[2 * r] = in[2 * (j + r * stride)];
            v[2 * r + 1] = in[2 * (j + r * stride) + 1];
        }
        if (k != 0) {
            const double* tw = &st->tw[2 * (size_t)k * (p - 1)];
            for (int r = 1; r < p; ++r) {
                double a = v[2 * r], b = v[2 * r + 1];
                double c = tw[2 * (r - 1)], d = tw[2 * (r - 1) + 1];
                v[2 * r] = a * c - b * d;
                v[2 * r + 1] = a * d + b * c;
            }
        }
        if (p == 2) {
            y[0] = v[0] + v[2]; y[1] = v[1] + v[3];
            y[2] = v[0] - v[2]; y[3] = v[1] - v[3];
        } else if (p == 4) {
            /* omega = sign * i */
            double s0r = v[0] + v[4], s0i = v[1] + v[5];
            double d0r = v[0] - v[4], d0i = v[1] - v[5];
            double s1r = v[2] + v[6], s1i = v[3] + v[7];
            double d1r = v[2] - v[6], d1i = v[3] - v[7];
            /* (sign i) * d1 = (-sign d1i, sign d1r) */
            double jr = -sign * d1i, ji = sign * d1r;
            y[0] = s0r + s1r; y[1] = s0i + s1i;
            y[2] = d0r + jr;  y[3] = d0i + ji;
            y[4] = s0r - s1r; y[5] = s0i - s1i;
            y[6] = d0r - jr;  y[7] = d0i - ji;
        } else if (p == 3) {
            const double h = 0.86602540378443864676372317075293618 * sign;
            double t1r = v[2] + v[4], t1i = v[3] + v[5];
            double t2r = v[0] - 0.5 * t1r, t2i = v[1] - 0.5 * t1i;
            double t3r = h * (v[2] - v[4]), t3i = h * (v[3] - v[5]);
            y[0] = v[0] + t1r; y[1] = v[1] + t1i;
            /* t2 + i t3 */
            y[2] = t2r - t3i; y[3] = t2i + t3r;
            y[4] = t2r + t3i; y[5] = t2i - t3r;
        } else {
            const double* w = st->w;
            for (int q = 0; q < p; ++q) {
                double ar = 0, ai = 0;
                int t = 0;
                for (int r = 0; r < p; ++r) {
                    double c = w[2 * t], d = w[2 * t + 1];
                    ar += v[2 * r] * c - v[2 * r + 1] * d;
                    ai += v[2 * r] * d + v[2 * r + 1] * c;
                    t += q;
                    if (t >= p) t -= p;
                }
                y[2 * q] = ar;
                y[2 * q + 1] = ai;
            }
        }
        const int base = (j / Ns) * Ns * p + k;
        for (int r = 0; r < p; ++r) {
            out[2 * (base + r * Ns)] = y[2 * r];
            out[2 * (base + r * Ns) + 1] = y[2 * r + 1];
        }
    }
}

fc_plan1d* fc_plan1d_create(int n, int sign) {
    if (n < 1) return NULL;
    fc_plan1d* p = (fc_plan1d*)calloc(1, sizeof(fc_plan1d));
    p->n = n;
    p->sign = sign < 0 ? -1 : 1;
    p->work = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    if (largest_prime_factor(n) > FC_GENERIC_MAX) {
        p->blue = 1;
        int m = 1;
        while (m < 2 * n - 1) m <<= 1;
        p->m = m;
        p->chirp = (double*)malloc(sizeof(double) * 2 * (size_t)n);
        for (int t = 0; t < n; ++t) {
            long long q = ((long long)t * t) % (2LL * n);
            cexp_angle(p->sign * FC_PI * (double)q / n, &p->chirp[2 * t], &p->chirp[2 * t + 1]);
        }
        p->fwd_m = fc_plan1d_create(m, -1);
        p->inv_m = fc_plan1d_create(m, +1);
        p->bhat = (double*)calloc(2 * (size_t)m, sizeof(double));
        p->abuf = (double*)malloc(sizeof(double) * 2 * (size_t)m);
        for (int t = 0; t < n; ++t) {
            /* b_t = conj(chirp_t), embedded at t and m - t */
            p->bhat[2 * t] = p->chirp[2 * t];
            p->bhat[2 * t + 1] = -p->chirp[2 * t + 1];
            if (t > 0) {
                p->bhat[2 * (m - t)] = p->chirp[2 * t];
                p->bhat[2 * (m - t) + 1] = -p->chirp[2 * t + 1];
            }
        }
        fc_exec1d(p->fwd_m, p->bhat);
    } else {
        build_stages(p);
    }
    return p;
}

void fc_plan1d_destroy(fc_plan1d* p) {
    if (!p) return;
    for (int s = 0; s < p->nstages; ++s) {
        free(p->st[s].tw);
        free(p->st[s].w);
    }
    free(p->work);
    free(p->chirp);
    free(p->bhat);
    free(p->abuf);
    fc_plan1d_destroy(p->fwd_m);
    fc_plan1d_destroy(p->inv_m);
    free(p);
}

void fc_exec1d(fc_plan1d* p, double* data) {
    const int n = p->n;
    if (p->blue) {
        const int m = p->m;
        double* a = p->abuf;
        for (int t = 0; t < n; ++t) {
            double xr = data[2 * t], xi = data[2 * t + 1];
            double cr = p->chirp[2 * t], ci = p->chirp[2 * t + 1];
            a[2 * t] = xr * cr - xi * ci;
            a[2 * t + 1] = xr * ci + xi * cr;
        }
        memset(a + 2 * (size_t)n, 0, sizeof(double) * 2 * (size_t)(m - n));
        fc_exec1d(p->fwd_m, a);
        for (int t = 0; t < m; ++t) {
            double xr = a[2 * t], xi = a[2 * t + 1];
            double br = p->bhat[2 * t], bi = p->bhat[2 * t + 1];
            a[2 * t] = xr * br - xi * bi;
            a[2 * t + 1] = xr * bi + xi * br;
        }
        fc_exec1d(p->inv_m, a);
        const double inv = 1.0 / m;
        for (int t = 0; t < n; ++t) {
            double xr = a[2 * t] * inv, xi = a[2 * t + 1] * inv;
            double cr = p->chirp[2 * t], ci = p->chirp[2 * t + 1];
            data[2 * t] = xr * cr - xi * ci;
            data[2 * t + 1] = xr * ci + xi * cr;
        }
        return;
    }
    if (p->nstages == 0) return; /* n == 1 */
    double* src = data;
    double* dst = p->work;
    for (int s = 0; s < p->nstages; ++s) {
        run_stage(&p->st[s], n, p->sign, src, dst);
        double* t = src;
        src = dst;
        dst = t;
    }
    if (src != data) memcpy(data, src, sizeof(double) * 2 * (size_t)n);
}

/* ---- batched path: LB lines at once, layout buf[j][b] (line index fastest),
 * so every butterfly's inner loop runs over LB independent lines with the
 * same twiddle (vectorisable).  Same per-element arithmetic as run_stage. */
enum { LB = 16 };

static void run_stage_batch(const fc_stage* st, int n, int sign, const double* in,
                            double* out) {
    const int p = st->p, Ns = st->Ns, stride = n / p;
    double v[2 * FC_GENERIC_MAX * LB];
    for (int j = 0; j < stride; ++j) {
        const int k = j % Ns;
        for (int r = 0; r < p; ++r)
            memcpy(&v[2 * r * LB], &in[2 * (size_t)(j + r * stride) * LB], sizeof(double) * 2 * LB);
        if (k != 0) {
            const double* tw = &st->tw[2 * (size_t)k * (p - 1)];
            for (int r = 1; r < p; ++r) {
                const double c = tw[2 * (r - 1)], d = tw[2 * (r - 1) + 1];
                double* x = &v[2 * r * LB];
                for (int b = 0; b < LB; ++b) {
                    const double a = x[2 * b], e = x[2 * b + 1];
                    x[2 * b] = a * c - e * d;
                    x[2 * b + 1] = a * d + e * c;
                }
            }
        }
        const int base = (j / Ns) * Ns * p + k;
        double* o[FC_GENERIC_MAX];
        for (int r = 0; r < p; ++r) o[r] = &out[2 * (size_t)(base + r * Ns) * LB];
        if (p == 2) {
            for (int b = 0; b < LB; ++b) {
                const double* x0 = &v[2 * b];
                const double* x1 = &v[2 * (LB + b)];
                o[0][2 * b] = x0[0] + x1[0]; o[0][2 * b + 1] = x0[1] + x1[1];
                o[1][2 * b] = x0[0] - x1[0]; o[1][2 * b + 1] = x0[1] - x1[1];
            }
        } else if (p == 4) {
            for (int b = 0; b < LB; ++b) {
                const double* x0 = &v[2 * b];
                const double* x1 = &v[2 * (LB + b)];
                const double* x2 = &v[2 * (2 * LB + b)];
                const double* x3 = &v[2 * (3 * LB + b)];
                double s0r = x0[0] + x2[0], s0i = x0[1] + x2[1];
                double d0r = x0[0] - x2[0], d0i = x0[1] - x2[1];
                double s1r = x1[0] + x3[0], s1i = x1[1] + x3[1];
                double d1r = x1[0] - x3[0], d1i = x1[1] - x3[1];
                double jr = -sign * d1i, ji = sign * d1r;
                o[0][2 * b] = s0r + s1r; o[0][2 * b + 1] = s0i + s1i;
                o[1][2 * b] = d0r + jr;  o[1][2 * b + 1] = d0i + ji;
                o[2][2 * b] = s0r - s1r; o[2][2 * b + 1] = s0i - s1i;
                o[3][2 * b] = d0r - jr;  o[3][2 * b + 1] = d0i - ji;
            }
        } else if (p == 3) {
            const double h = 0.86602540378443864676372317075293618 * sign;
            for (int b = 0; b < LB; ++b) {
                const double* x0 = &v[2 * b];
                const double* x1 = &v[2 * (LB + b)];
                const double* x2 = &v[2 * (2 * LB + b)];
                double t1r = x1[0] + x2[0], t1i = x1[1] + x2[1];
                double t2r = x0[0] - 0.5 * t1r, t2i = x0[1] - 0.5 * t1i;
                double t3r = h * (x1[0] - x2[0]), t3i = h * (x1[1] - x2[1]);
                o[0][2 * b] = x0[0] + t1r; o[0][2 * b + 1] = x0[1] + t1i;
                o[1][2 * b] = t2r - t3i;   o[1][2 * b + 1] = t2i + t3r;
                o[2][2 * b] = t2r + t3i;   o[2][2 * b + 1] = t2i - t3r;
            }
        } else {
            const double* w = st->w;
            for (int q = 0; q < p; ++q) {
                double acc[2 * LB];
                memset(acc, 0, sizeof acc);
                int t = 0;
                for (int r = 0; r < p; ++r) {
                    const double c = w[2 * t], d = w[2 * t + 1];
                    const double* x = &v[2 * r * LB];
                    for (int b = 0; b < LB; ++b) {
                        acc[2 * b] += x[2 * b] * c - x[2 * b + 1] * d;
                        acc[2 * b + 1] += x[2 * b] * d + x[2 * b + 1] * c;
                    }
                    t += q;
                    if (t >= p) t -= p;
                }
                memcpy(o[q], acc, sizeof acc);
            }
        }
    }
}

/* In-place transform of LB lines stored as buf[j][b]; work holds 2*n*LB doubles. */
static void exec_batch(fc_plan1d* p, double* buf, double* work, double* line) {
    const int n = p->n;
    if (p->blue || p->nstages == 0) {
        if (p->nstages == 0 && !p->blue) return;
        for (int b = 0; b < LB; ++b) {
            for (int j = 0; j < n; ++j) {
                line[2 * j] = buf[2 * ((size_t)j * LB + b)];
                line[2 * j + 1] = buf[2 * ((size_t)j * LB + b) + 1];
            }
            fc_exec1d(p, line);
            for (int j = 0; j < n; ++j) {
                buf[2 * ((size_t)j * LB + b)] = line[2 * j];
                buf[2 * ((size_t)j * LB + b) + 1] = line[2 * j + 1];
            }
        }
        return;
    }
    double* src = buf;
    double* dst = work;
    for (int s = 0; s < p->nstages; ++s) {
        run_stage_batch(&p->st[s], n, p->sign, src, dst);
        double* t = src;
        src = dst;
        dst = t;
    }
    if (src != buf) memcpy(buf, src, sizeof(double) * 2 * (size_t)n * LB);
}

/* Transform lines of length n with element stride `stride` (complex units):
 * line (o, c) starts at data + o*outer_stride + c*cstride.  LB lines are
 * gathered into buf[j][b]; the (outer, block) items are independent and split
 * over OpenMP threads, each with its own plan and buffers. */
static void lines_strided(double* data, size_t nlines_outer, size_t outer_stride, int n,
                          size_t stride, size_t count, size_t cstride, int sign) {
    const size_t nblk = (count + LB - 1) / LB;
    const long long items = (long long)(nlines_outer * nblk);
#pragma omp parallel
    {
        fc_plan1d* plan = fc_plan1d_create(n, sign);
        double* buf = (double*)calloc(2 * (size_t)n * LB, sizeof(double));
        double* work = (double*)malloc(sizeof(double) * 2 * (size_t)n * LB);
        double* line = (double*)malloc(sizeof(double) * 2 * (size_t)n);
#pragma omp for schedule(static)
        for (long long it = 0; it < items; ++it) {
            const size_t o = (size_t)it / nblk, c0 = ((size_t)it % nblk) * LB;
            double* base = data + 2 * o * outer_stride;
            const size_t nb = count - c0 < LB ? count - c0 : LB;
            for (int j = 0; j < n; ++j)
                for (size_t b = 0; b < nb; ++b) {
                    const double* src = base + 2 * ((size_t)j * stride + (c0 + b) * cstride);
                    buf[2 * ((size_t)j * LB + b)] = src[0];
                    buf[2 * ((size_t)j * LB + b) + 1] = src[1];
                }
            exec_batch(plan, buf, work, line);
            for (int j = 0; j < n; ++j)
                for (size_t b = 0; b < nb; ++b) {
                    double* dst = base + 2 * ((size_t)j * stride + (c0 + b) * cstride);
                    dst[0] = buf[2 * ((size_t)j * LB + b)];
                    dst[1] = buf[2 * ((size_t)j * LB + b) + 1];
                }
        }
        free(line);
        free(work);
        free(buf);
        fc_plan1d_destroy(plan);
    }
}

void fc_fft3d(double* data, int n0, int n1, int n2, int sign) {
    /* axis 2: contiguous rows (element stride 1, rows n2 apart) */
    lines_strided(data, 1, 0, n2, 1, (size_t)n0 * n1, (size_t)n2, sign);
    /* axis 1: stride n2, n0 outer blocks */
    lines_strided(data, (size_t)n0, (size_t)n1 * n2, n1, (size_t)n2, (size_t)n2, 1, sign);
    /* axis 0: stride n1*n2 */
    lines_strided(data, 1, 0, n0, (size_t)n1 * n2, (size_t)n1 * n2, 1, sign);
}
