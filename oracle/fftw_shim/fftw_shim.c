/*
 * fftw_shim.c -- TEST INFRASTRUCTURE (oracle): FFTW3 API over fft_core.c.
 * Unnormalised like FFTW; out-of-place plans copy `in` to `out` first.
 */
#include <stdlib.h>
#include <string.h>

#include "fft_core.h"
#include "fftw3.h"

struct fftw_plan_s {
    int n0, n1, n2, sign;
    double* in;
    double* out;
};

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags) {
    (void)flags;
    struct fftw_plan_s* p = (struct fftw_plan_s*)malloc(sizeof(*p));
    p->n0 = n0;
    p->n1 = n1;
    p->n2 = n2;
    p->sign = sign;
    p->in = (double*)in;
    p->out = (double*)out;
    return p;
}

void fftw_execute(const fftw_plan p) {
    const size_t total = (size_t)p->n0 * p->n1 * p->n2;
    if (p->out != p->in) memcpy(p->out, p->in, sizeof(double) * 2 * total);
    fc_fft3d(p->out, p->n0, p->n1, p->n2, p->sign);
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
