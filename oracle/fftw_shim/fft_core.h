/*
 * fft_core.h -- TEST INFRASTRUCTURE (oracle), not product code.
 *
 * Plain-C complex DFT of arbitrary length (mixed-radix Stockham for factors
 * 2/3/4/5/generic-odd <= 64, Bluestein for lengths with a larger prime factor)
 * and an in-place row-major 3D transform on top of it.
 *
 * It stands in for FFTW3, the unvendored, unpinned third-party dependency the
 * reference's FFT seam calls (/root/reference/proj/src/fft.cpp:13-30:
 * fftw_plan_dft_3d(..., FFTW_ESTIMATE) in place, unnormalised, sign -1 forward
 * / +1 backward).  FFTW's published contract is the plain DFT
 *     X[k] = sum_j x[j] exp(sign * 2 pi i j k / n)
 * per axis; that is what is implemented here (validated against numpy.fft in
 * tests/test_oracle_fft.py to <= 1e-14 relative).
 *
 * The 3D transform is OpenMP-parallel over independent 1D lines (it uses
 * omp_get_max_threads(), i.e. the reference's own thread setting).  The
 * reference as written runs FFTW single-threaded (fft.cpp never calls
 * fftw_plan_with_nthreads), so this shim makes the reference's FFT stage
 * FASTER than it would be with FFTW as built upstream: a conservative CPU
 * baseline.  Results do not depend on the thread count (each line is
 * transformed by the same sequential code).
 */
#ifndef FSE_ORACLE_FFT_CORE_H
#define FSE_ORACLE_FFT_CORE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fc_plan1d fc_plan1d;

/* sign = -1 forward, +1 backward (unnormalised either way). */
fc_plan1d* fc_plan1d_create(int n, int sign);
void fc_plan1d_destroy(fc_plan1d* p);
/* in-place transform of n interleaved (re,im) doubles */
void fc_exec1d(fc_plan1d* p, double* data);

/* in-place unnormalised 3D DFT of an n0 x n1 x n2 row-major complex array */
void fc_fft3d(double* data, int n0, int n1, int n2, int sign);

#ifdef __cplusplus
}
#endif

#endif
