/*
 * fftw3.h -- TEST INFRASTRUCTURE (oracle): minimal FFTW3-API shim.
 *
 * The reference's FFT seam (/root/reference/proj/src/fft.cpp:13-30) includes
 * <fftw3.h> and calls exactly fftw_plan_dft_3d (in place, FFTW_ESTIMATE),
 * fftw_execute and fftw_destroy_plan.  FFTW3 is not installed in this image
 * (unvendored and unpinned: proj/CMakeLists.txt:24 links plain "fftw3"), so
 * this header declares that surface and fftw_shim.c implements it over the
 * plain-C DFT in fft_core.c.  Only oracle/_ref (the reference compiled from
 * its own sources) is built against it.
 */
#ifndef FSE_ORACLE_FFTW3_SHIM_H
#define FSE_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif

#endif
