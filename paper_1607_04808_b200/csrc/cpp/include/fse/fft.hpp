// fse/fft.hpp -- drop-in for the reference's FFT seam (fft.hpp:11,14), on cuFFT.
#pragma once

#include <complex>

namespace fse {

void fft3d_forward(std::complex<double>* data, int n0, int n1, int n2);
void fft3d_inverse(std::complex<double>* data, int n0, int n1, int n2);  // scaled by 1/n

}  // namespace fse
