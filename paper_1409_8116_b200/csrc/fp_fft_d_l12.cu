// fp_fft_d_l12.cu -- FFT pass kernel instances: double, FFT lengths 2^12..2^13
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_l12, double, 12, 13)
