// fp_fft_d_l6.cu -- FFT pass kernel instances: double, FFT lengths 2^6..2^7
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_l6, double, 6, 7)
