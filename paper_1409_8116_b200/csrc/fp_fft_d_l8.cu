// fp_fft_d_l8.cu -- FFT pass kernel instances: double, FFT lengths 2^8..2^8
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_l8, double, 8, 8)
