// fp_fft_d_l9.cu -- FFT pass kernel instances: double, FFT lengths 2^9..2^10
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_l9, double, 9, 10)
