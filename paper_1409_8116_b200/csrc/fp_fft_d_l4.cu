// fp_fft_d_l4.cu -- FFT pass kernel instances: double, FFT lengths 2^4..2^5
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_l4, double, 4, 5)
