// fp_fft_d_l11.cu -- FFT pass kernel instances: double, FFT lengths 2^11..2^11
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_l11, double, 11, 11)
