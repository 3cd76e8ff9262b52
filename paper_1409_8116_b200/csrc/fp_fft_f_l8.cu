// fp_fft_f_l8.cu -- FFT pass kernel instances: float, FFT lengths 2^8..2^8
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_l8, float, 8, 8)
