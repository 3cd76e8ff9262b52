// fp_fft_f_l6.cu -- FFT pass kernel instances: float, FFT lengths 2^6..2^7
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_l6, float, 6, 7)
