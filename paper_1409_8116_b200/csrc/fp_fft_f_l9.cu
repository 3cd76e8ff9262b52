// fp_fft_f_l9.cu -- FFT pass kernel instances: float, FFT lengths 2^9..2^10
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_l9, float, 9, 10)
