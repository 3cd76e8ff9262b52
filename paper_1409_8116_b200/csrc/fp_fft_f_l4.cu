// fp_fft_f_l4.cu -- FFT pass kernel instances: float, FFT lengths 2^4..2^5
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_l4, float, 4, 5)
