// fp_fft_f_l12.cu -- FFT pass kernel instances: float, FFT lengths 2^12..2^13
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_l12, float, 12, 13)
FP_FFT_WIDE(pick_wide_f_l12, float, 12)
