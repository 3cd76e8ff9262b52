// fp_fft_f_l11.cu -- FFT pass kernel instances: float, FFT lengths 2^11..2^11
// (one translation unit per length group so the build runs them in parallel)
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_l11, float, 11, 11)
FP_FFT_WIDE(pick_wide_f_l11, float, 11)
