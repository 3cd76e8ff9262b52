// fp_fft_f_lo.cu -- FFT pass kernel instances: float, FFT lengths 2^4..2^8
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_lo, float, 4, 8)
