// fp_fft_d_lo.cu -- FFT pass kernel instances: double, FFT lengths 2^4..2^8
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_lo, double, 4, 8)
