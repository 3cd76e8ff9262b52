// fp_fft_d_hi.cu -- FFT pass kernel instances: double, FFT lengths 2^9..2^12
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_d_hi, double, 9, 12)
