// fp_fft_f_hi.cu -- FFT pass kernel instances: float, FFT lengths 2^9..2^12
#include "fp_fft.cuh"

FP_FFT_PICK(pick_fft_f_hi, float, 9, 12)
