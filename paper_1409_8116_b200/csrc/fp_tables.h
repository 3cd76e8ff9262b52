// fp_tables.h -- plan-time host tables (see fp_tables.cpp)
#pragma once
#include <vector>

namespace fpb {

struct AxisSpec {
    long long n;
    double length;
    int bc;    // FP_BC_*
    int kind;  // FP_GRID_*
};

void exact_cis(long long num, long long den, long double* c, long double* s);
void fft_tables(int n_real, int M, bool real_kind, std::vector<long double>& wfft,
                std::vector<long double>& wt, std::vector<long double>& ww);
// w_k t_k = e^{-5 i pi k/(2n)}, k = 0..M: the second twiddle of the folded DCT-II /
// DST-II MID step (fp_common.cuh mid_quad)
void mid_table(int n_real, int M, std::vector<long double>& wb);
double axis_dx(const AxisSpec& a);
std::vector<double> eigenvalue_table(const AxisSpec& a, int approx);
// kind: FP_DFT..FP_DCT3, or 100 (real-input DFT half spectrum), 101 (half spectrum -> real)
bool dense_matrix(int kind, int n, std::vector<double>& m, int* n_out, int* n_in, bool* cpx);
// mixed-radix engine: radices of N (16, 8, 4, 2, then odd primes <= max_prime,
// stage order); empty if N has a larger prime factor
std::vector<int> mr_factors(long long N, int max_prime);
// digit-reversed position of every input index for the in-place DIT over `fac`
std::vector<int> mr_perm(int N, const std::vector<int>& fac);
// roots e^{-2 pi i k/den}, k = 0..count-1, interleaved (re, im)
void root_table(long long den, long long count, std::vector<long double>& out);

}  // namespace fpb
