// fp_tables.cpp -- host-side plan-time tables.
//
//   * roots of unity for the FFT engine, correctly rounded: the angle 2*pi*num/den
//     is reduced in exact integer arithmetic to the first octant before the
//     long-double sin/cos (cf. verify.basis_vector, verify.py:107-133, which
//     reduces its arguments the same way for the same reason);
//   * per-axis eigenvalue tables with the reference's operation order
//     (eigenvalues.py:51-77) so the device factor matches _inv_lam
//     (solver.py:151-159) to the last bit wherever libm's sin agrees with numpy's;
//   * dense transform matrices (direct definitions, transforms.py:3-15 and
//     naive_transform transforms.py:188-229) for the dense engine.
#include "fp_tables.h"

#include <cmath>
#include <cstdint>
#include <cstdlib>

namespace fpb {

// cos / sin of 2*pi*num/den, num reduced mod den, via octant symmetry.
void exact_cis(long long num, long long den, long double* c, long double* s) {
    num %= den;
    if (num < 0) num += den;
    // quadrant: theta = pi/2 * (4*num/den)
    const long long q4 = 4 * num;
    const long long quad = q4 / den;          // 0..3
    long long rem = q4 - quad * den;          // theta' = pi/2 * rem/den, rem in [0, den)
    const long double halfpi = 1.57079632679489661923132169163975144L;
    long double cc, ss;
    if (2 * rem <= den) {
        const long double a = halfpi * (long double)rem / (long double)den;
        cc = cosl(a);
        ss = sinl(a);
    } else {
        const long double a = halfpi * (long double)(den - rem) / (long double)den;
        cc = sinl(a);
        ss = cosl(a);
    }
    if (rem == 0) { cc = 1.0L; ss = 0.0L; }
    switch (quad) {
        case 0: *c = cc; *s = ss; break;
        case 1: *c = -ss; *s = cc; break;
        case 2: *c = -cc; *s = -ss; break;
        default: *c = ss; *s = -cc; break;
    }
}

// e^{-2 pi i num/den}
static void root(long long num, long long den, long double* re, long double* im) {
    long double c, s;
    exact_cis(num, den, &c, &s);
    *re = c;
    *im = -s;
}

// Per-stage Stockham twiddles, r-major (see stage_tw_offset in fp_common.cuh):
// for every radix-16 stage with Ns = 2^l > 1, entries [r][e] = W_M^{r e M/(16 Ns)}.
static void stage_twiddles(int M, std::vector<long double>& out) {
    int logM = 0;
    while ((1 << logM) < M) ++logM;
    out.clear();
    int l = (logM & 3) ? (logM & 3) : 4;
    for (; l < logM; l += 4) {
        const long long ns = 1LL << l;
        const long long step = M >> (l + 4);
        for (long long r = 0; r < 16; ++r)
            for (long long e = 0; e < ns; ++e) {
                long double re, im;
                root((r * e * step) % M, M, &re, &im);
                out.push_back(re);
                out.push_back(im);
            }
    }
    if (out.empty()) { out.push_back(1.0L); out.push_back(0.0L); }
}

void fft_tables(int n_real, int M, bool real_kind, std::vector<long double>& wfft,
                std::vector<long double>& wt, std::vector<long double>& ww) {
    stage_twiddles(M, wfft);
    wt.clear();
    ww.clear();
    if (real_kind) {
        const int n = n_real;
        wt.assign(2 * (size_t)(M + 1), 0.0L);
        ww.assign(2 * (size_t)(M + 1), 0.0L);
        for (int k = 0; k <= M; ++k) {
            root(k, n, &wt[2 * k], &wt[2 * k + 1]);          // e^{-2 pi i k/n}
            root(k, 4LL * n, &ww[2 * k], &ww[2 * k + 1]);    // e^{-i pi k/(2n)}
        }
    }
}

void mid_table(int n_real, int M, std::vector<long double>& wb) {
    wb.assign(2 * (size_t)(M + 1), 0.0L);
    for (int k = 0; k <= M; ++k) root(5LL * k, 4LL * n_real, &wb[2 * k], &wb[2 * k + 1]);   // e^{-5 i pi k/(2n)}
}

double axis_dx(const AxisSpec& a) {
    if (a.kind == 1) return a.length / (double)a.n;          // staggered
    if (a.bc == 0) return a.length / (double)a.n;             // periodic
    if (a.bc == 1) return a.length / (double)(a.n + 1);       // Dirichlet regular
    return a.length / (double)(a.n - 1);                      // Neumann regular
}

// eigenvalues.py:51-77, same operation order as the numpy expressions
std::vector<double> eigenvalue_table(const AxisSpec& a, int approx) {
    const long long n = a.n;
    std::vector<double> v((size_t)n);
    const double pi = 3.141592653589793;  // np.pi
    if (approx == 0) {  // PSEUDO_SPECTRAL
        for (long long k = 0; k < n; ++k) {
            const double kd = (double)k;
            double t;
            if (a.bc == 0) {
                const double folded = std::fmin(kd, (double)n - kd);
                t = 2.0 * pi * folded / a.length;
            } else if (a.bc == 1) {
                t = pi * (kd + 1.0) / a.length;
            } else {
                t = pi * kd / a.length;
            }
            v[(size_t)k] = -(t * t);
        }
    } else {
        const double dx = axis_dx(a);
        for (long long k = 0; k < n; ++k) {
            const double kd = (double)k;
            double ang;
            if (a.bc == 0) ang = kd * pi / (double)n;
            else if (a.bc == 1) ang = pi * (kd + 1.0) / (2.0 * (double)(a.kind == 0 ? n + 1 : n));
            else ang = pi * kd / (2.0 * (double)(a.kind == 0 ? n - 1 : n));
            const double t = 2.0 * std::sin(ang) / dx;
            v[(size_t)k] = -(t * t);
        }
    }
    return v;
}

// Dense matrices, row-major [n_out][n_in]; complex ones interleaved (re, im).
// kind uses the public FP_* transform ids.
// every entry of a dense matrix is cis(2 pi num / den) for one den per kind: the
// den roots are computed once (correctly rounded via exact_cis) and looked up,
// so building an n x n matrix costs O(den) trig calls instead of O(n^2)
namespace {
struct Roots {
    long long den;
    std::vector<long double> c, s;
    explicit Roots(long long d) : den(d), c((size_t)d), s((size_t)d) {
        for (long long q = 0; q < d; ++q) exact_cis(q, d, &c[(size_t)q], &s[(size_t)q]);
    }
    void get(long long num, long double* cc, long double* ss) const {
        num %= den;
        if (num < 0) num += den;
        *cc = c[(size_t)num];
        *ss = s[(size_t)num];
    }
};
}  // namespace

bool dense_matrix(int kind, int n, std::vector<double>& m, int* n_out, int* n_in, bool* cpx) {
    m.clear();
    long double c, s;
    if (kind == 0 || kind == 1) {  // DFT / IDFT (unnormalized here)
        *n_out = n; *n_in = n; *cpx = true;
        m.assign(2 * (size_t)n * n, 0.0);
        const Roots r(n);
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j) {
                r.get((long long)k * j, &c, &s);
                m[2 * ((size_t)k * n + j)] = (double)c;
                m[2 * ((size_t)k * n + j) + 1] = (double)(kind == 0 ? -s : s);
            }
        return true;
    }
    if (kind == 100) {  // real-input DFT, outputs k = 0..n/2
        const int h = n / 2 + 1;
        *n_out = h; *n_in = n; *cpx = true;
        m.assign(2 * (size_t)h * n, 0.0);
        const Roots r(n);
        for (int k = 0; k < h; ++k)
            for (int j = 0; j < n; ++j) {
                r.get((long long)k * j, &c, &s);
                m[2 * ((size_t)k * n + j)] = (double)c;
                m[2 * ((size_t)k * n + j) + 1] = (double)-s;
            }
        return true;
    }
    if (kind == 101) {  // Hermitian half-spectrum -> real, unnormalized inverse
        const int h = n / 2 + 1;
        *n_out = n; *n_in = h; *cpx = true;
        m.assign(2 * (size_t)n * h, 0.0);
        const Roots r(n);
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < h; ++k) {
                long double w = 2.0L;
                if (k == 0 || (n % 2 == 0 && k == n / 2)) w = 1.0L;
                r.get((long long)j * k, &c, &s);
                m[2 * ((size_t)j * h + k)] = (double)(w * c);
                m[2 * ((size_t)j * h + k) + 1] = (double)(w * s);
            }
        return true;
    }
    *n_out = n; *n_in = n; *cpx = false;
    long long den;
    switch (kind) {
        case 2: den = 2LL * (n + 1); break;          // DST1
        case 3: case 4: case 6: case 7: den = 4LL * n; break;
        case 5: den = 2LL * (n > 1 ? n - 1 : 1); break;   // DCT1
        default: return false;
    }
    const Roots r(den);
    m.assign((size_t)n * n, 0.0);
    for (int k = 0; k < n; ++k) {
        for (int j = 0; j < n; ++j) {
            long double val = 0.0L;
            switch (kind) {
                case 2:  // DST1: 2 sin(pi (j+1)(k+1)/(n+1))
                    r.get((long long)(j + 1) * (k + 1), &c, &s);
                    val = 2.0L * s;
                    break;
                case 3:  // DST2: 2 sin(pi (j+1/2)(k+1)/n)
                    r.get((long long)(2 * j + 1) * (k + 1), &c, &s);
                    val = 2.0L * s;
                    break;
                case 4:  // DST3: 2 sin(pi (j+1)(k+1/2)/n); column n-1: (-1)^k
                    if (j == n - 1) val = (k % 2 == 0) ? 1.0L : -1.0L;
                    else {
                        r.get((long long)(j + 1) * (2 * k + 1), &c, &s);
                        val = 2.0L * s;
                    }
                    break;
                case 5:  // DCT1: 2 cos(pi j k/(n-1)); column 0: 1; column n-1: (-1)^k
                    if (j == 0) val = 1.0L;
                    else if (j == n - 1) val = (k % 2 == 0) ? 1.0L : -1.0L;
                    else {
                        r.get((long long)j * k, &c, &s);
                        val = 2.0L * c;
                    }
                    break;
                case 6:  // DCT2: 2 cos(pi (j+1/2) k/n)
                    r.get((long long)(2 * j + 1) * k, &c, &s);
                    val = 2.0L * c;
                    break;
                default:  // 7, DCT3: 2 cos(pi j (k+1/2)/n); column 0: 1
                    if (j == 0) val = 1.0L;
                    else {
                        r.get((long long)j * (2 * k + 1), &c, &s);
                        val = 2.0L * c;
                    }
                    break;
            }
            m[(size_t)k * n + j] = (double)val;
        }
    }
    return true;
}

std::vector<int> mr_factors(long long N, int max_prime) {
    std::vector<int> f;
    if (N < 2) return f;
    long long m = N;
    static const int maxp2 = [] { const char* v = std::getenv("FP_MR_MAXPOW2"); return (v && *v) ? std::atoi(v) : 16; }();
    for (int r : {16, 8, 4, 2})
        while (r <= maxp2 && m % r == 0) { f.push_back(r); m /= r; }
    for (int p = 3; p <= max_prime && m > 1; p += 2)
        while (m % p == 0) { f.push_back(p); m /= p; }
    if (m != 1) f.clear();
    return f;
}

// input index j = d_1 + R_1 (d_2 + R_2 (...)) is read by the last stage's
// butterfly as sub-sequence j mod R_s: position (j mod R_s) * N / R_s + pos'(j / R_s)
std::vector<int> mr_perm(int N, const std::vector<int>& fac) {
    std::vector<int> p((size_t)N);
    for (int j0 = 0; j0 < N; ++j0) {
        int j = j0, pos = 0, mult = N;
        for (int q = (int)fac.size() - 1; q >= 0; --q) {
            const int R = fac[(size_t)q];
            mult /= R;
            pos += (j % R) * mult;
            j /= R;
        }
        p[(size_t)j0] = pos;
    }
    return p;
}

void root_table(long long den, long long count, std::vector<long double>& out) {
    out.assign(2 * (size_t)count, 0.0L);
    for (long long k = 0; k < count; ++k) root(k, den, &out[2 * (size_t)k], &out[2 * (size_t)k + 1]);
}

}  // namespace fpb
