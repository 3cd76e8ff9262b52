// fp_blue.cu -- the Bluestein (chirp-z) line engine: every transform kind at ANY
// length, O(n log n).  It takes the axes neither the power-of-two FFT engine nor
// the mixed-radix engine can (a prime factor above 61, or lines longer than one
// CTA's shared memory), which the reference handles through scipy.fft at any n
// (transforms.py:70-77,128-177).
//
// Each kind is the complex DFT of length N of a recipe sequence z (the same
// recipes as the mixed-radix engine, fp_mr.cu; checked against scipy in
// oracle.blue_transform):
//   DFT / IDFT   z = x,                       N = n, sign - / +
//   real FFT     z = x (real),                N = n, sign -, outputs k <= n/2
//   inverse rFFT z = Hermitian extension,     N = n, sign +, x_j = Re v_j
//   DCT-II       z = Makhoul reordering of x, N = n, sign -, X_k = 2 Re(w_k Z_k)
//   DST-II       DCT-II of (-1)^j x, outputs reversed
//   DCT-III      z_0 = X_0, z_k = conj(w_k) (X_k - i X_{n-k}), N = n, sign +,
//                x_2j = Re v_j, x_2j+1 = Re v_{n-1-j}
//   DST-III      (-1)^j DCT-III(reversed X)
//   DCT-I        even extension, N = 2(n-1), sign -, X_k = Re Z_k
//   DST-I        odd extension [0, x, 0, -reversed x], N = 2(n+1), sign -, X_k = -Im Z_{k+1}
// and the DFT is Bluestein's identity jk = (j^2 + k^2 - (k-j)^2)/2:
//   Z_k = conj(c_k) sum_j (z_j conj(c_j)) c_{k-j},  c_m = e^{i pi m^2/N}   (sign -; conjugate all for +)
// -- a linear convolution of length 2N-1, done as a cyclic one of length L (power
// of two) with the FFT engine: forward FFT_L, pointwise product with the plan-time
// spectrum of the chirp filter (1/L folded in), inverse FFT_L.  Long L run as
// L1 x L2 four-step FFTs (fp_plan.cu run_blue); the four-step's output order needs
// no transpose because the filter spectrum is stored in that same order.
//
// Kernels (all elementwise, grid-stride, plan-typed scratch [line][L] complex):
//   blue_gather  recipe + pre-chirp + zero padding   (reads the lines once)
//   blue_mul     pointwise product with the filter spectrum
//   blue_twiddle four-step twiddles W_L^{-+k1 j2}
//   blue_emit    post-chirp + output recipe          (writes the lines once)
//   blue_filter / blue_scale: plan-time filter and its scaled spectrum
#include <cuda_runtime.h>

#include "../../include/fastpoisson_b200.h"
#include "fp_common.cuh"

namespace fpb {

namespace {

template <typename T>
__device__ __forceinline__ cx<T> chirp_at(const BluePass& p, long long m) {
    const cx<T> c = reinterpret_cast<const cx<T>*>(p.chirp)[m];
    return p.inv ? c : mkc<T>(c.x, -c.y);   // sign -: conj(c_m); sign +: c_m
}

// z_j of the kind's recipe (j < N) for the line at element offset `base`
template <typename T>
__device__ __forceinline__ cx<T> blue_src(const BluePass& p, long long base, long long j, bool& bad) {
    const Geometry& g = p.g;
    const long long n = p.n, st = g.in_st;
    auto rx = [&](long long i) {
        const T v = ld_real<T>(g.in, g.in_type, base + i * st);
        bad |= !finite_t(v);
        return v;
    };
    auto cxin = [&](long long i) {
        const cx<T> v = ld_cx<T>(g.in, g.in_type, base + i * st);
        bad |= !(finite_t(v.x) && finite_t(v.y));
        return v;
    };
    switch (p.kind) {
        case FP_DFT:
        case FP_IDFT:
            return cxin(j);
        case MR_RFFT:
            return mkc<T>(rx(j), 0);
        case MR_IRFFT: {
            const long long h = n / 2 + 1;
            if (j < h) return cxin(j);
            const cx<T> v = cxin(n - j);
            return mkc<T>(v.x, -v.y);
        }
        case FP_DCT2:
        case FP_DST2: {
            const long long i = (2 * j <= n - 1) ? 2 * j : 2 * (n - 1 - j) + 1;   // Makhoul: v_j = x_i
            T v = rx(i);
            if (p.kind == FP_DST2 && (i & 1)) v = -v;
            return mkc<T>(v, 0);
        }
        case FP_DCT3:
        case FP_DST3: {
            const bool dst = p.kind == FP_DST3;
            auto X = [&](long long k) { return rx(dst ? n - 1 - k : k); };
            if (j == 0) return mkc<T>(X(0), 0);
            const T a = X(j), b = X(n - j);
            const cx<T> w = reinterpret_cast<const cx<T>*>(p.wq)[j];
            return cmulc<T>(mkc<T>(a, -b), w);   // conj(w_j) (X_j - i X_{n-j})
        }
        case FP_DCT1: {
            const long long i = j <= n - 1 ? j : 2 * (n - 1) - j;
            return mkc<T>(rx(i), 0);
        }
        default: {   // FP_DST1
            if (j == 0 || j == n + 1) return mkc<T>(0, 0);
            if (j <= n) return mkc<T>(rx(j - 1), 0);
            return mkc<T>(-rx(2 * n + 1 - j), 0);
        }
    }
}

template <typename T>
__global__ void blue_gather(const BluePass p, cx<T>* __restrict__ S, long long l0, long long cl) {
    const long long total = cl * p.L;
    const int logL = __ffs(p.L) - 1;
    bool bad = false;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx >> logL;
        const long long j = idx & (p.L - 1);
        cx<T> z = mkc<T>(0, 0);
        if (j < p.N) {
            const long long l = l0 + c;
            const long long ia = l / p.g.nb, ib = l - ia * p.g.nb;
            const long long base = ia * p.g.in_sa + ib * p.g.in_sb;
            z = cmul<T>(blue_src<T>(p, base, j, bad), chirp_at<T>(p, j));
        }
        S[idx] = z;
    }
    if (bad && p.nonfinite) *p.nonfinite = 1;
}

template <typename T>
__device__ __forceinline__ cx<T> blue_Z(const BluePass& p, const cx<T>* S, long long row, long long m) {
    return cmul<T>(S[row + m], chirp_at<T>(p, m));
}

template <typename T>
__global__ void blue_emit(const BluePass p, const cx<T>* __restrict__ S, long long l0, long long cl) {
    const long long no = p.n_out, n = p.n;
    const long long total = cl * no;
    const Geometry& g = p.g;
    const T om = (T)p.out_mult;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / no;
        const long long k = idx - c * no;
        const long long l = l0 + c;
        const long long ia = l / g.nb, ib = l - ia * g.nb;
        const long long o = ia * g.out_sa + ib * g.out_sb + k * g.out_st;
        const long long row = c * p.L;
        switch (p.kind) {
            case FP_DFT:
            case FP_IDFT:
            case MR_RFFT:
                st_cx<T>(g.out, g.out_type, o, cscale<T>(blue_Z<T>(p, S, row, k), om));
                break;
            case MR_IRFFT:
            case FP_DCT1:
                st_real<T>(g.out, g.out_type, o, blue_Z<T>(p, S, row, k).x * om);
                break;
            case FP_DST1:
                st_real<T>(g.out, g.out_type, o, -blue_Z<T>(p, S, row, k + 1).y * om);
                break;
            case FP_DCT2:
            case FP_DST2: {
                const long long kk = p.kind == FP_DST2 ? n - 1 - k : k;
                const cx<T> w = reinterpret_cast<const cx<T>*>(p.wq)[kk];
                const cx<T> U = cmul<T>(w, blue_Z<T>(p, S, row, kk));
                st_real<T>(g.out, g.out_type, o, (T)2 * U.x * om);
                break;
            }
            default: {   // FP_DCT3 / FP_DST3
                const long long m = (k & 1) ? n - 1 - (k >> 1) : (k >> 1);
                T v = blue_Z<T>(p, S, row, m).x * om;
                if (p.kind == FP_DST3 && (k & 1)) v = -v;
                st_real<T>(g.out, g.out_type, o, v);
                break;
            }
        }
    }
}

template <typename T>
__global__ void blue_mul(cx<T>* __restrict__ S, const cx<T>* __restrict__ bhat, long long cl, int L) {
    const long long total = cl * L;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x)
        S[idx] = cmul<T>(S[idx], bhat[idx & (L - 1)]);
}

// element (k1, j2) of an L1 x L2 row (index k1 L2 + j2) times e^{-+2 pi i k1 j2 / L}
template <typename T>
__global__ void blue_twiddle(cx<T>* __restrict__ S, long long cl, int L1, int L2, int inv) {
    const long long L = (long long)L1 * L2;
    const long long total = cl * L;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long e = idx & (L - 1);
        const long long k1 = e / L2, j2 = e - k1 * L2;
        const long long r = (k1 * j2) & (L - 1);   // exact reduction of the angle
        double s, c;
        sincospi(2.0 * (double)r / (double)L, &s, &c);
        const cx<T> w = mkc<T>((T)c, inv ? (T)s : (T)-s);
        S[idx] = cmul<T>(S[idx], w);
    }
}

// the chirp filter h (one row of L): h_m = c_m, h_{L-m} = c_m (0 < m < N), 0 elsewhere;
// conjugated for sign +
template <typename T>
__global__ void blue_filter(cx<T>* __restrict__ S, const cx<T>* __restrict__ chirp, int N, int L, int conj) {
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L; m += gridDim.x * blockDim.x) {
        cx<T> h = mkc<T>(0, 0);
        if (m < N) h = chirp[m];
        else if (L - m < N) h = chirp[L - m];
        if (conj) h.y = -h.y;
        S[m] = h;
    }
}

template <typename T>
__global__ void blue_scale(cx<T>* __restrict__ dst, const cx<T>* __restrict__ S, int L, double s) {
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L; m += gridDim.x * blockDim.x)
        dst[m] = cscale<T>(S[m], (T)s);
}

unsigned grid_for(long long total) {
    long long b = (total + 255) / 256;
    const long long cap = 148LL * 16;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

cudaError_t launch_blue_gather(const BluePass& p, void* S, long long l0, long long cl, bool f32, cudaStream_t st) {
    const unsigned gr = grid_for(cl * p.L);
    if (f32) blue_gather<float><<<gr, 256, 0, st>>>(p, (cx<float>*)S, l0, cl);
    else blue_gather<double><<<gr, 256, 0, st>>>(p, (cx<double>*)S, l0, cl);
    return cudaGetLastError();
}
cudaError_t launch_blue_emit(const BluePass& p, const void* S, long long l0, long long cl, bool f32, cudaStream_t st) {
    const unsigned gr = grid_for(cl * p.n_out);
    if (f32) blue_emit<float><<<gr, 256, 0, st>>>(p, (const cx<float>*)S, l0, cl);
    else blue_emit<double><<<gr, 256, 0, st>>>(p, (const cx<double>*)S, l0, cl);
    return cudaGetLastError();
}
cudaError_t launch_blue_mul(void* S, const void* bhat, long long cl, int L, bool f32, cudaStream_t st) {
    const unsigned gr = grid_for(cl * L);
    if (f32) blue_mul<float><<<gr, 256, 0, st>>>((cx<float>*)S, (const cx<float>*)bhat, cl, L);
    else blue_mul<double><<<gr, 256, 0, st>>>((cx<double>*)S, (const cx<double>*)bhat, cl, L);
    return cudaGetLastError();
}
cudaError_t launch_blue_twiddle(void* S, long long cl, int L1, int L2, int inv, bool f32, cudaStream_t st) {
    const unsigned gr = grid_for(cl * (long long)L1 * L2);
    if (f32) blue_twiddle<float><<<gr, 256, 0, st>>>((cx<float>*)S, cl, L1, L2, inv);
    else blue_twiddle<double><<<gr, 256, 0, st>>>((cx<double>*)S, cl, L1, L2, inv);
    return cudaGetLastError();
}
cudaError_t launch_blue_filter(void* S, const void* chirp, int N, int L, int conj, bool f32, cudaStream_t st) {
    const unsigned gr = grid_for(L);
    if (f32) blue_filter<float><<<gr, 256, 0, st>>>((cx<float>*)S, (const cx<float>*)chirp, N, L, conj);
    else blue_filter<double><<<gr, 256, 0, st>>>((cx<double>*)S, (const cx<double>*)chirp, N, L, conj);
    return cudaGetLastError();
}
cudaError_t launch_blue_scale(void* dst, const void* S, int L, double s, bool f32, cudaStream_t st) {
    const unsigned gr = grid_for(L);
    if (f32) blue_scale<float><<<gr, 256, 0, st>>>((cx<float>*)dst, (const cx<float>*)S, L, s);
    else blue_scale<double><<<gr, 256, 0, st>>>((cx<double>*)dst, (const cx<double>*)S, L, s);
    return cudaGetLastError();
}

}  // namespace fpb
