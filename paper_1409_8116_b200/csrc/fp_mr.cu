// fp_mr.cu -- the mixed-radix line engine: every transform kind at any length
// whose FFT length factors into primes <= 61 (non-power-of-two grids such as
// 1000^3 or 384^3), O(n log n) instead of the dense engine's O(n^2).
//
// Reference behaviour: the same unnormalised scipy transform types as the FFT
// engine and the dense matrices (transforms.py:3-28, _REAL_DISPATCH
// transforms.py:70-77; fftn/ifftn solver.py:239,245).  Recipes (each checked
// against scipy.fft in oracle.mr_transform at odd and even lengths):
//   DCT-II   v = Makhoul reordering of x (v_j = x_2j, v_{n-1-j} = x_{2j+1}, any n),
//            V = FFT_n(v), X_k = 2 Re(w_k V_k), w_k = e^{-i pi k/(2n)}
//   DST-II   reverse(DCT-II(s x)), s_j = (-1)^j
//   DCT-III  W_0 = X_0, W_k = conj(w_k) (X_k - i X_{n-k}); v = unnormalised
//            inverse DFT of W; x_2j = v_j, x_{2j+1} = v_{n-1-j}
//   DST-III  s * DCT-III(reverse(X))
//   DCT-I    Re FFT_{2(n-1)} of the even extension;  DST-I: -Im FFT_{2(n+1)} of
//            the odd extension (shifted by one)
//   real FFT / inverse: complex FFT of the real line / of the Hermitian extension
//
// One CTA (256 threads) owns `lines` complete lines in shared memory (in-place
// passes stay safe).  The FFT is an in-place decimation-in-time transform: the
// loads scatter the line into mixed-radix digit-reversed order (plan table
// `perm`), then stage q (radix R, span L = product of the earlier radices)
// runs butterflies over positions {b L R + k1 + r L}, twiddled by W_{LR}^{r k1}
// from the N-point root table -- every element is touched by exactly one
// butterfly per stage, so one barrier per stage suffices.
#include <cuda_runtime.h>

#include "../../include/fastpoisson_b200.h"
#include "fp_attr.h"
#include "fp_common.cuh"

namespace fpb {

// four reals fetched together (half-length inverse recipes)
template <typename T> struct Quad { struct type { T x, y, z, w; }; };
template <typename T>
__device__ __forceinline__ typename Quad<T>::type make_double4_t(T a, T b, T c, T d) {
    typename Quad<T>::type q;
    q.x = a; q.y = b; q.z = c; q.w = d;
    return q;
}

// Makhoul position of input index j (any n)
__device__ __forceinline__ int mk_pos(int j, int n) { return (j & 1) ? n - 1 - (j >> 1) : (j >> 1); }

template <typename T>
__device__ __forceinline__ cx<T> conj_if(cx<T> w, bool c) { return c ? mkc<T>(w.x, -w.y) : w; }

// odd prime radix R (compile time) or generic (R = 0: runtime r, local arrays)
// cos / sin (2 pi m / R) for the compile-time radices, correctly rounded
__device__ __forceinline__ constexpr double odd_cos(int R, int m) {
    return R == 3 ? -0.5
         : R == 5 ? (m == 1 ? 0.30901699437494742410 : -0.80901699437494742410)
                  : (m == 1 ? 0.62348980185873353053 : m == 2 ? -0.22252093395631440429 : -0.90096886790241912624);
}
__device__ __forceinline__ constexpr double odd_sin(int R, int m) {
    return R == 3 ? 0.86602540378443864676
         : R == 5 ? (m == 1 ? 0.95105651629515357212 : 0.58778525229247312917)
                  : (m == 1 ? 0.78183148246802980871 : m == 2 ? 0.97492791218182360702 : 0.43388373911755812048);
}

template <typename T, int R>
__device__ __forceinline__ void dft_odd(cx<T>* a, const cx<T>* __restrict__ root, int N, bool inv) {
    constexpr int H = (R - 1) / 2;
    T C[H + 1], S[H + 1];
    (void)root;
    (void)N;
#pragma unroll
    for (int m = 1; m <= H; ++m) {
        C[m] = (T)odd_cos(R, m);
        S[m] = inv ? (T)-odd_sin(R, m) : (T)odd_sin(R, m);   // forward: sin; inverse: -sin
    }
    cx<T> p[H + 1], q[H + 1];
    cx<T> x0 = a[0];
#pragma unroll
    for (int j = 1; j <= H; ++j) {
        p[j] = cadd<T>(a[j], a[R - j]);
        q[j] = csub<T>(a[j], a[R - j]);
        x0 = cadd<T>(x0, p[j]);
    }
#pragma unroll
    for (int k = 1; k <= H; ++k) {
        cx<T> A = a[0], B = mkc<T>(0, 0);
#pragma unroll
        for (int j = 1; j <= H; ++j) {
            int m = (j * k) % R;
            const bool neg = m > H;
            if (neg) m = R - m;
            A.x += C[m] * p[j].x;
            A.y += C[m] * p[j].y;
            const T s = neg ? -S[m] : S[m];
            B.x += s * q[j].x;
            B.y += s * q[j].y;
        }
        // sum_j a_j e^{-+2 pi i jk/R} = A - i B  (B carries the sign of the direction)
        a[k] = mkc<T>(A.x + B.y, A.y - B.x);
        a[R - k] = mkc<T>(A.x - B.y, A.y + B.x);
    }
    a[0] = x0;
}

template <typename T>
__device__ void dft_generic(cx<T>* a, int R, const cx<T>* __restrict__ root, int N, bool inv) {
    // runtime odd prime R <= kMrMaxPrime: O(R^2) with the pair symmetry
    const int H = (R - 1) / 2;
    cx<T> p[kMrMaxPrime / 2 + 1], q[kMrMaxPrime / 2 + 1];
    cx<T> x0 = a[0];
    for (int j = 1; j <= H; ++j) {
        p[j] = cadd<T>(a[j], a[R - j]);
        q[j] = csub<T>(a[j], a[R - j]);
        x0 = cadd<T>(x0, p[j]);
    }
    const int st = N / R;
    for (int k = 1; k <= H; ++k) {
        cx<T> A = a[0], B = mkc<T>(0, 0);
        for (int j = 1; j <= H; ++j) {
            const int m = (j * k) % R;
            const cx<T> w = __ldg(&root[m * st]);
            const T s = inv ? w.y : -w.y;
            A.x += w.x * p[j].x;
            A.y += w.x * p[j].y;
            B.x += s * q[j].x;
            B.y += s * q[j].y;
        }
        a[k] = mkc<T>(A.x + B.y, A.y - B.x);
        a[R - k] = mkc<T>(A.x - B.y, A.y + B.x);
    }
    a[0] = x0;
}

template <typename T, int R>
__device__ __forceinline__ void mr_bfly(cx<T>* z, int base, int L, int k1, int step, const cx<T>* __restrict__ root,
                                        int N, bool inv) {
    cx<T> a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = z[P(base + r * L)];
    if (k1 != 0) {
        // one root load, the other powers by multiplication (the engine is LSU-bound,
        // its fp64 pipe mostly idle): w^r = (w^(r/2))^2 or w^(r-1) w
        cx<T> tw[R];
        tw[1] = conj_if<T>(__ldg(&root[k1 * step]), inv);
#pragma unroll
        for (int r = 2; r < R; ++r) tw[r] = (r & 1) ? cmul<T>(tw[r - 1], tw[1]) : cmul<T>(tw[r / 2], tw[r / 2]);
#pragma unroll
        for (int r = 1; r < R; ++r) a[r] = cmul<T>(a[r], tw[r]);
    }
    if constexpr (R == 2 || R == 4 || R == 8 || R == 16) {
        if (inv) dft_reg<R, true, T>(a);
        else dft_reg<R, false, T>(a);
    } else {
        dft_odd<T, R>(a, root, N, inv);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) z[P(base + r * L)] = a[r];
}

template <typename T>
__device__ __noinline__ void mr_bfly_generic(cx<T>* z, int R, int base, int L, int k1, int step,
                                             const cx<T>* __restrict__ root, int N, bool inv) {
    cx<T> a[kMrMaxPrime];
    for (int r = 0; r < R; ++r) a[r] = z[P(base + r * L)];
    if (k1 != 0)
        for (int r = 1; r < R; ++r) a[r] = cmul<T>(a[r], conj_if<T>(__ldg(&root[r * k1 * step]), inv));
    dft_generic<T>(a, R, root, N, inv);
    for (int r = 0; r < R; ++r) z[P(base + r * L)] = a[r];
}

__host__ __device__ inline int mr_line_slots(int N) { return N + (N - 1) / 16 + 1; }

// per-line bookkeeping, staged once per tile (no 64-bit divisions per element):
// global offsets, and for the MID the eigenvalue partial sums (LineInfo, shared
// with the FFT engine's eig_factor)
__host__ __device__ inline size_t mr_tile_bytes(int lines, int N, size_t cb) {
    return ((size_t)lines * mr_line_slots(N) * cb + 15) / 16 * 16;
}
// MID: reals per line of the spectrum buffer (physical spectral order)
__host__ __device__ inline int mr_spec_reals(int kind, int n) {
    if (kind == FP_DFT) return 2 * n;
    if (kind == MR_RFFT) return 2 * (n / 2 + 1);
    return n;
}
__host__ __device__ inline size_t mr_spec_bytes(const MrPass& p, size_t rb) {
    return p.mid ? ((size_t)p.lines * mr_spec_reals(p.kind, p.n) * rb + 15) / 16 * 16 : 0;
}

// element walk of a tile without divisions: lines adjacent in memory (strided
// axis) -> lanes walk across the lines of a row; contiguous lines -> the TPL
// threads of a line walk along it
template <typename F>
__device__ __forceinline__ void mr_walk(bool lminor, int cnt, int logLT, F&& fn) {
    const int tid = threadIdx.x;
    if (lminor) {
        const int l = tid & ((1 << logLT) - 1);
        for (int j = tid >> logLT; j < cnt; j += 256 >> logLT) fn(l, j);
    } else {
        const int logTPL = 8 - logLT;
        const int l = tid >> logTPL;
        for (int j = tid & ((1 << logTPL) - 1); j < cnt; j += 1 << logTPL) fn(l, j);
    }
}

// batched walk: every thread first issues U global loads (fetch), then places
// them (place) -- U loads in flight per thread instead of one (the passes are
// otherwise latency-bound on long_scoreboard at 8-16 resident warps per SM)
template <int U, typename FF, typename FP>
__device__ __forceinline__ void mr_walk_batched(bool lminor, int cnt, int logLT, FF&& fetch, FP&& place) {
    const int tid = threadIdx.x;
    int l, j0, stp;
    if (lminor) { l = tid & ((1 << logLT) - 1); j0 = tid >> logLT; stp = 256 >> logLT; }
    else { const int logTPL = 8 - logLT; l = tid >> logTPL; j0 = tid & ((1 << logTPL) - 1); stp = 1 << logTPL; }
    for (int j = j0; j < cnt; j += U * stp) {
        decltype(fetch(0, 0)) v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int jj = j + u * stp;
            if (jj < cnt) v[u] = fetch(l, jj);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int jj = j + u * stp;
            if (jj < cnt) place(l, jj, v[u]);
        }
    }
}

// one DIT stage of radix R over the line: butterfly bf -> (b, k1) = divmod(bf, L)
// by a float reciprocal (exact: bf < N <= 2^22, margin 0.5 / L)
template <typename T, int R>
__device__ __forceinline__ void mr_stage(cx<T>* z, int L, int N, int tl, int TPL, const cx<T>* __restrict__ root,
                                         bool inv) {
    const int Lq = L * R, step = N / Lq, nbf = N / R;
    const float invL = 1.0f / (float)L;
    for (int bf = tl; bf < nbf; bf += TPL) {
        const int b = __float2int_rz(((float)bf + 0.5f) * invL);
        const int k1 = bf - b * L;
        mr_bfly<T, R>(z, b * Lq + k1, L, k1, step, root, N, inv);
    }
}
template <typename T>
__device__ __forceinline__ void mr_stage_generic(cx<T>* z, int R, int L, int N, int tl, int TPL,
                                                 const cx<T>* __restrict__ root, bool inv) {
    const int Lq = L * R, step = N / Lq, nbf = N / R;
    const float invL = 1.0f / (float)L;
    for (int bf = tl; bf < nbf; bf += TPL) {
        const int b = __float2int_rz(((float)bf + 0.5f) * invL);
        const int k1 = bf - b * L;
        mr_bfly_generic<T>(z, R, b * Lq + k1, L, k1, step, root, N, inv);
    }
}

template <typename T>
struct MrCtx {
    cx<T>* zall;
    int slots, n, N, logLT;
    const int* __restrict__ perm;
    const cx<T>* __restrict__ wq;
    const cx<T>* __restrict__ wt;   // half-length recipes: e^{-2 pi i k/n}, k <= n/2
};

// Half-length recipes for even n (HALF): the real line packed as z_m =
// v_2m + i v_2m+1 (Makhoul order for DCT/DST, natural for the real FFT), one
// complex FFT of length M = n/2, then the real-FFT untangle (rsplit) on the way
// out -- and the inverse: tangle (rmerge), inverse FFT, de-interleave.  Same
// identities as the FFT engine (oracle.makhoul_dct2 / makhoul_dct3); half the
// shared-memory data and FFT work of the full-length recipes.
template <typename T>
__device__ __forceinline__ void put_half(cx<T>* z, const int* __restrict__ perm, int p, T x) {
    reinterpret_cast<T*>(&z[P(__ldg(&perm[p >> 1]))])[p & 1] = x;
}
template <typename T>
__device__ __forceinline__ T get_half(const cx<T>* z, int p) {
    return reinterpret_cast<const T*>(&z[P(p >> 1)])[p & 1];
}

// placement of one line set: input recipe of transform `kind`, values from
// getR(l, j) (real kinds) / getC(l, j) (complex); fetched in batches of U
template <typename T, int U, bool HALF, typename GR, typename GC>
__device__ __forceinline__ void mr_fill(const MrCtx<T>& c, int kind, bool lminor, int nin, GR&& getR, GC&& getC,
                                        bool chk, int& bad) {
    cx<T>* const zall = c.zall;
    const int slots = c.slots, n = c.n, N = c.N;
    const int* __restrict__ perm = c.perm;
    if constexpr (HALF) {
        const int M = n >> 1;
        if (kind == FP_DCT3 || kind == FP_DST3) {
            // Z_k = rmerge(V_k, V_{M-k}, t_k), V_k = conj(w_k)(X'_k - i X'_{n-k}) (V_0 = X'_0);
            // one thread builds the pair (Z_k, Z_{M-k}), k <= M/2
            const bool dst = kind == FP_DST3;
            auto xp = [&](int l, int k) { return getR(l, dst ? n - 1 - k : k); };   // X'_k, k < n
            mr_walk_batched<U>(lminor, M / 2 + 1, c.logLT, [&](int l, int k) {
                // X'_k, X'_{n-k} (0 at k = 0), X'_{M-k}, X'_{M+k}
                return make_double4_t<T>(xp(l, k), k > 0 ? xp(l, n - k) : (T)0, xp(l, M - k), xp(l, M + k));
            }, [&](int l, int k, typename Quad<T>::type q) {
                if (chk && !(finite_t(q.x) && finite_t(q.z))) bad = 1;
                auto V = [&](int kk, T a, T b) -> cx<T> {
                    if (kk == 0) return mkc<T>(a, 0);
                    const cx<T> w = __ldg(&c.wq[kk]);
                    return mkc<T>(w.x * a - w.y * b, -w.y * a - w.x * b);
                };
                const cx<T> vk = V(k, q.x, q.y), vm = V(M - k, q.z, q.w);
                cx<T>* z = zall + l * slots;
                z[P(__ldg(&perm[k]))] = rmerge<T>(vk, vm, __ldg(&c.wt[k]));
                if (k > 0 && 2 * k != M) z[P(__ldg(&perm[M - k]))] = rmerge<T>(vm, vk, __ldg(&c.wt[M - k]));
            });
        } else if (kind == MR_IRFFT) {
            mr_walk_batched<U>(lminor, M / 2 + 1, c.logLT, [&](int l, int k) {
                const cx<T> a = getC(l, k), b = getC(l, M - k);
                return make_double4_t<T>(a.x, a.y, b.x, b.y);
            }, [&](int l, int k, typename Quad<T>::type q) {
                if (chk && !(finite_t(q.x) && finite_t(q.y) && finite_t(q.z) && finite_t(q.w))) bad = 1;
                // the DC / Nyquist imaginary parts do not enter a real inverse (dense kind 101)
                const cx<T> xk = mkc<T>(q.x, k == 0 ? (T)0 : q.y), xm = mkc<T>(q.z, k == 0 ? (T)0 : q.w);
                cx<T>* z = zall + l * slots;
                z[P(__ldg(&perm[k]))] = rmerge<T>(xk, xm, __ldg(&c.wt[k]));
                if (k > 0 && 2 * k != M) z[P(__ldg(&perm[M - k]))] = rmerge<T>(xm, xk, __ldg(&c.wt[M - k]));
            });
        } else if (kind == FP_DCT1 || kind == FP_DST1) {
            // the 2N-point even (DCT-I, n = N + 1) / odd (DST-I, n = N - 1) extension, packed
            const int E = 2 * N;
            mr_walk_batched<U>(lminor, n, c.logLT, [&](int l, int j) { return getR(l, j); }, [&](int l, int j, T x) {
                if (chk && !finite_t(x)) bad = 1;
                cx<T>* z = zall + l * slots;
                if (kind == FP_DCT1) {
                    put_half<T>(z, perm, j, x);
                    if (j >= 1 && j <= N - 1) put_half<T>(z, perm, E - j, x);
                } else {
                    put_half<T>(z, perm, j + 1, x);
                    put_half<T>(z, perm, E - 1 - j, -x);
                    if (j == 0) { put_half<T>(z, perm, 0, (T)0); put_half<T>(z, perm, N, (T)0); }
                }
            });
        } else {
            // DCT-II / DST-II (Makhoul packing) and the real FFT (natural packing)
            mr_walk_batched<U>(lminor, n, c.logLT, [&](int l, int j) { return getR(l, j); }, [&](int l, int j, T x) {
                if (chk && !finite_t(x)) bad = 1;
                cx<T>* z = zall + l * slots;
                if (kind == MR_RFFT) put_half<T>(z, perm, j, x);
                else put_half<T>(z, perm, mk_pos(j, n), (kind == FP_DST2 && (j & 1)) ? -x : x);
            });
        }
        return;
    }
    if (kind == FP_DCT3 || kind == FP_DST3) {
        // W_k = conj(w_k) (X'_k - i X'_{n-k}), X' = X (DCT-III) or reverse(X) (DST-III), X'_n = 0
        const bool dst = kind == FP_DST3;
        mr_walk_batched<U>(lminor, n, c.logLT, [&](int l, int k) {
            const int ja = dst ? n - 1 - k : k, jb = dst ? k - 1 : n - k;
            return mkc<T>(getR(l, ja), k > 0 ? getR(l, jb) : (T)0);
        }, [&](int l, int k, cx<T> ab) {
            const T a = ab.x, b = ab.y;
            if (chk && !finite_t(a)) bad = 1;
            cx<T> W;
            if (k == 0) W = mkc<T>(a, 0);
            else {
                const cx<T> w = __ldg(&c.wq[k]);   // (c, -s): W = (c + i s)(a - i b)
                W = mkc<T>(w.x * a - w.y * b, -w.y * a - w.x * b);
            }
            zall[l * slots + P(__ldg(&perm[k]))] = W;
        });
    } else if (kind == FP_DFT || kind == FP_IDFT || kind == MR_IRFFT) {
        mr_walk_batched<U>(lminor, nin, c.logLT, [&](int l, int j) { return getC(l, j); },
                           [&](int l, int j, cx<T> v) {
            cx<T>* z = zall + l * slots;
            if (chk && !(finite_t(v.x) && finite_t(v.y))) bad = 1;
            z[P(__ldg(&perm[j]))] = v;
            if (kind == MR_IRFFT && j >= 1 && 2 * j < n) z[P(__ldg(&perm[n - j]))] = mkc<T>(v.x, -v.y);
        });
    } else {
        mr_walk_batched<U>(lminor, n, c.logLT, [&](int l, int j) { return getR(l, j); }, [&](int l, int j, T x) {
            cx<T>* z = zall + l * slots;
            if (chk && !finite_t(x)) bad = 1;
            switch (kind) {
                case FP_DCT2: z[P(__ldg(&perm[mk_pos(j, n)]))] = mkc<T>(x, 0); break;
                case FP_DST2: z[P(__ldg(&perm[mk_pos(j, n)]))] = mkc<T>((j & 1) ? -x : x, 0); break;
                case FP_DCT1:
                    z[P(__ldg(&perm[j]))] = mkc<T>(x, 0);
                    if (j >= 1 && j <= n - 2) z[P(__ldg(&perm[N - j]))] = mkc<T>(x, 0);
                    break;
                case FP_DST1:
                    z[P(__ldg(&perm[j + 1]))] = mkc<T>(x, 0);
                    z[P(__ldg(&perm[N - 1 - j]))] = mkc<T>(-x, 0);
                    if (j == 0) {
                        z[P(__ldg(&perm[0]))] = mkc<T>(0, 0);
                        z[P(__ldg(&perm[n + 1]))] = mkc<T>(0, 0);
                    }
                    break;
                default: z[P(__ldg(&perm[j]))] = mkc<T>(x, 0); break;   // real input into RFFT / DFT
            }
        });
    }
}

// output recipe of transform `kind`: putR(l, k, y) / putC(l, k, v) per output
template <typename T, bool HALF, typename PR, typename PC>
__device__ __forceinline__ void mr_emit(const MrCtx<T>& c, int kind, bool lminor, int nout, PR&& putR, PC&& putC) {
    const int slots = c.slots, n = c.n;
    if constexpr (HALF) {
        if (kind == FP_DCT1 || kind == FP_DST1) {
            // real FFT of the extension: V_q = rsplit(Z_q, Z_{N-q}, e^{-2 pi i q/(2N)});
            // DCT-I X_k = Re V_k (k <= N), DST-I X_k = -Im V_{k+1}
            const int N = c.N;
            mr_walk(lminor, nout, c.logLT, [&](int l, int k) {
                const cx<T>* z = c.zall + l * slots;
                const int q = kind == FP_DCT1 ? k : k + 1;
                const cx<T> V = rsplit<T>(z[P(q == N ? 0 : q)], z[P(q == 0 ? 0 : N - q)], __ldg(&c.wt[q]));
                putR(l, k, kind == FP_DCT1 ? V.x : -V.y);
            });
            return;
        }
        const int M = n >> 1;
        if (kind == FP_DCT2 || kind == FP_DST2) {
            // one untangle per pair: U_q = w_q V_q gives X_q = 2 Re U_q and X_{n-q} = -2 Im U_q
            // (DST-II: at the mirrored physical indices)
            const bool dst = kind == FP_DST2;
            mr_walk(lminor, M + 1, c.logLT, [&](int l, int q) {
                const cx<T>* z = c.zall + l * slots;
                const cx<T> V = rsplit<T>(z[P(q == M ? 0 : q)], z[P(q == 0 ? 0 : M - q)], __ldg(&c.wt[q]));
                const cx<T> U = cmul<T>(__ldg(&c.wq[q]), V);
                putR(l, dst ? n - 1 - q : q, (T)2 * U.x);
                if (q >= 1 && q < M) putR(l, dst ? q - 1 : n - q, (T)-2 * U.y);
            });
            return;
        }
        mr_walk(lminor, nout, c.logLT, [&](int l, int k) {
            const cx<T>* z = c.zall + l * slots;
            if (kind == MR_RFFT || kind == FP_DCT2 || kind == FP_DST2) {
                // untangle: V_q = rsplit(Z_q, Z_{M-q}, t_q), q <= M
                int q = k;
                bool hi = false;
                if (kind != MR_RFFT) {
                    const int kk = kind == FP_DST2 ? n - 1 - k : k;
                    hi = kk > M;
                    q = hi ? n - kk : kk;
                }
                const cx<T> V = rsplit<T>(z[P(q == M ? 0 : q)], z[P(q == 0 ? 0 : M - q)], __ldg(&c.wt[q]));
                if (kind == MR_RFFT) { putC(l, k, V); return; }
                const cx<T> U = cmul<T>(__ldg(&c.wq[q]), V);
                putR(l, k, hi ? (T)-2 * U.y : (T)2 * U.x);
                return;
            }
            // inverse kinds: de-interleave (Makhoul order for DCT-III / DST-III)
            T y;
            if (kind == MR_IRFFT) y = get_half<T>(z, k);
            else {
                y = get_half<T>(z, mk_pos(k, n));
                if (kind == FP_DST3 && (k & 1)) y = -y;
            }
            putR(l, k, y);
        });
        return;
    }
    const bool cout = kind == FP_DFT || kind == FP_IDFT || kind == MR_RFFT;
    mr_walk(lminor, nout, c.logLT, [&](int l, int k) {
        const cx<T>* z = c.zall + l * slots;
        if (cout) { putC(l, k, z[P(k)]); return; }
        T y;
        switch (kind) {
            case FP_DCT2: case FP_DST2: {
                const int kk = kind == FP_DST2 ? n - 1 - k : k;
                const cx<T> w = __ldg(&c.wq[kk]), v = z[P(kk)];
                y = (T)2 * (w.x * v.x - w.y * v.y);
                break;
            }
            case FP_DCT3: y = z[P(mk_pos(k, n))].x; break;
            case FP_DST3: y = (k & 1) ? -z[P(mk_pos(k, n))].x : z[P(mk_pos(k, n))].x; break;
            case FP_DST1: y = -z[P(k + 1)].y; break;
            default: y = z[P(k)].x; break;   // DCT-I, inverse real FFT
        }
        putR(l, k, y);
    });
}

template <typename T>
__device__ __forceinline__ void mr_fft(const MrCtx<T>& c, const MrPass& p, bool inv) {
    const int logTPL = 8 - c.logLT, TPL = 1 << logTPL;
    const int tid = threadIdx.x;
    const int li = tid >> logTPL, tl = tid & (TPL - 1);
    cx<T>* z = c.zall + li * c.slots;
    const cx<T>* __restrict__ root = reinterpret_cast<const cx<T>*>(p.root);
    const int N = c.N;
    int L = 1;
    for (int q = 0; q < p.nf; ++q) {
        const int R = p.fac[q];
        switch (R) {
            case 2: mr_stage<T, 2>(z, L, N, tl, TPL, root, inv); break;
            case 3: mr_stage<T, 3>(z, L, N, tl, TPL, root, inv); break;
            case 4: mr_stage<T, 4>(z, L, N, tl, TPL, root, inv); break;
            case 5: mr_stage<T, 5>(z, L, N, tl, TPL, root, inv); break;
            case 7: mr_stage<T, 7>(z, L, N, tl, TPL, root, inv); break;
            case 8: mr_stage<T, 8>(z, L, N, tl, TPL, root, inv); break;
            case 16: mr_stage<T, 16>(z, L, N, tl, TPL, root, inv); break;
            default: mr_stage_generic<T>(z, R, L, N, tl, TPL, root, inv); break;
        }
        L *= R;
        __syncthreads();
    }
}

#ifndef FP_MR_MINB
#define FP_MR_MINB 3   // <= 85 registers: 3 CTAs of 256 threads per SM (500^3 21.8 -> 13.2 ms)
#endif
// One pass: fill (forward or inverse recipe) -> FFT -> emit.  MID (the last
// forward axis): fill(kind) -> FFT -> emit into the spectrum buffer with the
// eigenvalue factor (solver.py:216-223: null capture, bscale / lambda) ->
// fill(ikind) from that buffer -> inverse-direction FFT -> emit(ikind).
// KIND / IKIND: the pass's transform (and, for a MID, its inverse; -1 otherwise)
// as compile-time constants, so every per-element recipe switch folds away;
// operands are plan-typed (the solve casts a foreign-typed rhs first)
template <typename T, int KIND, int IKIND, bool HALF>
__global__ void __launch_bounds__(256, FP_MR_MINB) mr_pass_kernel(const MrPass p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool MID = IKIND >= 0;
    const int N = p.N, n = p.n;
    const int LT = p.lines, logLT = p.log_lines;
    const int tid = threadIdx.x;
    MrCtx<T> c;
    c.zall = reinterpret_cast<cx<T>*>(smem_raw);
    c.slots = mr_line_slots(N);
    c.n = n;
    c.N = N;
    c.logLT = logLT;
    c.perm = p.perm;
    c.wq = reinterpret_cast<const cx<T>*>(p.wq);
    c.wt = reinterpret_cast<const cx<T>*>(p.wt);
    const size_t tb = mr_tile_bytes(LT, N, sizeof(cx<T>));
    T* spec = reinterpret_cast<T*>(smem_raw + tb);
    LineInfo* lines = reinterpret_cast<LineInfo*>(smem_raw + tb + mr_spec_bytes(p, sizeof(T)));
    const Geometry& g = p.g;
    const bool chk = p.nonfinite != nullptr;
    if (tid < LT) {
        const long long nlines = (long long)g.na * g.nb;
        const long long gl = (long long)blockIdx.x * LT + tid;
        LineInfo L{};
        L.valid = gl < nlines;
        const long long ia = L.valid ? gl / g.nb : 0, ib = L.valid ? gl % g.nb : 0;
        L.in_off = ia * g.in_sa + ib * g.in_sb;
        L.out_off = ia * g.out_sa + ib * g.out_sb;
        if (MID) {
            // eigenvalue partial sums in the reference's axis order (eigenvalues.py:104-108)
            const Scaling& Sc = p.s;
            const double la = Sc.lam_a ? Sc.lam_a[ia] : 0.0, lb = Sc.lam_b ? Sc.lam_b[ib] : 0.0;
            double before = 0.0, a1 = 0.0, a2 = 0.0;
            int nafter = 0;
            if (Sc.lam_a && Sc.pos_a < Sc.pos_t) before += la;
            if (Sc.lam_b && Sc.pos_b < Sc.pos_t) before += lb;
            if (Sc.lam_a && Sc.pos_a > Sc.pos_t) { a1 = la; nafter = 1; }
            if (Sc.lam_b && Sc.pos_b > Sc.pos_t) { if (nafter == 0) a1 = lb; else a2 = lb; ++nafter; }
            L.before = before; L.after1 = a1; L.after2 = a2; L.nafter = nafter;
            L.null_line = L.valid && ia == 0 && ib == 0;
        }
        lines[tid] = L;
    }
    __syncthreads();

    // ---- fill from global memory
    int bad = 0;
    const bool lmin_in = g.in_st != 1, lmin_out = g.out_st != 1;
    const T* __restrict__ in_r = reinterpret_cast<const T*>(g.in);
    const cx<T>* __restrict__ in_c = reinterpret_cast<const cx<T>*>(g.in);
    mr_fill<T, 8, HALF>(c, KIND, lmin_in, p.n_in,
        [&](int l, int j) {
            const LineInfo& Ln = lines[l];
            return Ln.valid ? __ldg(in_r + Ln.in_off + (long long)j * g.in_st) : (T)0;
        },
        [&](int l, int j) {
            const LineInfo& Ln = lines[l];
            return Ln.valid ? __ldg(in_c + Ln.in_off + (long long)j * g.in_st) : mkc<T>(0, 0);
        }, chk, bad);
    if (bad) *p.nonfinite = 1;
    __syncthreads();
    mr_fft<T>(c, p, KIND == FP_IDFT || KIND == FP_DCT3 || KIND == FP_DST3 || KIND == MR_IRFFT);

    if constexpr (MID) {
        // ---- spectrum -> scaled spectrum buffer (physical spectral order)
        const int sr = mr_spec_reals(KIND, n);
        const Scaling& Sc = p.s;
        const bool sing = Sc.singular && Sc.dc_out;
        const double cst = Sc.bscale * Sc.inv_np;
        const int nspec = (KIND == FP_DFT) ? n : (KIND == MR_RFFT ? n / 2 + 1 : n);
        mr_emit<T, HALF>(c, KIND, false, nspec,
            [&](int l, int k, T y) {
                const LineInfo& Ln = lines[l];
                if (k == 0 && sing && Ln.null_line) *Sc.dc_out = (double)y;
                spec[l * sr + k] = y * (k == 0 ? eig_factor<T>(Sc, Ln, 0) : eig_factor_nz<T>(Sc, Ln, k, cst));
            },
            [&](int l, int k, cx<T> v) {
                const LineInfo& Ln = lines[l];
                if (k == 0 && sing && Ln.null_line) *Sc.dc_out = (double)v.x;
                const T f = k == 0 ? eig_factor<T>(Sc, Ln, 0) : eig_factor_nz<T>(Sc, Ln, k, cst);
                spec[l * sr + 2 * k] = v.x * f;
                spec[l * sr + 2 * k + 1] = v.y * f;
            });
        __syncthreads();
        // ---- inverse recipe from the spectrum buffer
        constexpr int ik = IKIND;
        mr_fill<T, 1, HALF>(c, ik, false, (ik == MR_IRFFT) ? n / 2 + 1 : n,
            [&](int l, int j) { return spec[l * sr + j]; },
            [&](int l, int j) { return mkc<T>(spec[l * sr + 2 * j], spec[l * sr + 2 * j + 1]); }, false, bad);
        __syncthreads();
        mr_fft<T>(c, p, ik == FP_IDFT || ik == FP_DCT3 || ik == FP_DST3 || ik == MR_IRFFT);
    }

    // ---- store (output recipe of the pass's last transform)
    const T om = (T)p.out_mult;
    T* __restrict__ out_r = reinterpret_cast<T*>(g.out);
    cx<T>* __restrict__ out_c = reinterpret_cast<cx<T>*>(g.out);
    mr_emit<T, HALF>(c, MID ? IKIND : KIND, lmin_out, p.n_out,
        [&](int l, int k, T y) {
            const LineInfo& Ln = lines[l];
            if (Ln.valid) out_r[Ln.out_off + (long long)k * g.out_st] = y * om;
        },
        [&](int l, int k, cx<T> v) {
            const LineInfo& Ln = lines[l];
            if (Ln.valid) out_c[Ln.out_off + (long long)k * g.out_st] = cscale<T>(v, om);
        });
}

size_t mr_smem_bytes(const MrPass& p, bool f32) {
    return mr_tile_bytes(p.lines, p.N, f32 ? 8 : 16) + mr_spec_bytes(p, f32 ? 4 : 8) + (size_t)p.lines * sizeof(LineInfo);
}

using MrKernelFn = void (*)(const MrPass);

template <typename T, bool H>
static MrKernelFn mr_pick_h(int kind, bool mid) {
    if (mid) {
        switch (kind) {
            case FP_DCT2: return mr_pass_kernel<T, FP_DCT2, FP_DCT3, H>;
            case FP_DST2: return mr_pass_kernel<T, FP_DST2, FP_DST3, H>;
            case MR_RFFT: return mr_pass_kernel<T, MR_RFFT, MR_IRFFT, H>;
            case FP_DCT1: return mr_pass_kernel<T, FP_DCT1, FP_DCT1, H>;
            case FP_DST1: return mr_pass_kernel<T, FP_DST1, FP_DST1, H>;
            default: break;
        }
        if constexpr (!H) {
            switch (kind) {
                case FP_DFT: return mr_pass_kernel<T, FP_DFT, FP_IDFT, false>;
                default: break;
            }
        }
        return nullptr;
    }
    switch (kind) {
        case FP_DST2: return mr_pass_kernel<T, FP_DST2, -1, H>;
        case FP_DST3: return mr_pass_kernel<T, FP_DST3, -1, H>;
        case FP_DCT2: return mr_pass_kernel<T, FP_DCT2, -1, H>;
        case FP_DCT3: return mr_pass_kernel<T, FP_DCT3, -1, H>;
        case MR_RFFT: return mr_pass_kernel<T, MR_RFFT, -1, H>;
        case MR_IRFFT: return mr_pass_kernel<T, MR_IRFFT, -1, H>;
        case FP_DST1: return mr_pass_kernel<T, FP_DST1, -1, H>;
        case FP_DCT1: return mr_pass_kernel<T, FP_DCT1, -1, H>;
        default: break;
    }
    if constexpr (!H) {
        switch (kind) {
            case FP_DFT: return mr_pass_kernel<T, FP_DFT, -1, false>;
            case FP_IDFT: return mr_pass_kernel<T, FP_IDFT, -1, false>;
            default: break;
        }
    }
    return nullptr;
}
template <typename T>
static MrKernelFn mr_pick(int kind, bool mid, bool half) {
    return half ? mr_pick_h<T, true>(kind, mid) : mr_pick_h<T, false>(kind, mid);
}

cudaError_t launch_mr_pass(const MrPass& p, bool f32, cudaStream_t st) {
    // operands must be plan-typed: real T, or complex T for the complex-side kinds
    const int rt = f32 ? ET_F32 : ET_F64, ct = f32 ? ET_C64 : ET_C128;
    const bool cin = p.cin != 0;
    const bool cout = p.mid ? p.ikind == FP_IDFT : p.cout != 0;
    if (p.g.in_type != (cin ? ct : rt) || p.g.out_type != (cout ? ct : rt)) return cudaErrorInvalidValue;
    MrKernelFn fn = f32 ? mr_pick<float>(p.kind, p.mid != 0, p.half != 0) : mr_pick<double>(p.kind, p.mid != 0, p.half != 0);
    if (!fn) return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem_attr((const void*)fn);
    if (e != cudaSuccess) return e;
    fn<<<p.tiles, 256, mr_smem_bytes(p, f32), st>>>(p);
    return cudaGetLastError();
}

}  // namespace fpb
