// fp_common.cuh -- device building blocks shared by the sm_100a kernels:
// complex arithmetic, in-register DFTs, compile-time Stockham stages, the
// real-FFT untangle/tangle, typed loads/stores, per-line tile bookkeeping.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "fp_types.h"

namespace fpb {

// every pass kernel starts here: when launched as a programmatic dependent (fp_attr.h
// launch_pass) it may be resident before the previous pass has finished -- wait for it
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ----------------------------------------------------------------------------
// complex helpers
template <typename T> struct CxOf;
template <> struct CxOf<double> { using type = double2; };
template <> struct CxOf<float> { using type = float2; };
template <typename T> using cx = typename CxOf<T>::type;

template <typename T> __device__ __forceinline__ cx<T> mkc(T a, T b) { cx<T> r; r.x = a; r.y = b; return r; }
template <typename T> __device__ __forceinline__ cx<T> cadd(cx<T> a, cx<T> b) { return mkc<T>(a.x + b.x, a.y + b.y); }
template <typename T> __device__ __forceinline__ cx<T> csub(cx<T> a, cx<T> b) { return mkc<T>(a.x - b.x, a.y - b.y); }
template <typename T> __device__ __forceinline__ cx<T> cmul(cx<T> a, cx<T> b) {
    return mkc<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename T> __device__ __forceinline__ cx<T> cmulc(cx<T> a, cx<T> b) {
    return mkc<T>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename T> __device__ __forceinline__ cx<T> cscale(cx<T> a, T s) { return mkc<T>(a.x * s, a.y * s); }

// padded shared-memory index: one pad slot per 16 complex elements keeps the
// Stockham scatter (stride R) and the column accesses bank-conflict free.
__device__ __forceinline__ int P(int i) { return i + (i >> 4); }
// padded index for the real-valued view used by the DCT-III/DST-III loads
__device__ __forceinline__ int PR(int i) { return i + (i >> 5); }

// ----------------------------------------------------------------------------
// in-register DFT of size R (2,4,8,16), natural order in and out.
// 16th roots of unity, correctly rounded.
__device__ __forceinline__ double c16(int m) {
    switch (m & 15) {
        case 0: return 1.0;
        case 1: return 0.92387953251128673848259;
        case 2: return 0.70710678118654752440084;
        case 3: return 0.38268343236508977172846;
        case 4: return 0.0;
        case 5: return -0.38268343236508977172846;
        case 6: return -0.70710678118654752440084;
        case 7: return -0.92387953251128673848259;
        case 8: return -1.0;
        case 9: return -0.92387953251128673848259;
        case 10: return -0.70710678118654752440084;
        case 11: return -0.38268343236508977172846;
        case 12: return 0.0;
        case 13: return 0.38268343236508977172846;
        case 14: return 0.70710678118654752440084;
        default: return 0.92387953251128673848259;
    }
}
__device__ __forceinline__ double s16(int m) { return c16(m - 4); }  // sin(2 pi m/16)

// multiply by w = e^{-+2 pi i m/16} (forward: minus); m is a compile-time constant after unrolling
template <bool INV, typename T>
__device__ __forceinline__ cx<T> rot16(cx<T> c, int m) {
    if (m == 0) return c;
    if (m == 4) return INV ? mkc<T>(-c.y, c.x) : mkc<T>(c.y, -c.x);
    const T wr = (T)c16(m);
    const T wi = INV ? (T)s16(m) : (T)(-s16(m));
    return mkc<T>(c.x * wr - c.y * wi, c.x * wi + c.y * wr);
}

template <int R> __device__ __forceinline__ constexpr int brev(int i) {
    return R == 2 ? i
         : R == 4 ? (((i & 1) << 1) | ((i >> 1) & 1))
         : R == 8 ? (((i & 1) << 2) | (i & 2) | ((i >> 2) & 1))
                  : (((i & 1) << 3) | ((i & 2) << 1) | ((i >> 1) & 2) | ((i >> 3) & 1));
}

template <int R, bool INV, typename T>
__device__ __forceinline__ void dft_reg(cx<T>* v) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int j = brev<R>(i);
        if (j > i) { cx<T> t = v[i]; v[i] = v[j]; v[j] = t; }
    }
#pragma unroll
    for (int s = 2; s <= R; s *= 2) {
        const int h = s / 2;
#pragma unroll
        for (int k = 0; k < h; ++k) {
            const int m = k * (16 / s);
#pragma unroll
            for (int b = 0; b < R; b += s) {
                const cx<T> a = v[b + k];
                const cx<T> c = rot16<INV, T>(v[b + k + h], m);
                v[b + k] = cadd<T>(a, c);
                v[b + k + h] = csub<T>(a, c);
            }
        }
    }
}

// ----------------------------------------------------------------------------
// one Stockham stage of radix R over every line of the tile (in place, two
// barriers).  Compile-time M, R and Ns: every shared-memory address is the
// thread's base plus a constant.  Thread -> (line, jt); 16/R butterflies each.
template <int R> struct LogR { static constexpr int v = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4; };

// Per-stage twiddle tables: stage (R, Ns) of an M-point FFT multiplies input r
// of butterfly j by W_M^{r (j mod Ns) M/(Ns R)}.  The host stores, for every
// stage with Ns > 1, a table tw[r][e] (r < R, e < Ns) -- r-major, so the lanes
// of a warp (consecutive e) read consecutive entries: coalesced, L1-resident,
// and no fp64 work for the twiddles.  Offsets of the stages are compile-time.
__host__ __device__ constexpr int stage_tw_offset(int logM, int logNs) {
    // stages with Ns > 1 are the radix-16 stages at LOGNS = rem, rem+4, ... (rem = logM & 3),
    // plus LOGNS = 4 when rem == 0; each holds 16 * Ns entries
    int off = 0;
    int l = (logM & 3) ? (logM & 3) : 4;
    while (l < logNs) { off += 16 << l; l += 4; }
    return off;
}
__host__ __device__ constexpr int stage_tw_total(int logM) { return stage_tw_offset(logM, logM); }

// radix-16 stages form 9 of their 15 twiddles as products of two table
// entries (per precision; A/B switches for variant builds)
#ifndef FP_TW2_F32
#define FP_TW2_F32 1
#endif
#ifndef FP_TW2_F64
#define FP_TW2_F64 1
#endif
template <typename T> inline constexpr bool kTwoLevelTwiddles = sizeof(T) == 4 ? FP_TW2_F32 : FP_TW2_F64;

// TWP: radix-16 twiddles from two table loads (w, w^4) and products instead of six
// loads -- for the LSU-bound passes; the fp64-bound real-line MID keeps the loads
template <int R, int LOGNS, bool INV, typename T, int LOGM, bool FROM_REG = false, bool TO_REG = false, bool TWP = false>
__device__ __forceinline__ void stockham_stage(cx<T>* line, int jt, const void* __restrict__ W,
                                               cx<T>* vio = nullptr) {
    // FROM_REG: butterfly inputs come from vio[s] = z[jt + TL s] (the layout the
    //           last radix-16 stage leaves in registers) instead of shared memory
    // TO_REG:   outputs stay in registers: vio[r] = z[jt + TL r] (last stage only)
    constexpr int M = 1 << LOGM;
    constexpr int LOGR = LogR<R>::v;
    constexpr int NB = 16 / R;
    constexpr int TL = M / 16;
    constexpr int NS = 1 << LOGNS;
    constexpr int STRIDE_IN = M >> LOGR;
    cx<T> v[16];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = jt + b * TL;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if constexpr (FROM_REG) v[b * R + r] = vio[b + NB * r];
            else v[b * R + r] = line[P(j + r * STRIDE_IN)];
        }
        if (LOGNS > 0) {
            const cx<T>* tw = reinterpret_cast<const cx<T>*>(W) + stage_tw_offset(LOGM, LOGNS) + (j & (NS - 1));
            if constexpr (R == 16 && kTwoLevelTwiddles<T>) {
                // two-level twiddles: load w^r for r in {1,2,3,4,8,12} and form the
                // other nine as w^(r&3) * w^(r&12) (6 loads instead of 15)
                cx<T> w[16];
                if constexpr (TWP) {
                    w[1] = __ldg(&tw[NS]); w[4] = __ldg(&tw[4 * NS]);
                    w[2] = cmul<T>(w[1], w[1]); w[3] = cmul<T>(w[2], w[1]);
                    w[8] = cmul<T>(w[4], w[4]); w[12] = cmul<T>(w[8], w[4]);
                } else {
                    w[1] = __ldg(&tw[NS]); w[2] = __ldg(&tw[2 * NS]); w[3] = __ldg(&tw[3 * NS]);
                    w[4] = __ldg(&tw[4 * NS]); w[8] = __ldg(&tw[8 * NS]); w[12] = __ldg(&tw[12 * NS]);
                }
#pragma unroll
                for (int h = 4; h < 16; h += 4)
#pragma unroll
                    for (int l = 1; l < 4; ++l) w[h + l] = cmul<T>(w[h], w[l]);
#pragma unroll
                for (int r = 1; r < R; ++r) v[b * R + r] = INV ? cmulc<T>(v[b * R + r], w[r]) : cmul<T>(v[b * R + r], w[r]);
            } else {
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    const cx<T> w = __ldg(&tw[r * NS]);
                    v[b * R + r] = INV ? cmulc<T>(v[b * R + r], w) : cmul<T>(v[b * R + r], w);
                }
            }
        }
        dft_reg<R, INV, T>(v + b * R);
    }
    if constexpr (TO_REG) {
        static_assert(NB == 1 && NS == TL, "only the last radix-16 stage keeps its outputs in registers");
#pragma unroll
        for (int r = 0; r < 16; ++r) vio[r] = v[r];
        return;
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = jt + b * TL;
        const int base = ((j >> LOGNS) << (LOGNS + LOGR)) + (j & (NS - 1));
#pragma unroll
        for (int r = 0; r < R; ++r) line[P(base + r * NS)] = v[b * R + r];
    }
    __syncthreads();
}

template <int LOGNS, bool INV, typename T, int LOGM, bool TWP = false>
__device__ __forceinline__ void radix16_stages(cx<T>* line, int jt, const void* __restrict__ W) {
    if constexpr (LOGNS < LOGM) {
        stockham_stage<16, LOGNS, INV, T, LOGM, false, false, TWP>(line, jt, W);
        radix16_stages<LOGNS + 4, INV, T, LOGM, TWP>(line, jt, W);
    }
}

template <bool INV, typename T, int LOGM, bool TWP = false>
__device__ __forceinline__ void fft_tile(cx<T>* line, int jt, const void* __restrict__ W) {
    constexpr int REM = LOGM & 3;
    if constexpr (REM == 1) stockham_stage<2, 0, INV, T, LOGM>(line, jt, W);
    if constexpr (REM == 2) stockham_stage<4, 0, INV, T, LOGM>(line, jt, W);
    if constexpr (REM == 3) stockham_stage<8, 0, INV, T, LOGM>(line, jt, W);
    radix16_stages<REM, INV, T, LOGM, TWP>(line, jt, W);
}

template <int LOGNS, int LIMIT, bool INV, typename T, int LOGM, bool TWP = false>
__device__ __forceinline__ void radix16_stages_upto(cx<T>* line, int jt, const void* __restrict__ W) {
    if constexpr (LOGNS < LIMIT) {
        stockham_stage<16, LOGNS, INV, T, LOGM, false, false, TWP>(line, jt, W);
        radix16_stages_upto<LOGNS + 4, LIMIT, INV, T, LOGM, TWP>(line, jt, W);
    }
}

// all stages; the last (radix-16, Ns = TL) keeps its outputs in registers:
// v[r] = Z[jt + TL r]
template <bool INV, typename T, int LOGM, bool TWP = false>
__device__ __forceinline__ void fft_tile_to_reg(cx<T>* line, int jt, const void* __restrict__ W, cx<T>* v) {
    constexpr int REM = LOGM & 3;
    if constexpr (REM == 1) stockham_stage<2, 0, INV, T, LOGM>(line, jt, W);
    if constexpr (REM == 2) stockham_stage<4, 0, INV, T, LOGM>(line, jt, W);
    if constexpr (REM == 3) stockham_stage<8, 0, INV, T, LOGM>(line, jt, W);
    constexpr int FIRST16 = REM;
    if constexpr (LOGM - 4 > FIRST16) radix16_stages_upto<FIRST16, LOGM - 4, INV, T, LOGM, TWP>(line, jt, W);
    stockham_stage<16, LOGM - 4, INV, T, LOGM, false, true, TWP>(line, jt, W, v);
}

// all stages; the first takes its inputs from registers v[s] = z[jt + TL s]
template <bool INV, typename T, int LOGM, bool TWP = false>
__device__ __forceinline__ void fft_tile_from_reg(cx<T>* line, int jt, const void* __restrict__ W, cx<T>* v) {
    constexpr int REM = LOGM & 3;
    if constexpr (REM == 1) { stockham_stage<2, 0, INV, T, LOGM, true>(line, jt, W, v); radix16_stages<1, INV, T, LOGM, TWP>(line, jt, W); }
    if constexpr (REM == 2) { stockham_stage<4, 0, INV, T, LOGM, true>(line, jt, W, v); radix16_stages<2, INV, T, LOGM, TWP>(line, jt, W); }
    if constexpr (REM == 3) { stockham_stage<8, 0, INV, T, LOGM, true>(line, jt, W, v); radix16_stages<3, INV, T, LOGM, TWP>(line, jt, W); }
    if constexpr (REM == 0) { stockham_stage<16, 0, INV, T, LOGM, true, false, TWP>(line, jt, W, v); radix16_stages<4, INV, T, LOGM, TWP>(line, jt, W); }
}

// twiddles of the mirrored index M-q from those of q (n = 2M):
//   t_{M-q} = e^{-2 pi i (M-q)/n} = -conj(t_q)
//   w_{M-q} = e^{-i pi (M-q)/(2n)} = e^{-i pi/4} conj(w_q)
template <typename T> __device__ __forceinline__ cx<T> t_mirror(cx<T> t) { return mkc<T>(-t.x, t.y); }
template <typename T> __device__ __forceinline__ cx<T> w_mirror(cx<T> w) {
    const T c = (T)0.70710678118654752440084;
    return mkc<T>(c * (w.x - w.y), -c * (w.x + w.y));
}

// ----------------------------------------------------------------------------
// real-FFT untangle / tangle (half-length trick)
// split: V_k = 1/2 (Z_k + conj Z_{M-k}) - 1/2 i t_k (Z_k - conj Z_{M-k}),  t_k = e^{-2 pi i k/n}
template <typename T>
__device__ __forceinline__ cx<T> rsplit(cx<T> zk, cx<T> zm, cx<T> tk) {
    const cx<T> A = mkc<T>(zk.x + zm.x, zk.y - zm.y);
    const cx<T> B = mkc<T>(zk.x - zm.x, zk.y + zm.y);
    const cx<T> tB = cmul<T>(tk, B);
    return mkc<T>((T)0.5 * (A.x + tB.y), (T)0.5 * (A.y - tB.x));
}
// merge: Z_k = (V_k + conj V_{M-k}) + i conj(t_k) (V_k - conj V_{M-k})
template <typename T>
__device__ __forceinline__ cx<T> rmerge(cx<T> vk, cx<T> vm, cx<T> tk) {
    const cx<T> A = mkc<T>(vk.x + vm.x, vk.y - vm.y);
    const cx<T> B = mkc<T>(vk.x - vm.x, vk.y + vm.y);
    const cx<T> cB = cmulc<T>(B, tk);  // B * conj(t)
    return mkc<T>(A.x - cB.y, A.y + cB.x);
}

// ----------------------------------------------------------------------------
// typed global loads / stores with conversion
template <typename T>
__device__ __forceinline__ T ld_real(const void* p, int type, long long off) {
    if (type == ET_F32) return (T)__ldg(reinterpret_cast<const float*>(p) + off);
    return (T)__ldg(reinterpret_cast<const double*>(p) + off);
}
template <typename T>
__device__ __forceinline__ cx<T> ld_cx(const void* p, int type, long long off) {
    if (type == ET_C64) { const float2 v = __ldg(reinterpret_cast<const float2*>(p) + off); return mkc<T>((T)v.x, (T)v.y); }
    if (type == ET_C128) { const double2 v = __ldg(reinterpret_cast<const double2*>(p) + off); return mkc<T>((T)v.x, (T)v.y); }
    return mkc<T>(ld_real<T>(p, type, off), (T)0);  // real input into a complex transform
}
template <typename T>
__device__ __forceinline__ void st_real(void* p, int type, long long off, T v) {
    if (type == ET_F32) reinterpret_cast<float*>(p)[off] = (float)v;
    else reinterpret_cast<double*>(p)[off] = (double)v;
}
template <typename T>
__device__ __forceinline__ void st_cx(void* p, int type, long long off, cx<T> v) {
    if (type == ET_C64) reinterpret_cast<float2*>(p)[off] = make_float2((float)v.x, (float)v.y);
    else reinterpret_cast<double2*>(p)[off] = make_double2((double)v.x, (double)v.y);
}

template <typename T> __device__ __forceinline__ bool finite_t(T x) { return isfinite(x); }

// per-line bookkeeping of a tile
struct LineInfo {
    long long in_off, out_off;
    double before, after1, after2;  // eigenvalue partial sums (axis order)
    int nafter, valid, null_line, lb;   // lb: global line index along b (rhs producers)
};
// the line table is padded so the complex tile behind it is 16-byte aligned
__host__ __device__ __forceinline__ size_t linfo_bytes(int lines) {
    return (sizeof(LineInfo) * (size_t)lines + 15) & ~(size_t)15;
}

// 1 / x in fp64 from rcp.approx.ftz.f64 (MUFU.RCP64H, 2^-19.9 relative on sm_100a:
// profiles/r02/rcp_probe.txt) and one cubic refinement r (1 + e + e^2), e = 1 - x r:
// error <= 1 ulp over 2^28 samples (two Newton steps: 4 DFMA, correctly rounded; this: 3)
__device__ __forceinline__ double recip_f64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// eigenvalue factor for transform-axis index kt on line `L`
template <typename T>
__device__ __forceinline__ T eig_factor(const Scaling& s, const LineInfo& L, int kt) {
    // absent axes contribute +0.0 (exact), so the adds are unconditional and
    // the sum keeps the reference's axis order ((l0 + l1) + l2)
    const double lam = ((L.before + __ldg(&s.lam_t[kt])) + L.after1) + L.after2;
    // bscale / lam via rcp.approx + a cubic refinement (within 1 ulp of the IEEE
    // quotient of solver.py:158); the null mode (lam == 0) maps to 0
    const double r = recip_f64(lam);
    const double f = lam != 0.0 ? (s.bscale * r) * s.inv_np : 0.0;
    return (T)f;
}

// cst / lam for modes off the null mode (lam < 0 strictly): no select needed
template <typename T>
__device__ __forceinline__ T eig_factor_nz(const Scaling& s, const LineInfo& L, int kt, double cst) {
    // absent axes contribute +0.0 (exact), so the adds are unconditional and
    // the sum keeps the reference's axis order ((l0 + l1) + l2)
    const double lam = ((L.before + __ldg(&s.lam_t[kt])) + L.after1) + L.after2;
    const double r = recip_f64(lam);
    return (T)(cst * r);
}

// ----------------------------------------------------------------------------
// Folded DCT-II / DST-II MID step.  The eigenvalue sum of a line is lam_t[k] + C
// with C = the line's other-axis sum (one add per mode instead of three; the
// reference's axis order only changes the last bit of lam), and the factor is
// 1 / lam -- the constant bscale / prod n_p is applied once at the store.
__device__ __forceinline__ double line_lam_sum(const LineInfo& L) { return L.before + (L.after1 + L.after2); }

template <typename T>
__device__ __forceinline__ T eig_recip_nz(const double* __restrict__ lam_t, int kt, double C) {
    const double lam = __ldg(&lam_t[kt]) + C;
    const double r = recip_f64(lam);
    return (T)r;
}
// the four factors of a folded-MID quad from the pair table: (q, n-q) and (M-q, M+q)
template <typename T>
__device__ __forceinline__ void eig_quad(const double* __restrict__ lam_pair, int q, int M, double C, T& fq, T& fnq,
                                         T& fmq, T& fpq) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(lam_pair) + q);
    const double2 b = __ldg(reinterpret_cast<const double2*>(lam_pair) + (M - q));
    fq = (T)recip_f64(a.x + C);
    fnq = (T)recip_f64(a.y + C);
    fmq = (T)recip_f64(b.x + C);
    fpq = (T)recip_f64(b.y + C);
}
// ... and 0 on the null mode (lam == 0)
template <typename T>
__device__ __forceinline__ T eig_recip(const double* __restrict__ lam_t, int kt, double C) {
    const double lam = __ldg(&lam_t[kt]) + C;
    const double r = recip_f64(lam);
    return lam != 0.0 ? (T)r : (T)0;
}

// One quad {q, n-q, M-q, M+q} (0 < q < M/2) of the DCT-II -> 1/lam -> DCT-III MID
// on the half-length spectrum pair (zk, zm) = (Z_q, Z_{M-q}), in place.  The
// untangle, the quarter-wave post-twiddle, the scale, the DCT-III pre-twiddle and
// the tangle are one real-linear map of (Z_q, Z_{M-q}); with a = w_q, b = w_q t_q
// (w_q = e^{-i pi q/2n}, t_q = e^{-2 pi i q/n}) and c = 1/sqrt 2:
//   E = Z_q + conj Z_{M-q},  O = -i (Z_q - conj Z_{M-q}),  P = a E,  Q = b O
//   P + Q           = 2 w_q V_q           -> (X_q, -X_{n-q})
//   G = (1 - i) conj(P - Q) = 2 w_{M-q} V_{M-q} / c -> (X_{M-q}, -X_{M+q}) / c
//   Y = (U.x f_q, U.y f_{n-q}),  Yg = (G.x f_{M-q}, G.y f_{M+q})
//   H = (1 - i) conj(Yg)   (the inverse's w-twiddle of the mirrored value times 2)
//   Z'_q = conj(a) (Y + H/2) + i conj(b) (Y - H/2),  Z'_{M-q} = conj(conj(a) (Y + H/2) - i conj(b) (Y - H/2))
// 40 flops instead of the 64 of the step-by-step form (rsplit / cmul / scale / cmulc / rmerge);
// identical to it up to rounding.  f* = eigenvalue factors at the PHYSICAL indices.
template <typename T>
__device__ __forceinline__ void mid_quad(cx<T>& zk, cx<T>& zm, cx<T> a, cx<T> b, T fq, T fnq, T fmq, T fpq) {
    const cx<T> E = mkc<T>(zk.x + zm.x, zk.y - zm.y);
    const cx<T> O = mkc<T>(zk.y + zm.y, zm.x - zk.x);
    const cx<T> P = cmul<T>(a, E), Q = cmul<T>(b, O);
    const cx<T> U = cadd<T>(P, Q), D = csub<T>(P, Q);
    const cx<T> Y = mkc<T>(U.x * fq, U.y * fnq);
    const cx<T> Yg = mkc<T>((D.x - D.y) * fmq, -(D.x + D.y) * fpq);
    const cx<T> H = mkc<T>(Yg.x - Yg.y, -(Yg.x + Yg.y));
    const cx<T> Sp = mkc<T>(fma((T)0.5, H.x, Y.x), fma((T)0.5, H.y, Y.y));
    const cx<T> Sm = mkc<T>(fma((T)-0.5, H.x, Y.x), fma((T)-0.5, H.y, Y.y));
    const cx<T> Ep = cmulc<T>(Sp, a), R = cmulc<T>(Sm, b);
    zk = mkc<T>(Ep.x - R.y, Ep.y + R.x);
    zm = mkc<T>(Ep.x + R.y, R.x - Ep.y);
}

}  // namespace fpb
