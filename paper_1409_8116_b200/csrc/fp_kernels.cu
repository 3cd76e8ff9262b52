// fp_kernels.cu -- sm_100a kernels of the PoisFFT solve path.
//
// FFT line engine (power-of-two lengths)
//   A CTA owns a TILE of `lines` complete lines of one axis.  The tile is read
//   from HBM once (coalesced: contiguous rows for FAM_CONTIG, W adjacent
//   columns per row for FAM_STRIDED), transformed on chip, and written back
//   once -- one HBM read + one HBM write per element per pass, the algorithmic
//   minimum of SURVEY.md section 8(d).
//
//   Real-to-real and real-to-complex transforms run on a HALF-length complex
//   FFT (M = n/2): DCT-II = Makhoul even/odd reordering + real-FFT untangling
//   + quarter-wave post-twiddle; DST-II = DCT-II of the sign-alternated line,
//   reversed; DCT-III / DST-III / inverse real FFT are the exact inverses of
//   those recipes (identities restated in DESIGN.md).  The
//   complex FFT is a Stockham auto-sort radix-16 (plus one radix-2/4/8 stage)
//   in shared memory; each thread holds 16 complex values in registers per
//   stage; twiddles come from correctly rounded fp64 root tables (no sin/cos on
//   device, no recurrences).
//
//   The MID pass fuses: last forward axis -> null-mode capture -> eigenvalue
//   division -> first inverse axis, on the same on-chip tile
//   (reference: solver.py:216-223, the `work *= self._inv_lam` diagonal).
//   The eigenvalue sum is evaluated per element from the per-axis tables in
//   the reference's summation order (eigenvalues.py:104-108) instead of a dense
//   N-element array (solver.py:149-159), which would cost N*8 extra bytes.
//
// Dense engine: direct summation with a host-built, correctly rounded matrix
//   for every other (kind, n) the reference supports (DST-I, DCT-I, odd n,
//   tiny n).  Tile-exclusive, so in-place safe.
#include <cuda_runtime.h>
#include <stdint.h>
#include "fp_types.h"

namespace fpb {

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
// barriers).  Thread -> (line li, jt); each thread runs 16/R butterflies.
template <int R, bool INV, typename T>
__device__ __forceinline__ void stockham_stage(cx<T>* sm, int ls, int M, int logM, int logNs,
                                               const cx<T>* __restrict__ W, int logTL) {
    constexpr int LOGR = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
    constexpr int NB = 16 / R;
    const int tid = threadIdx.x;
    const int TL = 1 << logTL;
    const int li = tid >> logTL;
    const int jt = tid & (TL - 1);
    const int Ns = 1 << logNs;
    const int strideIn = M >> LOGR;
    cx<T>* line = sm + li * ls;
    cx<T> v[16];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = jt + b * TL;
#pragma unroll
        for (int r = 0; r < R; ++r) v[b * R + r] = line[P(j + r * strideIn)];
        if (logNs > 0) {
            const int e = (j & (Ns - 1)) << (logM - logNs - LOGR);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const cx<T> w = __ldg(&W[(r * e) & (M - 1)]);
                v[b * R + r] = INV ? cmulc<T>(v[b * R + r], w) : cmul<T>(v[b * R + r], w);
            }
        }
        dft_reg<R, INV, T>(v + b * R);
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = jt + b * TL;
        const int base = ((j >> logNs) << (logNs + LOGR)) + (j & (Ns - 1));
#pragma unroll
        for (int r = 0; r < R; ++r) line[P(base + r * Ns)] = v[b * R + r];
    }
    __syncthreads();
}

template <bool INV, typename T>
__device__ __forceinline__ void fft_tile(cx<T>* sm, int ls, int M, int logM,
                                         const cx<T>* __restrict__ W, int logTL) {
    int logNs = 0;
    const int rem = logM & 3;
    if (rem == 1) { stockham_stage<2, INV, T>(sm, ls, M, logM, 0, W, logTL); logNs = 1; }
    else if (rem == 2) { stockham_stage<4, INV, T>(sm, ls, M, logM, 0, W, logTL); logNs = 2; }
    else if (rem == 3) { stockham_stage<8, INV, T>(sm, ls, M, logM, 0, W, logTL); logNs = 3; }
    for (; logNs < logM; logNs += 4) stockham_stage<16, INV, T>(sm, ls, M, logM, logNs, W, logTL);
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
    int nafter, valid, null_line, pad;
};
// the line table is padded so the complex tile behind it is 16-byte aligned
__host__ __device__ __forceinline__ size_t linfo_bytes(int lines) {
    return (sizeof(LineInfo) * (size_t)lines + 15) & ~(size_t)15;
}

// eigenvalue factor for transform-axis index kt on line `L`
template <typename T>
__device__ __forceinline__ T eig_factor(const Scaling& s, const LineInfo& L, int kt) {
    double lam = L.before + __ldg(&s.lam_t[kt]);
    if (L.nafter > 0) lam += L.after1;
    if (L.nafter > 1) lam += L.after2;
    double f = 0.0;
    if (lam != 0.0) f = (s.bscale / lam) * s.inv_np;
    return (T)f;
}

// ----------------------------------------------------------------------------
// the FFT pass kernel
template <typename T>
__global__ void __launch_bounds__(sizeof(T) == 8 ? 512 : 1024) fft_pass_kernel(const FftPass p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw + linfo_bytes(p.lines));

    const int tid = threadIdx.x;
    const int nth = blockDim.x;
    const int Lc = p.lines, logL = p.logLines;
    const int M = p.M, logM = p.logM, n = p.n;
    const int ls = p.ls;
    const int logTL = logM - 4;
    const bool strided = p.family == FAM_STRIDED;
    const cx<T>* __restrict__ W = reinterpret_cast<const cx<T>*>(p.wfft);
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    const Geometry& g = p.g;

    // ---- per-line setup
    if (tid < Lc) {
        LineInfo L;
        int ia, ib;
        bool valid;
        if (!strided) {
            const long long l = (long long)blockIdx.x * Lc + tid;
            valid = l < (long long)g.na * g.nb;
            ia = valid ? (int)(l / g.nb) : 0;
            ib = valid ? (int)(l % g.nb) : 0;
        } else {
            ia = blockIdx.x / p.nbt;
            ib = (blockIdx.x % p.nbt) * Lc + tid;
            valid = ib < g.nb;
            if (!valid) ib = 0;
        }
        L.valid = valid;
        L.in_off = (long long)ia * g.in_sa + (long long)ib * g.in_sb;
        L.out_off = (long long)ia * g.out_sa + (long long)ib * g.out_sb;
        L.null_line = (ia == 0 && ib == 0);
        double before = 0.0, a1 = 0.0, a2 = 0.0;
        int nafter = 0;
        if (p.op == OP_MID) {
            const double la = p.s.lam_a ? p.s.lam_a[ia] : 0.0;
            const double lb = p.s.lam_b ? p.s.lam_b[ib] : 0.0;
            // axes a < b (absent axes have pos -1 and no table)
            const bool ha = p.s.lam_a != nullptr, hb = p.s.lam_b != nullptr;
            if (ha && p.s.pos_a < p.s.pos_t) before += la;
            if (hb && p.s.pos_b < p.s.pos_t) before += lb;
            if (ha && p.s.pos_a > p.s.pos_t) { a1 = la; nafter = 1; }
            if (hb && p.s.pos_b > p.s.pos_t) { if (nafter == 0) a1 = lb; else a2 = lb; ++nafter; }
        }
        L.before = before; L.after1 = a1; L.after2 = a2; L.nafter = nafter; L.pad = 0;
        linfo[tid] = L;
    }
    __syncthreads();

    const bool fwd_in = p.op != OP_INV;
    int nonfinite = 0;

    // =============== LOAD
    if (fwd_in) {
        if (p.fkind == FK_CFFT) {
            const int total = Lc << logM;
            for (int idx = tid; idx < total; idx += nth) {
                int li, k;
                if (strided) { li = idx & (Lc - 1); k = idx >> logL; }
                else { li = idx >> logM; k = idx & (M - 1); }
                const LineInfo& L = linfo[li];
                cx<T> v = mkc<T>(0, 0);
                if (L.valid) {
                    v = ld_cx<T>(g.in, g.in_type, L.in_off + (long long)k * g.in_st);
                    if (p.nonfinite && !(finite_t(v.x) && finite_t(v.y))) nonfinite = 1;
                }
                sm[li * ls + P(k)] = v;
            }
        } else {
            const int kind = p.fkind;
            if (!strided) {
                // pairs (x_j, x_{j+1}), j even: one 16-byte vector load per thread
                const int total = Lc << logM;  // M pairs per line
                for (int idx = tid; idx < total; idx += nth) {
                    const int li = idx >> logM;
                    const int pi = idx & (M - 1);
                    const int j = 2 * pi;
                    const LineInfo& L = linfo[li];
                    T x0 = 0, x1 = 0;
                    if (L.valid) {
                        const long long off = L.in_off + (long long)j * g.in_st;
                        if (p.vec_in) {
                            const cx<T> v = *reinterpret_cast<const cx<T>*>(reinterpret_cast<const T*>(g.in) + off);
                            x0 = v.x; x1 = v.y;
                        } else {
                            x0 = ld_real<T>(g.in, g.in_type, off);
                            x1 = ld_real<T>(g.in, g.in_type, off + g.in_st);
                        }
                        if (p.nonfinite && !(finite_t(x0) && finite_t(x1))) nonfinite = 1;
                    }
                    T* zr = reinterpret_cast<T*>(sm + li * ls);
                    if (kind == FK_RFFT) {
                        cx<T>* z = sm + li * ls;
                        z[P(pi)] = mkc<T>(x0, x1);
                    } else {
                        // Makhoul: v_{j/2} = x_j, v_{n-1-j/2} = x_{j+1}; z_m = v_{2m} + i v_{2m+1}
                        if (kind == FK_DST2) x1 = -x1;
                        const int pa = pi, pb = n - 1 - pi;
                        zr[2 * P(pa >> 1) + (pa & 1)] = x0;
                        zr[2 * P(pb >> 1) + (pb & 1)] = x1;
                    }
                }
            } else {
                const int total = Lc * n;
                for (int idx = tid; idx < total; idx += nth) {
                    const int li = idx & (Lc - 1);
                    const int j = idx >> logL;
                    const LineInfo& L = linfo[li];
                    T x = 0;
                    if (L.valid) {
                        x = ld_real<T>(g.in, g.in_type, L.in_off + (long long)j * g.in_st);
                        if (p.nonfinite && !finite_t(x)) nonfinite = 1;
                    }
                    int pv;
                    if (kind == FK_RFFT) pv = j;
                    else {
                        pv = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
                        if (kind == FK_DST2 && (j & 1)) x = -x;
                    }
                    T* zr = reinterpret_cast<T*>(sm + li * ls);
                    zr[2 * P(pv >> 1) + (pv & 1)] = x;
                }
            }
        }
    } else {
        // inverse: natural-order spectrum
        const int ik = p.ikind;
        if (ik == IK_DCT3 || ik == IK_DST3) {
            const int total = Lc * n;
            for (int idx = tid; idx < total; idx += nth) {
                int li, k;
                if (strided) { li = idx & (Lc - 1); k = idx >> logL; }
                else { li = idx / n; k = idx - li * n; }
                const LineInfo& L = linfo[li];
                T x = 0;
                if (L.valid) {
                    x = ld_real<T>(g.in, g.in_type, L.in_off + (long long)k * g.in_st);
                    if (p.nonfinite && !finite_t(x)) nonfinite = 1;
                }
                const int kk = (ik == IK_DST3) ? (n - 1 - k) : k;
                T* zr = reinterpret_cast<T*>(sm + li * ls);
                zr[PR(kk)] = x;
            }
        } else {
            const int ext = (ik == IK_IRFFT) ? M + 1 : M;
            const int total = Lc * ext;
            for (int idx = tid; idx < total; idx += nth) {
                int li, k;
                if (strided) { li = idx & (Lc - 1); k = idx >> logL; }
                else { li = idx / ext; k = idx - li * ext; }
                const LineInfo& L = linfo[li];
                cx<T> v = mkc<T>(0, 0);
                if (L.valid) {
                    v = ld_cx<T>(g.in, g.in_type, L.in_off + (long long)k * g.in_st);
                    if (p.nonfinite && !(finite_t(v.x) && finite_t(v.y))) nonfinite = 1;
                }
                sm[li * ls + P(k)] = v;
            }
        }
    }
    if (nonfinite) *p.nonfinite = 1;
    __syncthreads();

    const int half = M >> 1;
    const int logHalf = logM - 1;
    const int nItems = Lc << logHalf;  // quads / pairs per tile

    // =============== FORWARD FFT (+ post / mid)
    if (fwd_in) {
        fft_tile<false, T>(sm, ls, M, logM, W, logTL);

        if (p.op == OP_FWD) {
            const int kind = p.fkind;
            const T om = (T)p.out_mult;
            if (kind == FK_CFFT) {
                const int total = Lc << logM;
                for (int idx = tid; idx < total; idx += nth) {
                    int li, k;
                    if (strided) { li = idx & (Lc - 1); k = idx >> logL; }
                    else { li = idx >> logM; k = idx & (M - 1); }
                    const LineInfo& L = linfo[li];
                    if (!L.valid) continue;
                    st_cx<T>(g.out, g.out_type, L.out_off + (long long)k * g.out_st, cscale<T>(sm[li * ls + P(k)], om));
                }
            } else {
                for (int idx = tid; idx < nItems; idx += nth) {
                    int li, q;
                    if (strided) { li = idx & (Lc - 1); q = idx >> logL; }
                    else { li = idx >> logHalf; q = idx & (half - 1); }
                    const LineInfo& L = linfo[li];
                    if (!L.valid) continue;
                    const cx<T>* z = sm + li * ls;
                    const long long ob = L.out_off;
                    const long long os = g.out_st;
                    if (kind == FK_RFFT) {
                        if (q == 0) {
                            const cx<T> z0 = z[P(0)];
                            st_cx<T>(g.out, g.out_type, ob, mkc<T>((z0.x + z0.y) * om, 0));
                            st_cx<T>(g.out, g.out_type, ob + (long long)M * os, mkc<T>((z0.x - z0.y) * om, 0));
                            const cx<T> zh = z[P(half)];
                            st_cx<T>(g.out, g.out_type, ob + (long long)half * os,
                                     cscale<T>(rsplit<T>(zh, zh, Wt[half]), om));
                        } else {
                            const cx<T> zk = z[P(q)], zm = z[P(M - q)];
                            st_cx<T>(g.out, g.out_type, ob + (long long)q * os, cscale<T>(rsplit<T>(zk, zm, Wt[q]), om));
                            st_cx<T>(g.out, g.out_type, ob + (long long)(M - q) * os,
                                     cscale<T>(rsplit<T>(zm, zk, Wt[M - q]), om));
                        }
                    } else {
                        const bool dst = kind == FK_DST2;
#define EMIT(K, X) st_real<T>(g.out, g.out_type, ob + (long long)(dst ? (n - 1 - (K)) : (K)) * os, (X) * om)
                        if (q == 0) {
                            const cx<T> z0 = z[P(0)];
                            const T v0 = z0.x + z0.y, vM = z0.x - z0.y;
                            const cx<T> wM = Ww[M];
                            EMIT(0, (T)2 * v0);
                            EMIT(M, (T)2 * vM * wM.x);
                            const cx<T> zh = z[P(half)];
                            const cx<T> U = cmul<T>(Ww[half], rsplit<T>(zh, zh, Wt[half]));
                            EMIT(half, (T)2 * U.x);
                            EMIT(n - half, (T)-2 * U.y);
                        } else {
                            const cx<T> zk = z[P(q)], zm = z[P(M - q)];
                            const cx<T> U1 = cmul<T>(Ww[q], rsplit<T>(zk, zm, Wt[q]));
                            const cx<T> U2 = cmul<T>(Ww[M - q], rsplit<T>(zm, zk, Wt[M - q]));
                            EMIT(q, (T)2 * U1.x);
                            EMIT(n - q, (T)-2 * U1.y);
                            EMIT(M - q, (T)2 * U2.x);
                            EMIT(M + q, (T)-2 * U2.y);
                        }
#undef EMIT
                    }
                }
            }
            return;
        }

        // ---- OP_MID: post -> capture -> scale -> pre, in place on each quad/pair
        {
            const int kind = p.fkind;
            const Scaling& S = p.s;
            if (kind == FK_CFFT) {
                const int total = Lc << logM;
                for (int idx = tid; idx < total; idx += nth) {
                    const int li = idx >> logM, k = idx & (M - 1);
                    const LineInfo& L = linfo[li];
                    cx<T> X = sm[li * ls + P(k)];
                    if (S.singular && S.dc_out && L.null_line && k == 0 && L.valid) *S.dc_out = (double)X.x;
                    sm[li * ls + P(k)] = cscale<T>(X, eig_factor<T>(S, L, k));
                }
            } else if (kind == FK_RFFT) {
                for (int idx = tid; idx < nItems; idx += nth) {
                    const int li = idx >> logHalf, q = idx & (half - 1);
                    const LineInfo& L = linfo[li];
                    cx<T>* z = sm + li * ls;
                    if (q == 0) {
                        const cx<T> z0 = z[P(0)];
                        T x0 = z0.x + z0.y, xM = z0.x - z0.y;
                        if (S.singular && S.dc_out && L.null_line && L.valid) *S.dc_out = (double)x0;
                        x0 *= eig_factor<T>(S, L, 0);
                        xM *= eig_factor<T>(S, L, M);
                        z[P(0)] = mkc<T>(x0 + xM, x0 - xM);
                        const cx<T> zh = z[P(half)];
                        const cx<T> xh = cscale<T>(rsplit<T>(zh, zh, Wt[half]), eig_factor<T>(S, L, half));
                        z[P(half)] = rmerge<T>(xh, xh, Wt[half]);
                    } else {
                        const cx<T> zk = z[P(q)], zm = z[P(M - q)];
                        const cx<T> tq = Wt[q], tm = Wt[M - q];
                        const cx<T> xk = cscale<T>(rsplit<T>(zk, zm, tq), eig_factor<T>(S, L, q));
                        const cx<T> xm = cscale<T>(rsplit<T>(zm, zk, tm), eig_factor<T>(S, L, M - q));
                        z[P(q)] = rmerge<T>(xk, xm, tq);
                        z[P(M - q)] = rmerge<T>(xm, xk, tm);
                    }
                }
            } else {
                const bool dst = kind == FK_DST2;
#define KPHYS(K) (dst ? (n - 1 - (K)) : (K))
                for (int idx = tid; idx < nItems; idx += nth) {
                    const int li = idx >> logHalf, q = idx & (half - 1);
                    const LineInfo& L = linfo[li];
                    cx<T>* z = sm + li * ls;
                    if (q == 0) {
                        const cx<T> z0 = z[P(0)];
                        const cx<T> wM = Ww[M];
                        T X0 = (T)2 * (z0.x + z0.y);
                        T XM = (T)2 * (z0.x - z0.y) * wM.x;
                        if (S.singular && S.dc_out && L.null_line && L.valid && !dst) *S.dc_out = (double)X0;
                        X0 *= eig_factor<T>(S, L, KPHYS(0));
                        XM *= eig_factor<T>(S, L, KPHYS(M));
                        const cx<T> V0 = mkc<T>(X0, 0);
                        const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                        z[P(0)] = rmerge<T>(V0, VM, mkc<T>(1, 0));
                        const cx<T> zh = z[P(half)];
                        const cx<T> wh = Ww[half], th = Wt[half];
                        const cx<T> U = cmul<T>(wh, rsplit<T>(zh, zh, th));
                        const T Xa = (T)2 * U.x * eig_factor<T>(S, L, KPHYS(half));
                        const T Xb = (T)-2 * U.y * eig_factor<T>(S, L, KPHYS(n - half));
                        const cx<T> Vh = cmulc<T>(mkc<T>(Xa, -Xb), wh);
                        z[P(half)] = rmerge<T>(Vh, Vh, th);
                    } else {
                        const cx<T> zk = z[P(q)], zm = z[P(M - q)];
                        const cx<T> tq = Wt[q], tm = Wt[M - q];
                        const cx<T> wq = Ww[q], wm = Ww[M - q];
                        const cx<T> U1 = cmul<T>(wq, rsplit<T>(zk, zm, tq));
                        const cx<T> U2 = cmul<T>(wm, rsplit<T>(zm, zk, tm));
                        const T Xq = (T)2 * U1.x * eig_factor<T>(S, L, KPHYS(q));
                        const T Xnq = (T)-2 * U1.y * eig_factor<T>(S, L, KPHYS(n - q));
                        const T Xmq = (T)2 * U2.x * eig_factor<T>(S, L, KPHYS(M - q));
                        const T Xpq = (T)-2 * U2.y * eig_factor<T>(S, L, KPHYS(M + q));
                        const cx<T> Vk = cmulc<T>(mkc<T>(Xq, -Xnq), wq);
                        const cx<T> Vm = cmulc<T>(mkc<T>(Xmq, -Xpq), wm);
                        z[P(q)] = rmerge<T>(Vk, Vm, tq);
                        z[P(M - q)] = rmerge<T>(Vm, Vk, tm);
                    }
                }
#undef KPHYS
            }
            __syncthreads();
        }
    } else {
        // =============== INVERSE pre-processing
        const int ik = p.ikind;
        if (ik == IK_DCT3 || ik == IK_DST3) {
            // two-phase: the real-valued view overlaps the complex slots
            // nItems == 8 * nth exactly (threads = lines * M/16), so every
            // thread owns 8 quads and the hold buffer stays in registers
            cx<T> hold[16];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int idx = tid + it * nth;
                const int li = idx >> logHalf, q = idx & (half - 1);
                const T* zr = reinterpret_cast<const T*>(sm + li * ls);
                if (q == 0) {
                    const T X0 = zr[PR(0)], XM = zr[PR(M)];
                    const cx<T> wM = Ww[M];
                    const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                    hold[2 * it] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                    const cx<T> wh = Ww[half], th = Wt[half];
                    const cx<T> Vh = cmulc<T>(mkc<T>(zr[PR(half)], -zr[PR(n - half)]), wh);
                    hold[2 * it + 1] = rmerge<T>(Vh, Vh, th);
                } else {
                    const cx<T> wq = Ww[q], wm = Ww[M - q];
                    const cx<T> tq = Wt[q], tm = Wt[M - q];
                    const cx<T> Vk = cmulc<T>(mkc<T>(zr[PR(q)], -zr[PR(n - q)]), wq);
                    const cx<T> Vm = cmulc<T>(mkc<T>(zr[PR(M - q)], -zr[PR(M + q)]), wm);
                    hold[2 * it] = rmerge<T>(Vk, Vm, tq);
                    hold[2 * it + 1] = rmerge<T>(Vm, Vk, tm);
                }
            }
            __syncthreads();
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int idx = tid + it * nth;
                const int li = idx >> logHalf, q = idx & (half - 1);
                cx<T>* z = sm + li * ls;
                z[P(q)] = hold[2 * it];
                z[P(q == 0 ? half : M - q)] = hold[2 * it + 1];
            }
            __syncthreads();
        } else if (ik == IK_IRFFT) {
            for (int idx = tid; idx < nItems; idx += nth) {
                const int li = idx >> logHalf, q = idx & (half - 1);
                cx<T>* z = sm + li * ls;
                if (q == 0) {
                    const cx<T> x0 = z[P(0)], xM = z[P(M)];
                    z[P(0)] = rmerge<T>(x0, xM, mkc<T>(1, 0));
                    const cx<T> xh = z[P(half)];
                    z[P(half)] = rmerge<T>(xh, xh, Wt[half]);
                } else {
                    const cx<T> xk = z[P(q)], xm = z[P(M - q)];
                    z[P(q)] = rmerge<T>(xk, xm, Wt[q]);
                    z[P(M - q)] = rmerge<T>(xm, xk, Wt[M - q]);
                }
            }
            __syncthreads();
        }
    }

    // =============== INVERSE FFT + store (INV and MID)
    fft_tile<true, T>(sm, ls, M, logM, W, logTL);
    {
        const int ik = p.ikind;
        const T om = (T)p.out_mult;
        if (ik == IK_ICFFT) {
            const int total = Lc << logM;
            for (int idx = tid; idx < total; idx += nth) {
                int li, k;
                if (strided) { li = idx & (Lc - 1); k = idx >> logL; }
                else { li = idx >> logM; k = idx & (M - 1); }
                const LineInfo& L = linfo[li];
                if (!L.valid) continue;
                st_cx<T>(g.out, g.out_type, L.out_off + (long long)k * g.out_st, cscale<T>(sm[li * ls + P(k)], om));
            }
        } else {
            // real output x_j from v / z
            const bool dct = ik != IK_IRFFT;
            const bool dst = ik == IK_DST3;
            if (!strided) {
                const int total = Lc << logM;  // output pairs (x_{2m}, x_{2m+1})
                for (int idx = tid; idx < total; idx += nth) {
                    const int li = idx >> logM, m = idx & (M - 1);
                    const LineInfo& L = linfo[li];
                    if (!L.valid) continue;
                    const T* zr = reinterpret_cast<const T*>(sm + li * ls);
                    T x0, x1;
                    if (dct) {
                        const int pa = m, pb = n - 1 - m;
                        x0 = zr[2 * P(pa >> 1) + (pa & 1)];
                        x1 = zr[2 * P(pb >> 1) + (pb & 1)];
                        if (dst) x1 = -x1;
                    } else {
                        const cx<T> v = sm[li * ls + P(m)];
                        x0 = v.x; x1 = v.y;
                    }
                    x0 *= om; x1 *= om;
                    const long long off = L.out_off + (long long)(2 * m) * g.out_st;
                    if (p.vec_out) {
                        *reinterpret_cast<cx<T>*>(reinterpret_cast<T*>(g.out) + off) = mkc<T>(x0, x1);
                    } else {
                        st_real<T>(g.out, g.out_type, off, x0);
                        st_real<T>(g.out, g.out_type, off + g.out_st, x1);
                    }
                }
            } else {
                const int total = Lc * n;
                for (int idx = tid; idx < total; idx += nth) {
                    const int li = idx & (Lc - 1), j = idx >> logL;
                    const LineInfo& L = linfo[li];
                    if (!L.valid) continue;
                    const T* zr = reinterpret_cast<const T*>(sm + li * ls);
                    int pv;
                    if (dct) pv = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
                    else pv = j;
                    T x = zr[2 * P(pv >> 1) + (pv & 1)];
                    if (dst && (j & 1)) x = -x;
                    st_real<T>(g.out, g.out_type, L.out_off + (long long)j * g.out_st, x * om);
                }
            }
        }
    }
}

// ----------------------------------------------------------------------------
// dense engine: out_k = sum_j mat[k][j] * in_j, one tile of lines per CTA
template <typename T>
__global__ void __launch_bounds__(256) dense_pass_kernel(const DensePass p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    const Geometry& g = p.g;
    const int tid = threadIdx.x, nth = blockDim.x;
    const long long nlines = (long long)g.na * g.nb;
    const long long l0 = (long long)blockIdx.x * p.lines;
    const bool cin = (p.cls == DC_C2C || p.cls == DC_C2R);
    const bool cout = (p.cls == DC_C2C || p.cls == DC_R2C);
    const int nin = p.n_in, nout = p.n_out;
    int nonfinite = 0;
    // load
    for (int idx = tid; idx < p.lines * nin; idx += nth) {
        const int li = idx / nin, j = idx - li * nin;
        const long long l = l0 + li;
        T re = 0, im = 0;
        if (l < nlines) {
            const long long ia = l / g.nb, ib = l % g.nb;
            const long long off = ia * g.in_sa + ib * g.in_sb + (long long)j * g.in_st;
            if (cin) { const cx<T> v = ld_cx<T>(g.in, g.in_type, off); re = v.x; im = v.y; }
            else re = ld_real<T>(g.in, g.in_type, off);
            if (p.nonfinite && !(finite_t(re) && finite_t(im))) nonfinite = 1;
        }
        if (cin) { sm[li * p.in_ls + 2 * j] = re; sm[li * p.in_ls + 2 * j + 1] = im; }
        else sm[li * p.in_ls + j] = re;
    }
    if (nonfinite) *p.nonfinite = 1;
    __syncthreads();
    const T om = (T)p.out_mult;
    for (int idx = tid; idx < p.lines * nout; idx += nth) {
        const int li = idx / nout, k = idx - li * nout;
        const long long l = l0 + li;
        if (l >= nlines) continue;
        const T* x = sm + li * p.in_ls;
        T sr = 0, si = 0;
        if (p.cls == DC_R2R) {
            const T* row = reinterpret_cast<const T*>(p.mat) + (long long)k * nin;
            for (int j = 0; j < nin; ++j) sr += __ldg(&row[j]) * x[j];
        } else {
            const cx<T>* row = reinterpret_cast<const cx<T>*>(p.mat) + (long long)k * nin;
            if (p.cls == DC_R2C) {
                for (int j = 0; j < nin; ++j) { const cx<T> m = __ldg(&row[j]); sr += m.x * x[j]; si += m.y * x[j]; }
            } else if (p.cls == DC_C2C) {
                for (int j = 0; j < nin; ++j) {
                    const cx<T> m = __ldg(&row[j]);
                    const T xr = x[2 * j], xi = x[2 * j + 1];
                    sr += m.x * xr - m.y * xi;
                    si += m.x * xi + m.y * xr;
                }
            } else {  // C2R: Re(sum m_j X_j)
                for (int j = 0; j < nin; ++j) {
                    const cx<T> m = __ldg(&row[j]);
                    sr += m.x * x[2 * j] - m.y * x[2 * j + 1];
                }
            }
        }
        const long long ia = l / g.nb, ib = l % g.nb;
        const long long off = ia * g.out_sa + ib * g.out_sb + (long long)k * g.out_st;
        if (cout) st_cx<T>(g.out, g.out_type, off, mkc<T>(sr * om, si * om));
        else st_real<T>(g.out, g.out_type, off, sr * om);
    }
}

// stand-alone eigenvalue scale (used when the middle axis is on the dense engine)
template <typename T>
__global__ void scale_kernel(const ScalePass p) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    const bool cpx = (p.type == ET_C128 || p.type == ET_C64);
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long k2 = idx % p.ext[2];
        const long long r = idx / p.ext[2];
        const long long k1 = r % p.ext[1];
        const long long k0 = r / p.ext[1];
        const long long ks[3] = {k0, k1, k2};
        double lam = 0.0;
        for (int a = 0; a < p.ndim; ++a) lam += p.lam[a][ks[3 - p.ndim + a]];
        const double f = lam != 0.0 ? (p.bscale / lam) * p.inv_np : 0.0;
        const long long off = k0 * p.st[0] + k1 * p.st[1] + k2 * p.st[2];
        if (cpx) {
            cx<T>* d = reinterpret_cast<cx<T>*>(p.data) + off;
            cx<T> v = *d;
            if (idx == 0 && p.singular && p.dc_out) *p.dc_out = (double)v.x;
            *d = cscale<T>(v, (T)f);
        } else {
            T* d = reinterpret_cast<T*>(p.data) + off;
            if (idx == 0 && p.singular && p.dc_out) *p.dc_out = (double)*d;
            *d = *d * (T)f;
        }
    }
}

// ----------------------------------------------------------------------------
// exact mean removal (solver.py:224-225): needed where the null coefficient is
// not the arithmetic mean (DCT-I / regular Neumann axes).  Deterministic:
// fixed-order block partials -> one-block final sum -> subtract.
template <typename T>
__device__ __forceinline__ long long mean_offset(const MeanPass& p, long long idx) {
    const long long k2 = idx % p.ext[2];
    const long long r = idx / p.ext[2];
    const long long k1 = r % p.ext[1];
    const long long k0 = r / p.ext[1];
    return k0 * p.st[0] + k1 * p.st[1] + k2 * p.st[2];
}

template <typename T>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    return s;
}

template <typename T>
__global__ void __launch_bounds__(256) mean_partial_kernel(const MeanPass p) {
    __shared__ double red[8];
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    const T* d = reinterpret_cast<const T*>(p.data);
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
        acc += (double)d[mean_offset<T>(p, i)];
    const double s = block_sum<T>(acc, red);
    if (threadIdx.x == 0) p.partials[blockIdx.x] = s;
}

template <typename T>
__global__ void __launch_bounds__(256) mean_final_kernel(const MeanPass p, int nparts) {
    __shared__ double red[8];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += p.partials[i];
    const double s = block_sum<T>(acc, red);
    const double total = (double)p.ext[0] * p.ext[1] * p.ext[2];
    if (threadIdx.x == 0) p.partials[nparts] = s / total;
}

template <typename T>
__global__ void __launch_bounds__(256) mean_sub_kernel(const MeanPass p, int nparts) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    T* d = reinterpret_cast<T*>(p.data);
    const T m = (T)p.partials[nparts];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long off = mean_offset<T>(p, i);
        d[off] = d[off] - m;
    }
}

// ----------------------------------------------------------------------------
// launchers (host)
size_t fft_pass_smem_bytes(const FftPass& p, int real_bytes) {
    return linfo_bytes(p.lines) + (size_t)p.lines * p.ls * 2 * real_bytes;
}

static cudaError_t set_smem_attr() {
    static bool done = false;
    if (done) return cudaSuccess;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(fft_pass_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fft_pass_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(dense_pass_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(dense_pass_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
    done = true;
    return cudaSuccess;
}

cudaError_t launch_fft_pass(const FftPass& p, bool f32, cudaStream_t st) {
    cudaError_t e = set_smem_attr();
    if (e != cudaSuccess) return e;
    const int threads = p.lines << (p.logM - 4);
    const size_t smem = fft_pass_smem_bytes(p, f32 ? 4 : 8);
    if (f32) fft_pass_kernel<float><<<p.tiles, threads, smem, st>>>(p);
    else fft_pass_kernel<double><<<p.tiles, threads, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_dense_pass(const DensePass& p, bool f32, cudaStream_t st) {
    cudaError_t e = set_smem_attr();
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)p.lines * p.in_ls * (f32 ? 4 : 8);
    if (f32) dense_pass_kernel<float><<<p.tiles, 256, smem, st>>>(p);
    else dense_pass_kernel<double><<<p.tiles, 256, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_scale_pass(const ScalePass& p, bool f32, cudaStream_t st) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    long long blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    if (f32) scale_kernel<float><<<(int)blocks, 256, 0, st>>>(p);
    else scale_kernel<double><<<(int)blocks, 256, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_mean_pass(const MeanPass& p, bool f32, cudaStream_t st) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    long long blocks = (total + 255) / 256;
    if (blocks > kMeanParts) blocks = kMeanParts;
    if (blocks < 1) blocks = 1;
    const int nb = (int)blocks;
    if (f32) {
        mean_partial_kernel<float><<<nb, 256, 0, st>>>(p);
        mean_final_kernel<float><<<1, 256, 0, st>>>(p, nb);
        mean_sub_kernel<float><<<nb, 256, 0, st>>>(p, nb);
    } else {
        mean_partial_kernel<double><<<nb, 256, 0, st>>>(p);
        mean_final_kernel<double><<<1, 256, 0, st>>>(p, nb);
        mean_sub_kernel<double><<<nb, 256, 0, st>>>(p, nb);
    }
    return cudaGetLastError();
}

}  // namespace fpb
