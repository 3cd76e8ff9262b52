// fp_fft.cuh -- the FFT line-engine pass kernels (see fp_kernels.cu header for
// the algorithm).  Instantiated per (precision, log2 FFT length, family, op) in
// the fp_fft_*.cu translation units, which are compiled in parallel.
//
// fft_pass_kernel: one tile of complete lines per CTA; every thread's global
// loads are issued (into registers) before the first shared-memory store.
// Operands are plan-typed (real T or complex T); strides are arbitrary.
//
// Thread mappings (nth = lines * M/16 threads, TL = M/16):
//   line-major  (FFT stages, MID step):  line = tid / TL, jt = tid % TL
//   I/O mapping (loads/stores):          CONTIG = line-major (lanes walk along a
//     line), STRIDED = column-major (lanes walk across the W adjacent lines so
//     each row segment of W elements is one coalesced access).
#pragma once
#include <cstdlib>
#include <type_traits>

#include "fp_common.cuh"

namespace fpb {

using FftKernelFn = void (*)(const FftPass);

template <int LOGM> struct Shape {
    static constexpr int M = 1 << LOGM;
    static constexpr int LOGTL = LOGM - 4;
    static constexpr int TL = 1 << LOGTL;
    static constexpr int HALF = M / 2;
    static constexpr int LS = ((M + M / 16 + 1) & 1) ? (M + M / 16 + 1) : (M + M / 16 + 2);
};

// shared-memory line stride (complex elements).  With one line per warp
// (TL >= 32) the stride only shapes the strided I/O, so the planner picks it
// per tile (FftPass::ls) to keep those accesses bank-conflict free; otherwise
// it is the compile-time odd stride the multi-line FFT stages need.
template <typename T, int LOGM, bool STRIDED>
__device__ __forceinline__ int line_stride(const FftPass& p) {
    if constexpr (STRIDED && Shape<LOGM>::TL >= 32) return p.ls;
    else return Shape<LOGM>::LS;
}

// The OP template parameter: the pass op in the low 4 bits; a MID specialised
// on its line kind carries kind + 1 above them (0 = kind read at run time from
// FftPass).  One kind per kernel keeps the MID's code small (ncu: c3 MID lost
// ~9 % of its issue slots to instruction-cache misses with all four kinds).
__host__ __device__ constexpr int opb(int op) { return op & 15; }
__host__ __device__ constexpr int opkind(int op) { return (op >> 4) - 1; }
__host__ __device__ constexpr int mid_op(int kind) { return OP_MID | ((kind + 1) << 4); }
// radix-16 twiddle source per pass: products of two loads for the LSU-bound fp64
// passes (c4 11.24 -> 11.11 ms), six loads for the fp64-bound MID of real lines
// (kind-specialised DCT / DST / rFFT: 0.713 -> 0.820 ms with products) and for fp32
// (the products' extra rounding costs the 2048^3 planted-mode check its 1e-5 margin)
// quad post / pre-processing twiddles t_q, w_q (q = jt + TL r) as running products
// of t_jt, w_jt by t_TL, w_TL in the fp64 forward / inverse passes (2 + 2 loads
// instead of 16)
template <typename T, int OP>
inline constexpr bool kTwPowQ = sizeof(T) == 8 && opb(OP) != OP_MID;
template <typename T, bool PROD>
struct QuadTw {
    cx<T> t, w, dt, dw;
    const cx<T>* Wt;
    const cx<T>* Ww;
    __device__ __forceinline__ QuadTw(const cx<T>* wt, const cx<T>* ww, int jt, int TL) : Wt(wt), Ww(ww) {
        if constexpr (PROD) { t = Wt[jt]; w = Ww ? Ww[jt] : mkc<T>(1, 0); dt = Wt[TL]; dw = Ww ? Ww[TL] : mkc<T>(1, 0); }
    }
    // twiddles of q (PROD: the running value for the current r), then step to r + 1
    __device__ __forceinline__ void get(int q, cx<T>& tq, cx<T>& wq) {
        if constexpr (PROD) { tq = t; wq = w; t = cmul<T>(t, dt); w = cmul<T>(w, dw); }
        else { tq = Wt[q]; wq = Ww ? Ww[q] : mkc<T>(1, 0); }
    }
};

template <typename T, int OP>
inline constexpr bool kTwPow = sizeof(T) == 8 && !(opb(OP) == OP_MID && opkind(OP) >= 0 && opkind(OP) != FK_CFFT);

template <int OP>
__device__ __forceinline__ int fkind_of(const FftPass& p) {
    if constexpr (opkind(OP) >= 0) return opkind(OP);
    else return p.fkind;
}
template <int OP>   // forward and inverse kinds of a pair share their enum value
__device__ __forceinline__ int ikind_of(const FftPass& p) {
    if constexpr (opkind(OP) >= 0) return opkind(OP);
    else return p.ikind;
}

// a MID on DCT-II / DST-II lines runs the folded quad step (fp_common.cuh mid_quad):
// its factors are 1 / lam and the constant bscale / prod n_p moves to the store
template <int OP>
__device__ __forceinline__ bool mid_folded(const FftPass& p) {
    return opb(OP) == OP_MID && (fkind_of<OP>(p) == FK_DCT2 || fkind_of<OP>(p) == FK_DST2);
}
template <int OP>
__device__ __forceinline__ double mid_store_scale(const FftPass& p) {
    return mid_folded<OP>(p) ? p.s.bscale * p.s.inv_np : 1.0;
}

// does this (op, kind) read complex lines?
template <int OP>
__device__ __forceinline__ bool complex_input(const FftPass& p) {
    if (opb(OP) == OP_INV) return ikind_of<OP>(p) == IK_ICFFT || ikind_of<OP>(p) == IK_IRFFT;
    return fkind_of<OP>(p) == FK_CFFT;
}

// ----------------------------------------------------------------------------
// per-line bookkeeping of tile `tile` (threads < lines)
template <bool STRIDED, int OP>
__device__ __forceinline__ void setup_lines(const FftPass& p, int tile, LineInfo* linfo) {
    const int tid = threadIdx.x;
    const Geometry& g = p.g;
    if (tid >= p.lines) return;
    LineInfo L;
    int ia, ib;
    bool valid;
    if (!STRIDED) {
        const long long l = (long long)tile * p.lines + tid;
        valid = l < (long long)g.na * g.nb;
        ia = 0;
        ib = 0;
        if (valid) {
            if (l <= 0x7fffffffLL) {   // (a 64-bit divide is ~100 instructions: a third of a one-warp CTA's setup)
                const unsigned lu = (unsigned)l;
                ia = (int)(lu / (unsigned)g.nb);
                ib = (int)(lu - (unsigned)ia * (unsigned)g.nb);
            } else {
                ia = (int)(l / g.nb);
                ib = (int)(l % g.nb);
            }
        }
    } else {
        ia = tile / p.nbt;
        ib = (tile % p.nbt) * p.lines + tid;
        valid = ib < g.nb;
        if (!valid) ib = 0;
    }
    const int part = g.pair_b ? (ib & 1) : 0;           // real view: 0 = real, 1 = imaginary part
    const int ibc = g.pair_b ? (ib >> 1) : ib;
    const int iag = ia + g.a_off, ibg = ibc + g.b_off;   // global line indices
    if ((g.a_lim > 0 && iag >= g.a_lim) || (g.b_lim > 0 && ibg >= g.b_lim)) valid = false;
    L.valid = valid;
    L.in_off = (long long)ia * g.in_sa + (long long)ibc * g.in_sb + part;
    L.out_off = (long long)ia * g.out_sa + (long long)ibc * g.out_sb + part;
    L.null_line = (iag == 0 && ibg == 0 && part == 0);
    double before = 0.0, a1 = 0.0, a2 = 0.0;
    int nafter = 0;
    if (opb(OP) == OP_MID) {
        const bool ha = p.s.lam_a != nullptr, hb = p.s.lam_b != nullptr;
        const double la = (ha && valid) ? p.s.lam_a[iag] : 0.0;
        const double lb = (hb && valid) ? p.s.lam_b[ibg] : 0.0;
        if (ha && p.s.pos_a < p.s.pos_t) before += la;
        if (hb && p.s.pos_b < p.s.pos_t) before += lb;
        if (ha && p.s.pos_a > p.s.pos_t) { a1 = la; nafter = 1; }
        if (hb && p.s.pos_b > p.s.pos_t) { if (nafter == 0) a1 = lb; else a2 = lb; ++nafter; }
    }
    L.before = before; L.after1 = a1; L.after2 = a2; L.nafter = nafter; L.lb = ibg;
    linfo[tid] = L;
}

// ----------------------------------------------------------------------------
// line loads (all of a thread's loads issued before any use; the uniform
// valid / unit-stride conditions are hoisted out of the unrolled loops)
template <typename T, int CNT, int STEP>
__device__ __forceinline__ void load_cx(cx<T>* v, const cx<T>* base, long long st, bool valid, bool unit) {
    if (!valid) {
#pragma unroll
        for (int it = 0; it < CNT; ++it) v[it] = mkc<T>(0, 0);
    } else if (unit) {
#pragma unroll
        for (int it = 0; it < CNT; ++it) v[it] = __ldg(base + it * STEP);
    } else {
        const long long step = (long long)STEP * st;
#pragma unroll
        for (int it = 0; it < CNT; ++it, base += step) v[it] = __ldg(base);
    }
}
template <typename T, int CNT, int STEP>
__device__ __forceinline__ void load_real(T* v, const T* base, long long st, bool valid) {
    if (!valid) {
#pragma unroll
        for (int it = 0; it < CNT; ++it) v[it] = 0;
    } else {
        const long long step = (long long)STEP * st;
#pragma unroll
        for (int it = 0; it < CNT; ++it, base += step) v[it] = __ldg(base);
    }
}
// blocked transform axis (distributed exchange layout): row j at
// (j >> lg) * hi + (j & (2^lg - 1)) * st
// (or, with g.row_tab, at row_tab[j]: uneven slabs / any rank count)
__device__ __forceinline__ bool blocked(const Geometry& g) { return g.blk_lg > 0 || g.row_tab != nullptr; }
__device__ __forceinline__ long long blk_row(const Geometry& g, int j, long long st, long long hi) {
    if (g.row_tab) return __ldg(&g.row_tab[j]);
    const int lg = g.blk_lg, msk = (1 << lg) - 1;
    return (long long)(j >> lg) * hi + (long long)(j & msk) * st;
}
template <typename T, int CNT, int STEP>
__device__ __forceinline__ void load_real_blk(T* v, const T* line, int j0, const Geometry& g, bool valid) {
#pragma unroll
    for (int it = 0; it < CNT; ++it) {
        const int j = j0 + it * STEP;
        v[it] = valid ? __ldg(line + blk_row(g, j, g.in_st, g.in_st_hi)) : (T)0;
    }
}
template <typename T, int CNT, int STEP>
__device__ __forceinline__ void load_cx_blk(cx<T>* v, const cx<T>* line, int j0, const Geometry& g, bool valid) {
#pragma unroll
    for (int it = 0; it < CNT; ++it) {
        const int j = j0 + it * STEP;
        v[it] = valid ? __ldg(line + blk_row(g, j, g.in_st, g.in_st_hi)) : mkc<T>(0, 0);
    }
}

// CONTIG real pairs (x_{2p}, x_{2p+1}), p = bio + TL it
template <typename T, int TL>
__device__ __forceinline__ void load_pairs(cx<T>* v, const T* line, long long st, bool valid, bool vec, int bio) {
    if (!valid) {
#pragma unroll
        for (int it = 0; it < 16; ++it) v[it] = mkc<T>(0, 0);
    } else if (vec) {
        const cx<T>* s = reinterpret_cast<const cx<T>*>(line) + bio;
#pragma unroll
        for (int it = 0; it < 16; ++it) v[it] = __ldg(s + it * TL);
    } else {
        const T* s = line + (long long)(2 * bio) * st;
        const long long step = (long long)(2 * TL) * st;
#pragma unroll
        for (int it = 0; it < 16; ++it, s += step) v[it] = mkc<T>(__ldg(s), __ldg(s + st));
    }
}

// the staggered divergence of a projection step as the line values of the first
// (contiguous, axis-1) pass: pairs (rhs_{2p}, rhs_{2p+1}) of line i = L.lb, p = bio + TL it
template <typename T, int TL>
__device__ __forceinline__ void load_divergence_pairs(cx<T>* v, const Producer& q, const LineInfo& L, int bio) {
    if (!L.valid) {
#pragma unroll
        for (int it = 0; it < 16; ++it) v[it] = mkc<T>(0, 0);
        return;
    }
    const int i = L.lb;
    const int ip = (i + 1 == q.nx) ? 0 : i + 1;
    const T* u0 = reinterpret_cast<const T*>(q.u) + (long long)i * q.us0;
    const T* u1 = reinterpret_cast<const T*>(q.u) + (long long)ip * q.us0;
    const T* w0 = reinterpret_cast<const T*>(q.w) + (long long)i * q.ws0;
    const T sx = (T)q.sx, sz = (T)q.sz;
#pragma unroll
    for (int it = 0; it < 16; ++it) {
        const int j = 2 * (bio + it * TL);
        const int j2 = (q.w_periodic && j + 2 == q.nz) ? 0 : j + 2;
        const T du0 = __ldg(u1 + (long long)j * q.us1) - __ldg(u0 + (long long)j * q.us1);
        const T du1 = __ldg(u1 + (long long)(j + 1) * q.us1) - __ldg(u0 + (long long)(j + 1) * q.us1);
        const T wa = __ldg(w0 + (long long)j * q.ws1), wb = __ldg(w0 + (long long)(j + 1) * q.ws1);
        const T wc = __ldg(w0 + (long long)j2 * q.ws1);
        v[it] = mkc<T>(du0 * sx + (wb - wa) * sz, du1 * sx + (wc - wb) * sz);
    }
}

// ----------------------------------------------------------------------------
// STRIDED tiles: thread (column c, block b) owns the contiguous rows
// j = 32 b + i (real lines, n = 2M rows) or k = 16 b + i (complex, M rows), so
// the W lanes of a warp still read/write 128-byte row segments while every
// padded shared-memory address is a per-thread base plus a compile-time offset:
//   complex k = 16b + i          -> P(k)  = 17 b + i
//   real (half-FFT packing) j    -> 2 P(j >> 1) + (j & 1) = 34 b + i
//   Makhoul v index of j (DCT):  even i = 2m: pv = 16 b + m           -> 16 b + 2 (b >> 1) + m
//                                odd  i = 2m+1: pv = n-1-16b-m         -> base_o - m,
//                                base_o = 16 K - 1 + 2 ((K-1) >> 1), K = n/16 - b
//   PR(k), k = 32 b + i          -> 33 b + i;  PR(n-1-k) -> 33 K' - 2 - i, K' = n/32 - b
struct RowBlk {
    int cpx17, r34, mk_e, mk_o, pr, prr;
    __device__ __forceinline__ RowBlk(int b, int n) {
        cpx17 = 17 * b;
        r34 = 34 * b;
        mk_e = 16 * b + 2 * (b >> 1);
        const int K = n / 16 - b;
        mk_o = 16 * K - 1 + 2 * ((K - 1) >> 1);
        pr = 33 * b;
        prr = 33 * (n / 32 - b) - 2;
    }
    // real-tile index of row j = 32 b + i under the Makhoul reordering
    __device__ __forceinline__ int makhoul(int i) const { return (i & 1) ? (mk_o - (i >> 1)) : (mk_e + (i >> 1)); }
};

// 2 V_k of the real-FFT untangle (same as rsplit2 below; needed earlier in the file)
template <typename T>
__device__ __forceinline__ cx<T> rsplit2_fwd(cx<T> zk, cx<T> zm, cx<T> tk) {
    const cx<T> A = mkc<T>(zk.x + zm.x, zk.y - zm.y);
    const cx<T> B = mkc<T>(zk.x - zm.x, zk.y + zm.y);
    const cx<T> tB = cmul<T>(tk, B);
    return mkc<T>(A.x + tB.y, A.y - tB.x);
}
// ----------------------------------------------------------------------------
// DCT-I / DST-I as a real FFT of length 2M (identities checked against scipy in
// oracle.r1_via_rfft): with z the even extension of x (DCT-I, n = M + 1,
// z_j = x_j for j <= M, x_{2M-j} above) or the odd one (DST-I, n = M - 1, z_0 =
// z_M = 0, z_j = x_{j-1} below M, -x_{2M-j-1} above) and V = rFFT_2M(z):
//   DCT-I X_k = Re V_k (k = 0..M),  DST-I X_{k-1} = -Im V_k (k = 1..M-1);
// the inverse of either is the unnormalised inverse real FFT of the half
// spectrum (X_k, 0) resp. (0, -X_{k-1}), truncated to the n outputs.
template <int OP>
__device__ __forceinline__ bool is_r1(const FftPass& p) {
    return (opb(OP) == OP_INV ? ikind_of<OP>(p) : fkind_of<OP>(p)) >= FK_DCT1;
}
// index of x feeding z_j (always a valid index) and the factor (0, 1 or -1) it enters with
template <int M>
__device__ __forceinline__ int r1_src(bool d1, int j, int* sgn) {
    if (d1) { *sgn = 1; return j <= M ? j : 2 * M - j; }
    if (j == 0 || j == M) { *sgn = 0; return 0; }
    if (j < M) { *sgn = 1; return j - 1; }
    *sgn = -1;
    return 2 * M - j - 1;
}
template <typename T>
__device__ __forceinline__ T r1_apply(T v, int sgn) { return sgn == 0 ? (T)0 : (sgn < 0 ? -v : v); }

// forward outputs of the pair (q, M - q), 0 < q < M/2, from the tile values zk = Z_q, zm = Z_{M-q}
template <typename T, int M>
__device__ __forceinline__ void r1_store_pair(T* pb, long long os, bool d1, int q, cx<T> zk, cx<T> zm, cx<T> tq, T omh) {
    const cx<T> Vq = rsplit2_fwd<T>(zk, zm, tq), Vm = rsplit2_fwd<T>(zm, zk, t_mirror<T>(tq));
    if (d1) {
        pb[(long long)q * os] = Vq.x * omh;
        pb[(long long)(M - q) * os] = Vm.x * omh;
    } else {
        pb[(long long)(q - 1) * os] = -Vq.y * omh;
        pb[(long long)(M - q - 1) * os] = -Vm.y * omh;
    }
}
// ... and of the self-paired entries k = 0, M (from Z_0) and M/2
template <typename T, int M>
__device__ __forceinline__ void r1_store_dc(T* pb, long long os, bool d1, cx<T> z0, cx<T> zh, cx<T> th, T om, T omh) {
    const cx<T> Vh = rsplit2_fwd<T>(zh, zh, th);
    if (d1) {
        pb[0] = (z0.x + z0.y) * om;
        pb[(long long)M * os] = (z0.x - z0.y) * om;
        pb[(long long)(M / 2) * os] = Vh.x * omh;
    } else {
        pb[(long long)(M / 2 - 1) * os] = -Vh.y * omh;
    }
}

// ----------------------------------------------------------------------------
// placement: line values -> padded complex tile in the layout the FFT expects
// (Makhoul reordering / half-length packing for real kinds).  Returns the
// non-finite flag of the values it read.
template <typename T, int LOGM, bool STRIDED, int OP>
__device__ __forceinline__ bool place_tile(const FftPass& p, const LineInfo& Lio, cx<T>* line_io, int bio) {
    using S = Shape<LOGM>;
    constexpr int M = S::M, TL = S::TL;
    constexpr bool fwd_in = opb(OP) != OP_INV;
    constexpr int n = 2 * M;   // real kinds (unused by the complex ones)
    T* zr_io = reinterpret_cast<T*>(line_io);
    bool bad = false;
    const bool chk = p.nonfinite != nullptr;
    const T* rline = reinterpret_cast<const T*>(p.g.in) + Lio.in_off;
    const cx<T>* cline = reinterpret_cast<const cx<T>*>(p.g.in) + Lio.in_off;
    const long long st = p.g.in_st;
    cx<T> v[16];
    if (is_r1<OP>(p)) {
        const bool d1 = (fwd_in ? fkind_of<OP>(p) : ikind_of<OP>(p)) == FK_DCT1;
        if constexpr (fwd_in) {
            // the extension z (2M reals) in the half-FFT packing
            T z[32];
            int sg[32];
            if (!STRIDED) {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int j0 = 2 * (bio + it * TL);
                    const int i0 = r1_src<M>(d1, j0, &sg[2 * it]), i1 = r1_src<M>(d1, j0 + 1, &sg[2 * it + 1]);
                    z[2 * it] = Lio.valid ? __ldg(rline + (long long)i0 * st) : (T)0;
                    z[2 * it + 1] = Lio.valid ? __ldg(rline + (long long)i1 * st) : (T)0;
                }
            } else {
                const bool blk = blocked(p.g);   // distributed MID: the receive layout
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int i0 = r1_src<M>(d1, 32 * bio + it, &sg[it]);
                    const long long o = blk ? blk_row(p.g, i0, st, p.g.in_st_hi) : (long long)i0 * st;
                    z[it] = Lio.valid ? __ldg(rline + o) : (T)0;
                }
            }
            if (chk) {
#pragma unroll
                for (int it = 0; it < 32; ++it) bad |= !finite_t(z[it]);
            }
#pragma unroll
            for (int it = 0; it < 32; ++it) z[it] = r1_apply<T>(z[it], sg[it]);
            if (!STRIDED) {
#pragma unroll
                for (int it = 0; it < 16; ++it) line_io[P(bio + it * TL)] = mkc<T>(z[2 * it], z[2 * it + 1]);
            } else {
                const RowBlk rb(bio, n);
#pragma unroll
                for (int it = 0; it < 32; ++it) zr_io[rb.r34 + it] = z[it];
            }
        } else {
            // the half spectrum (X_k, 0) (DCT-I) or (0, -X_{k-1}) (DST-I), k = 0..M
            T x[16];
            int kk[16];
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                kk[it] = STRIDED ? 16 * bio + it : bio + it * TL;
                const int src = d1 ? kk[it] : (kk[it] == 0 ? 0 : kk[it] - 1);
                x[it] = Lio.valid ? __ldg(rline + (long long)src * st) : (T)0;
            }
            if (chk) {
#pragma unroll
                for (int it = 0; it < 16; ++it) bad |= !finite_t(x[it]);
            }
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                const cx<T> s = d1 ? mkc<T>(x[it], 0) : mkc<T>(0, kk[it] == 0 ? (T)0 : -x[it]);
                if (STRIDED) line_io[17 * bio + it] = s;
                else line_io[P(kk[it])] = s;
            }
            if (bio == 0) {   // k = M: X_M (DCT-I; n = M + 1) or 0 (DST-I)
                T xm = (d1 && Lio.valid) ? __ldg(rline + (long long)M * st) : (T)0;
                if (chk) bad |= !finite_t(xm);
                line_io[P(M)] = mkc<T>(xm, 0);
            }
        }
        return bad && Lio.valid;
    }
    if (fwd_in && fkind_of<OP>(p) != FK_CFFT) {
        const int kind = fkind_of<OP>(p);
        if (!STRIDED) {
            if (p.prod.active) load_divergence_pairs<T, TL>(v, p.prod, Lio, bio);
            else load_pairs<T, TL>(v, rline, st, Lio.valid, p.vec_in, bio);
            if (chk) {
#pragma unroll
                for (int it = 0; it < 16; ++it) bad |= !(finite_t(v[it].x) && finite_t(v[it].y));
            }
            if (kind == FK_RFFT) {
#pragma unroll
                for (int it = 0; it < 16; ++it) line_io[P(bio + it * TL)] = v[it];
            } else {
                // Makhoul: v_pi = x_j, v_{n-1-pi} = x_{j+1} (DST-II: sign-alternated input)
                const T sgn = (kind == FK_DST2) ? (T)-1 : (T)1;
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int pa = bio + it * TL, pb = n - 1 - pa;
                    zr_io[2 * P(pa >> 1) + (pa & 1)] = v[it].x;
                    zr_io[2 * P(pb >> 1) + (pb & 1)] = sgn * v[it].y;
                }
            }
        } else {
            T xr[32];
            if (blocked(p.g)) load_real_blk<T, 32, 1>(xr, rline, 32 * bio, p.g, Lio.valid);
            else load_real<T, 32, 1>(xr, rline + (long long)(32 * bio) * st, st, Lio.valid);
            const RowBlk rb(bio, n);
            if (chk) {
#pragma unroll
                for (int it = 0; it < 32; ++it) bad |= !finite_t(xr[it]);
            }
            if (kind == FK_RFFT) {
#pragma unroll
                for (int it = 0; it < 32; ++it) zr_io[rb.r34 + it] = xr[it];
            } else {
                const T sgn = (kind == FK_DST2) ? (T)-1 : (T)1;
#pragma unroll
                for (int it = 0; it < 32; ++it) zr_io[rb.makhoul(it)] = (it & 1) ? sgn * xr[it] : xr[it];
            }
        }
    } else if (complex_input<OP>(p)) {
        if constexpr (STRIDED) {
            if (blocked(p.g)) load_cx_blk<T, 16, 1>(v, cline, 16 * bio, p.g, Lio.valid);
            else load_cx<T, 16, 1>(v, cline + (long long)(16 * bio) * st, st, Lio.valid, false);
            if (chk) {
#pragma unroll
                for (int it = 0; it < 16; ++it) bad |= !(finite_t(v[it].x) && finite_t(v[it].y));
            }
#pragma unroll
            for (int it = 0; it < 16; ++it) line_io[17 * bio + it] = v[it];
        } else {
            load_cx<T, 16, TL>(v, cline + (long long)bio * st, st, Lio.valid, st == 1);
            if (chk) {
#pragma unroll
                for (int it = 0; it < 16; ++it) bad |= !(finite_t(v[it].x) && finite_t(v[it].y));
            }
#pragma unroll
            for (int it = 0; it < 16; ++it) line_io[P(bio + it * TL)] = v[it];
        }
    } else {
        // DCT-III / DST-III: real spectrum of n = 2M entries
        const bool dst = ikind_of<OP>(p) == IK_DST3;
        if (!STRIDED) {
            load_pairs<T, TL>(v, rline, st, Lio.valid, p.vec_in, bio);
            if (chk) {
#pragma unroll
                for (int it = 0; it < 16; ++it) bad |= !(finite_t(v[it].x) && finite_t(v[it].y));
            }
            if (dst) {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int kk = 2 * (bio + it * TL);
                    zr_io[PR(n - 1 - kk)] = v[it].x;
                    zr_io[PR(n - 2 - kk)] = v[it].y;
                }
            } else {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int kk = 2 * (bio + it * TL);
                    zr_io[PR(kk)] = v[it].x;
                    zr_io[PR(kk + 1)] = v[it].y;
                }
            }
        } else {
            T xr[32];
            load_real<T, 32, 1>(xr, rline + (long long)(32 * bio) * st, st, Lio.valid);
            const RowBlk rb(bio, n);
            if (chk) {
#pragma unroll
                for (int it = 0; it < 32; ++it) bad |= !finite_t(xr[it]);
            }
            if (dst) {
#pragma unroll
                for (int it = 0; it < 32; ++it) zr_io[rb.prr - it] = xr[it];
            } else {
#pragma unroll
                for (int it = 0; it < 32; ++it) zr_io[rb.pr + it] = xr[it];
            }
        }
    }
    return bad && Lio.valid;
}

// the Nyquist entry k = M of an inverse half spectrum always comes from HBM
template <typename T, int LOGM, int OP>
__device__ __forceinline__ bool place_nyquist(const FftPass& p, const LineInfo& Lio, cx<T>* line_io, int bio) {
    constexpr int M = 1 << LOGM;
    if (opb(OP) != OP_INV || ikind_of<OP>(p) != IK_IRFFT || bio != 0) return false;
    cx<T> xm = mkc<T>(0, 0);
    if (Lio.valid) xm = __ldg(reinterpret_cast<const cx<T>*>(p.g.in) + Lio.in_off + (long long)M * p.g.in_st);
    line_io[P(M)] = xm;
    return Lio.valid && p.nonfinite && !(finite_t(xm.x) && finite_t(xm.y));
}

// store of an inverse-transformed tile (natural-order data in shared memory)
template <typename T, int LOGM, bool STRIDED, int OP>
__device__ __forceinline__ void compute_store_tail(const FftPass& p, const LineInfo* linfo, cx<T>* sm, int bio_off = 0,
                                                   double oscale = 1.0) {
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL;
    const int LS = line_stride<T, LOGM, STRIDED>(p);
    constexpr int n = 2 * M;
    const int tid = threadIdx.x;
    const int Lc = p.lines, logL = p.logLines;
    const Geometry& g = p.g;
    const int lio = STRIDED ? (tid & (Lc - 1)) : (tid >> LOGTL);
    const int bio = (STRIDED ? (tid >> logL) : (tid & (TL - 1))) + bio_off;
    cx<T>* line_io = sm + lio * LS;
    const T* zr_io = reinterpret_cast<const T*>(line_io);
    const LineInfo Lio = linfo[lio];
        if (!Lio.valid) return;
        const int ik = ikind_of<OP>(p);
        const T om = (T)(p.out_mult * oscale);
        const long long ob = Lio.out_off;
        const long long os = g.out_st;
        if (STRIDED && blocked(g)) {
            // distributed exchange layout: blocked transform axis
            const long long hi = g.out_st_hi;
            if (ik == IK_ICFFT) {
                cx<T>* pb = reinterpret_cast<cx<T>*>(g.out) + ob;
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int k = bio + it * TL;
                    pb[blk_row(g, k, os, hi)] = cscale<T>(line_io[P(k)], om);
                }
            } else if (ik >= IK_DCT1) {
                // DCT-I keeps z_0..z_M, DST-I z_1..z_{M-1} (shifted down by one)
                const bool d1 = ik == IK_DCT1;
                T* pb = reinterpret_cast<T*>(g.out) + ob;
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int j = bio + it * TL;
                    const T x = zr_io[2 * P(j >> 1) + (j & 1)];
                    if (d1 ? (j <= M) : (j >= 1 && j < M)) pb[blk_row(g, d1 ? j : j - 1, os, hi)] = x * om;
                }
            } else {
                const bool dct = ik == IK_DCT3 || ik == IK_DST3;
                const bool dst = ik == IK_DST3;
                T* pb = reinterpret_cast<T*>(g.out) + ob;
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int j = bio + it * TL;
                    const int pv = dct ? ((j & 1) ? (n - 1 - (j >> 1)) : (j >> 1)) : j;
                    T x = zr_io[2 * P(pv >> 1) + (pv & 1)];
                    if (dst && (j & 1)) x = -x;
                    pb[blk_row(g, j, os, hi)] = x * om;
                }
            }
            return;
        }
        if (ik == IK_ICFFT) {
            if constexpr (STRIDED) {
                cx<T>* po = reinterpret_cast<cx<T>*>(g.out) + ob + (long long)(16 * bio) * os;
#pragma unroll
                for (int it = 0; it < 16; ++it, po += os) *po = cscale<T>(line_io[17 * bio + it], om);
            } else {
                cx<T>* po = reinterpret_cast<cx<T>*>(g.out) + ob + (long long)bio * os;
                const long long step = (long long)TL * os;
#pragma unroll
                for (int it = 0; it < 16; ++it, po += step) *po = cscale<T>(line_io[P(bio + it * TL)], om);
            }
        } else {
            const bool dct = ik == IK_DCT3 || ik == IK_DST3;
            const bool dst = ik == IK_DST3;
            T* const pb = reinterpret_cast<T*>(g.out) + ob;
            if (!STRIDED) {
                // output pairs (x_{2m}, x_{2m+1}), m = bio + TL it
                T xv[32];
                if (dct) {
                    const T sgn = dst ? -om : om;
#pragma unroll
                    for (int it = 0; it < 16; ++it) {
                        const int pa = bio + it * TL, pbv = n - 1 - pa;
                        xv[2 * it] = zr_io[2 * P(pa >> 1) + (pa & 1)] * om;
                        xv[2 * it + 1] = zr_io[2 * P(pbv >> 1) + (pbv & 1)] * sgn;
                    }
                } else {
#pragma unroll
                    for (int it = 0; it < 16; ++it) {
                        const cx<T> v = line_io[P(bio + it * TL)];
                        xv[2 * it] = v.x * om;
                        xv[2 * it + 1] = v.y * om;
                    }
                }
                if (ik >= IK_DCT1) {
                    // DCT-I keeps z_0..z_M, DST-I z_1..z_{M-1} (shifted down by one)
                    const bool d1 = ik == IK_DCT1;
#pragma unroll
                    for (int it = 0; it < 32; ++it) {
                        const int j = 2 * (bio + (it >> 1) * TL) + (it & 1);
                        if (d1 ? (j <= M) : (j >= 1 && j < M)) pb[(long long)(d1 ? j : j - 1) * os] = xv[it];
                    }
                } else if (p.vec_out) {
                    cx<T>* po = reinterpret_cast<cx<T>*>(pb) + bio;
#pragma unroll
                    for (int it = 0; it < 16; ++it) po[it * TL] = mkc<T>(xv[2 * it], xv[2 * it + 1]);
                } else {
                    T* po = pb + (long long)(2 * bio) * os;
                    const long long step = (long long)(2 * TL) * os;
#pragma unroll
                    for (int it = 0; it < 16; ++it, po += step) { po[0] = xv[2 * it]; po[os] = xv[2 * it + 1]; }
                }
            } else {
                T* po = pb + (long long)(32 * bio) * os;
                const RowBlk rb(bio, n);
                if (dct) {
                    const T sgn = dst ? -om : om;   // DST-III: odd outputs negated
#pragma unroll
                    for (int it = 0; it < 32; ++it, po += os) *po = zr_io[rb.makhoul(it)] * ((it & 1) ? sgn : om);
                } else if (ik >= IK_DCT1) {
                    const bool d1 = ik == IK_DCT1;
#pragma unroll
                    for (int it = 0; it < 32; ++it) {
                        const int j = 32 * bio + it;
                        if (d1 ? (j <= M) : (j >= 1 && j < M))
                            pb[(long long)(d1 ? j : j - 1) * os] = zr_io[rb.r34 + it] * om;
                    }
                } else {
#pragma unroll
                    for (int it = 0; it < 32; ++it, po += os) *po = zr_io[rb.r34 + it] * om;
                }
            }
        }
    }

// ----------------------------------------------------------------------------
// Quad / pair helpers.  In every quad loop q = j + TL*it; only it == 0 can give
// q == 0 (the DC / Nyquist / self-paired special case), so that iteration is
// peeled and the seven others run branch-free.

// 2 V_k: the real-FFT untangle without its factor 1/2
template <typename T>
__device__ __forceinline__ cx<T> rsplit2(cx<T> zk, cx<T> zm, cx<T> tk) {
    const cx<T> A = mkc<T>(zk.x + zm.x, zk.y - zm.y);
    const cx<T> B = mkc<T>(zk.x - zm.x, zk.y + zm.y);
    const cx<T> tB = cmul<T>(tk, B);
    return mkc<T>(A.x + tB.y, A.y - tB.x);
}


// STRIDED forward post-processing + store of a transformed tile (natural-order
// spectrum in shared memory): real-FFT untangle / DCT-II quarter-wave twiddle per
// quad, written straight to HBM row by row (I/O mapping: lanes across the columns)
template <typename T, int LOGM, int OP>
__device__ __forceinline__ void fwd_strided_post(const FftPass& p, const LineInfo& Lio, const cx<T>* line_io, int bio) {
    using S = Shape<LOGM>;
    constexpr int M = S::M, HALF = S::HALF;
    constexpr int n = 2 * M;
    const Geometry& g = p.g;
    const int kind = fkind_of<OP>(p);
    const T om = (T)p.out_mult;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    // thread (column, block b) owns quads q = 8 b + i, i < 8 (CFFT: k = 16 b + i):
    //   P(q) = 8 b + (b >> 1) + i;  P(M - q) = 8 K2 - i + (i ? (K2 - 1) >> 1 : K2 >> 1), K2 = M/8 - b
    if (Lio.valid) {
        const long long ob = Lio.out_off;
        const long long os = g.out_st;
        const int b = bio;
        const int pq0 = 8 * b + (b >> 1);
        const int K2 = M / 8 - b;
        const int pm0 = 8 * K2 + (K2 >> 1), pm1 = 8 * K2 + ((K2 - 1) >> 1);
#define PM(I) ((I) == 0 ? pm0 : (pm1 - (I)))
        if (kind == FK_CFFT) {
            cx<T>* po = reinterpret_cast<cx<T>*>(g.out) + ob + (long long)(16 * b) * os;
#pragma unroll
            for (int it = 0; it < 16; ++it, po += os) *po = cscale<T>(line_io[17 * b + it], om);
        } else if (kind == FK_RFFT) {
            cx<T>* const pb = reinterpret_cast<cx<T>*>(g.out) + ob;
            cx<T>* pq = pb + (long long)(8 * b) * os;
            cx<T>* pm = pb + (long long)(M - 8 * b) * os;
            const T omh = om * (T)0.5;
            QuadTw<T, kTwPowQ<T, OP>> qt(Wt, nullptr, 8 * b, 1);   // q = 8b + it: step t_1
#pragma unroll
            for (int it = 0; it < 8; ++it, pq += os, pm -= os) {
                const int q = 8 * b + it;
                cx<T> tq, wq_unused;
                qt.get(q, tq, wq_unused);
                if (it == 0 && b == 0) {
                    const cx<T> z0 = line_io[P(0)];
                    pb[0] = mkc<T>((z0.x + z0.y) * om, 0);
                    pb[(long long)M * os] = mkc<T>((z0.x - z0.y) * om, 0);
                    const cx<T> zh = line_io[P(HALF)];
                    pb[(long long)HALF * os] = cscale<T>(rsplit2<T>(zh, zh, Wt[HALF]), omh);
                } else {
                    const cx<T> zk = line_io[pq0 + it], zm = line_io[PM(it)];
                    *pq = cscale<T>(rsplit2<T>(zk, zm, tq), omh);
                    *pm = cscale<T>(rsplit2<T>(zm, zk, t_mirror<T>(tq)), omh);
                }
            }
        } else if (kind >= FK_DCT1) {
            const bool d1 = kind == FK_DCT1;
            T* const pb = reinterpret_cast<T*>(g.out) + ob;
            const T omh = om * (T)0.5;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int q = 8 * b + it;
                if (it == 0 && b == 0)
                    r1_store_dc<T, M>(pb, os, d1, line_io[P(0)], line_io[P(HALF)], Wt[HALF], om, omh);
                else
                    r1_store_pair<T, M>(pb, os, d1, q, line_io[pq0 + it], line_io[PM(it)], Wt[q], omh);
            }
        } else {
            const bool dst = kind == FK_DST2;
            T* const pb = reinterpret_cast<T*>(g.out) + ob;
            const long long s1 = dst ? -os : os;
            T* const p0 = dst ? pb + (long long)(n - 1) * os : pb;
            T* pa = p0 + (long long)(8 * b) * s1;
            T* pn = p0 + (long long)(n - 8 * b) * s1;
            T* pm = p0 + (long long)(M - 8 * b) * s1;
            T* pp = p0 + (long long)(M + 8 * b) * s1;
            QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, 8 * b, 1);   // q = 8b + it: steps t_1, w_1
#pragma unroll
            for (int it = 0; it < 8; ++it, pa += s1, pn -= s1, pm -= s1, pp += s1) {
                const int q = 8 * b + it;
                cx<T> tq, wq;
                qt.get(q, tq, wq);
                if (it == 0 && b == 0) {
                    const cx<T> z0 = line_io[P(0)];
                    const cx<T> wM = Ww[M];
                    p0[0] = (T)2 * (z0.x + z0.y) * om;
                    p0[(long long)M * s1] = (T)2 * (z0.x - z0.y) * wM.x * om;
                    const cx<T> zh = line_io[P(HALF)];
                    const cx<T> U = cmul<T>(Ww[HALF], rsplit2<T>(zh, zh, Wt[HALF]));
                    p0[(long long)HALF * s1] = U.x * om;
                    p0[(long long)(n - HALF) * s1] = -U.y * om;
                } else {
                    const cx<T> zk = line_io[pq0 + it], zm = line_io[PM(it)];
                    const cx<T> U1 = cmul<T>(wq, rsplit2<T>(zk, zm, tq));
                    const cx<T> U2 = cmul<T>(w_mirror<T>(wq), rsplit2<T>(zm, zk, t_mirror<T>(tq)));
                    *pa = U1.x * om;
                    *pn = -U1.y * om;
                    *pm = U2.x * om;
                    *pp = -U2.y * om;
                }
            }
        }
#undef PM
    }
}

// ----------------------------------------------------------------------------
// transform + post/mid/pre + store of one placed tile (contains barriers;
// every thread of the CTA must call it).
template <typename T, int LOGM, bool STRIDED, int OP>
__device__ __forceinline__ void compute_store(const FftPass& p, const LineInfo* linfo, cx<T>* sm) {
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL, HALF = S::HALF;
    const int LS = line_stride<T, LOGM, STRIDED>(p);
    constexpr bool fwd_in = opb(OP) != OP_INV;
    const int tid = threadIdx.x;
    const int Lc = p.lines, logL = p.logLines;
    constexpr int n = 2 * M;   // real kinds (unused by the complex ones)
    const void* __restrict__ W = p.wfft;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    const Geometry& g = p.g;
    const int lf = tid >> LOGTL;
    const int jt = tid & (TL - 1);
    const int lio = STRIDED ? (tid & (Lc - 1)) : lf;
    const int bio = STRIDED ? (tid >> logL) : jt;
    cx<T>* line_f = sm + lf * LS;
    cx<T>* line_io = sm + lio * LS;
    const T* zr_io = reinterpret_cast<const T*>(line_io);
    const LineInfo Lio = linfo[lio];

    if constexpr (opb(OP) == OP_MID) {
        if (fkind_of<OP>(p) == FK_CFFT) {
            // complex lines: the eigenvalue divide is pointwise, so the forward FFT
            // ends in registers (v[r] = Z[jt + TL r]), is scaled there, and the
            // inverse FFT starts from them -- two shared-memory round trips fewer
            const Scaling& Sc = p.s;
            const LineInfo L = linfo[lf];
            const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
            const double cst = Sc.bscale * Sc.inv_np;
            cx<T> v[16];
            fft_tile_to_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
            if (jt == 0) {
                if (cap) *Sc.dc_out = (double)v[0].x;
                v[0] = cscale<T>(v[0], eig_factor<T>(Sc, L, 0));
            } else {
                v[0] = cscale<T>(v[0], eig_factor_nz<T>(Sc, L, jt, cst));
            }
#pragma unroll
            for (int it = 1; it < 16; ++it) v[it] = cscale<T>(v[it], eig_factor_nz<T>(Sc, L, jt + it * TL, cst));
            fft_tile_from_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
            compute_store_tail<T, LOGM, STRIDED, OP>(p, linfo, sm);
            return;
        }
    }

    if constexpr (fwd_in) {
        fft_tile<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W);

        if constexpr (opb(OP) == OP_FWD) {
            const int kind = fkind_of<OP>(p);
            const T om = (T)p.out_mult;
            if constexpr (STRIDED) {
                fwd_strided_post<T, LOGM, OP>(p, Lio, line_io, bio);
                return;
            }
            if (Lio.valid) {
                const long long ob = Lio.out_off;
                const long long os = g.out_st;
                if (kind == FK_CFFT) {
                    cx<T>* po = reinterpret_cast<cx<T>*>(g.out) + ob + (long long)bio * os;
                    const long long step = (long long)TL * os;
#pragma unroll
                    for (int it = 0; it < 16; ++it, po += step) *po = cscale<T>(line_io[P(bio + it * TL)], om);
                } else if (kind == FK_RFFT) {
                    cx<T>* const pb = reinterpret_cast<cx<T>*>(g.out) + ob;
                    cx<T>* pq = pb + (long long)bio * os;
                    cx<T>* pm = pb + (long long)(M - bio) * os;
                    const long long step = (long long)TL * os;
                    const T omh = om * (T)0.5;
                    auto pair = [&](int q) {
                        const cx<T> zk = line_io[P(q)], zm = line_io[P(M - q)];
                        const cx<T> tq = Wt[q];
                        *pq = cscale<T>(rsplit2<T>(zk, zm, tq), omh);
                        *pm = cscale<T>(rsplit2<T>(zm, zk, t_mirror<T>(tq)), omh);
                    };
                    if (bio == 0) {
                        const cx<T> z0 = line_io[P(0)];
                        pb[0] = mkc<T>((z0.x + z0.y) * om, 0);
                        pb[(long long)M * os] = mkc<T>((z0.x - z0.y) * om, 0);
                        const cx<T> zh = line_io[P(HALF)];
                        pb[(long long)HALF * os] = cscale<T>(rsplit2<T>(zh, zh, Wt[HALF]), omh);
                    } else {
                        pair(bio);
                    }
                    pq += step; pm -= step;
#pragma unroll
                    for (int it = 1; it < 8; ++it, pq += step, pm -= step) pair(bio + it * TL);
                } else if (kind >= FK_DCT1) {
                    const bool d1 = kind == FK_DCT1;
                    T* const pb = reinterpret_cast<T*>(g.out) + ob;
                    const T omh = om * (T)0.5;
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int q = bio + it * TL;
                        if (it == 0 && bio == 0)
                            r1_store_dc<T, M>(pb, os, d1, line_io[P(0)], line_io[P(HALF)], Wt[HALF], om, omh);
                        else
                            r1_store_pair<T, M>(pb, os, d1, q, line_io[P(q)], line_io[P(M - q)], Wt[q], omh);
                    }
                } else {
                    // DCT-II quads {q, n-q, M-q, M+q} (DST-II: mirrored indices)
                    const bool dst = kind == FK_DST2;
                    T* const pb = reinterpret_cast<T*>(g.out) + ob;
                    const long long s1 = dst ? -os : os;                      // direction of index k
                    T* const p0 = dst ? pb + (long long)(n - 1) * os : pb;   // address of k = 0
                    T* pa = p0 + (long long)bio * s1;             // k = q
                    T* pn = p0 + (long long)(n - bio) * s1;       // k = n - q
                    T* pm = p0 + (long long)(M - bio) * s1;       // k = M - q
                    T* pp = p0 + (long long)(M + bio) * s1;       // k = M + q
                    const long long step = (long long)TL * s1;
                    QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, bio, TL);   // q = bio + TL it, ascending
                    auto quad = [&](int q) {
                        const cx<T> zk = line_io[P(q)], zm = line_io[P(M - q)];
                        cx<T> tq, wq;
                        qt.get(q, tq, wq);
                        const cx<T> U1 = cmul<T>(wq, rsplit2<T>(zk, zm, tq));        // X_q = Re, X_{n-q} = -Im
                        const cx<T> U2 = cmul<T>(w_mirror<T>(wq), rsplit2<T>(zm, zk, t_mirror<T>(tq)));
                        *pa = U1.x * om;
                        *pn = -U1.y * om;
                        *pm = U2.x * om;
                        *pp = -U2.y * om;
                    };
                    if (bio == 0) {
                        const cx<T> z0 = line_io[P(0)];
                        const cx<T> wM = Ww[M];
                        p0[0] = (T)2 * (z0.x + z0.y) * om;
                        p0[(long long)M * s1] = (T)2 * (z0.x - z0.y) * wM.x * om;
                        const cx<T> zh = line_io[P(HALF)];
                        const cx<T> U = cmul<T>(Ww[HALF], rsplit2<T>(zh, zh, Wt[HALF]));
                        p0[(long long)HALF * s1] = U.x * om;
                        p0[(long long)(n - HALF) * s1] = -U.y * om;
                        cx<T> t0, w0;
                        qt.get(0, t0, w0);   // keep the running twiddles in step
                    } else {
                        quad(bio);
                    }
                    pa += step; pn -= step; pm -= step; pp += step;
#pragma unroll
                    for (int it = 1; it < 8; ++it, pa += step, pn -= step, pm -= step, pp += step) quad(bio + it * TL);
                }
            }
            return;
        } else {
            // ---- OP_MID: post -> capture -> scale -> pre, in place on each quad/pair
            const int kind = fkind_of<OP>(p);
            const Scaling& Sc = p.s;
            const LineInfo L = linfo[lf];
            const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
            const double cst = Sc.bscale * Sc.inv_np;
            if (kind == FK_CFFT) {
                if (jt == 0) {
                    const cx<T> X = line_f[P(0)];
                    if (cap) *Sc.dc_out = (double)X.x;
                    line_f[P(0)] = cscale<T>(X, eig_factor<T>(Sc, L, 0));
                } else {
                    line_f[P(jt)] = cscale<T>(line_f[P(jt)], eig_factor_nz<T>(Sc, L, jt, cst));
                }
#pragma unroll
                for (int it = 1; it < 16; ++it) {
                    const int k = jt + it * TL;
                    line_f[P(k)] = cscale<T>(line_f[P(k)], eig_factor_nz<T>(Sc, L, k, cst));
                }
            } else if (kind == FK_RFFT || kind >= FK_DCT1) {
                const double csth = cst * 0.5;   // the untangle's 1/2
                // DCT-I keeps the real part of the spectrum, DST-I the imaginary one (the
                // other vanishes for the extended line; its eigenvalue index is k - 1,
                // which the planner folds into lam_t)
                const int r1 = kind == FK_DCT1 ? 1 : (kind == FK_DST1 ? 2 : 0);
                auto proj = [&](cx<T> x) { return r1 == 1 ? mkc<T>(x.x, 0) : (r1 == 2 ? mkc<T>(0, x.y) : x); };
                auto pair = [&](int q) {
                    const cx<T> zk = line_f[P(q)], zm = line_f[P(M - q)];
                    const cx<T> tq = Wt[q], tm = t_mirror<T>(tq);
                    const cx<T> xk = cscale<T>(proj(rsplit2<T>(zk, zm, tq)), eig_factor_nz<T>(Sc, L, q, csth));
                    const cx<T> xm = cscale<T>(proj(rsplit2<T>(zm, zk, tm)), eig_factor_nz<T>(Sc, L, M - q, csth));
                    line_f[P(q)] = rmerge<T>(xk, xm, tq);
                    line_f[P(M - q)] = rmerge<T>(xm, xk, tm);
                };
                if (jt == 0) {
                    const cx<T> z0 = line_f[P(0)];
                    if (r1 == 2) {
                        line_f[P(0)] = mkc<T>(0, 0);   // DST-I: V_0 = V_M = 0
                    } else {
                        T x0 = z0.x + z0.y, xM = z0.x - z0.y;
                        if (cap) *Sc.dc_out = (double)x0;
                        x0 *= eig_factor<T>(Sc, L, 0);
                        xM *= eig_factor<T>(Sc, L, M);
                        line_f[P(0)] = mkc<T>(x0 + xM, x0 - xM);
                    }
                    const cx<T> zh = line_f[P(HALF)];
                    const cx<T> xh = cscale<T>(proj(rsplit<T>(zh, zh, Wt[HALF])), eig_factor<T>(Sc, L, HALF));
                    line_f[P(HALF)] = rmerge<T>(xh, xh, Wt[HALF]);
                } else {
                    pair(jt);
                }
#pragma unroll
                for (int it = 1; it < 8; ++it) pair(jt + it * TL);
            } else {
                const bool dst = kind == FK_DST2;
#define KPHYS(K) (dst ? (n - 1 - (K)) : (K))
                const cx<T>* __restrict__ Wb = reinterpret_cast<const cx<T>*>(p.wb);
                const double* __restrict__ lt = Sc.lam_t;
                const double C = line_lam_sum(L);
                auto quad = [&](int q) {
                    cx<T> zk = line_f[P(q)], zm = line_f[P(M - q)];
                    T f0, f1, f2, f3;
                    eig_quad<T>(Sc.lam_pair, q, M, C, f0, f1, f2, f3);
                    mid_quad<T>(zk, zm, Ww[q], Wb[q], f0, f1, f2, f3);
                    line_f[P(q)] = zk;
                    line_f[P(M - q)] = zm;
                };
                if (jt == 0) {
                    const cx<T> z0 = line_f[P(0)];
                    const cx<T> wM = Ww[M];
                    T X0 = (T)2 * (z0.x + z0.y);
                    T XM = (T)2 * (z0.x - z0.y) * wM.x;
                    if (cap && !dst) *Sc.dc_out = (double)X0;
                    X0 *= eig_recip<T>(lt, KPHYS(0), C);
                    XM *= eig_recip<T>(lt, KPHYS(M), C);
                    const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                    line_f[P(0)] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                    const cx<T> zh = line_f[P(HALF)];
                    const cx<T> wh = Ww[HALF], th = Wt[HALF];
                    const cx<T> U = cmul<T>(wh, rsplit<T>(zh, zh, th));
                    const T Xa = (T)2 * U.x * eig_recip<T>(lt, KPHYS(HALF), C);
                    const T Xb = (T)-2 * U.y * eig_recip<T>(lt, KPHYS(n - HALF), C);
                    const cx<T> Vh = cmulc<T>(mkc<T>(Xa, -Xb), wh);
                    line_f[P(HALF)] = rmerge<T>(Vh, Vh, th);
                } else {
                    quad(jt);
                }
#pragma unroll 1
                for (int it = 1; it < 8; ++it) quad(jt + it * TL);
#undef KPHYS
            }
            __syncthreads();
        }
    } else {
        // =============== INVERSE pre-processing (line-major mapping)
        const int ik = ikind_of<OP>(p);
        if (ik == IK_DCT3 || ik == IK_DST3) {
            // two-phase: the real-valued view overlaps the complex slots
            const T* zr = reinterpret_cast<const T*>(line_f);
            cx<T> hold[16];
            QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);   // q = jt + TL it, ascending
            auto quad = [&](int q, int it) {
                cx<T> tq, wq;
                qt.get(q, tq, wq);
                const cx<T> wm = w_mirror<T>(wq);
                const cx<T> tm = t_mirror<T>(tq);
                const cx<T> Vk = cmulc<T>(mkc<T>(zr[PR(q)], -zr[PR(n - q)]), wq);
                const cx<T> Vm = cmulc<T>(mkc<T>(zr[PR(M - q)], -zr[PR(M + q)]), wm);
                hold[2 * it] = rmerge<T>(Vk, Vm, tq);
                hold[2 * it + 1] = rmerge<T>(Vm, Vk, tm);
            };
            if (jt == 0) {
                const T X0 = zr[PR(0)], XM = zr[PR(M)];
                const cx<T> wM = Ww[M];
                const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                hold[0] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                const cx<T> wh = Ww[HALF], th = Wt[HALF];
                const cx<T> Vh = cmulc<T>(mkc<T>(zr[PR(HALF)], -zr[PR(n - HALF)]), wh);
                hold[1] = rmerge<T>(Vh, Vh, th);
                cx<T> t0, w0;
                qt.get(0, t0, w0);   // keep the running twiddles in step
            } else {
                quad(jt, 0);
            }
#pragma unroll
            for (int it = 1; it < 8; ++it) quad(jt + it * TL, it);
            __syncthreads();
            line_f[P(jt)] = hold[0];
            line_f[P(jt == 0 ? HALF : M - jt)] = hold[1];
#pragma unroll
            for (int it = 1; it < 8; ++it) {
                const int q = jt + it * TL;
                line_f[P(q)] = hold[2 * it];
                line_f[P(M - q)] = hold[2 * it + 1];
            }
            __syncthreads();
        } else if (ik == IK_IRFFT || ik >= IK_DCT1) {   // DCT-I / DST-I: placed as a half spectrum
            auto pair = [&](int q) {
                const cx<T> xk = line_f[P(q)], xm = line_f[P(M - q)];
                const cx<T> tq = Wt[q];
                line_f[P(q)] = rmerge<T>(xk, xm, tq);
                line_f[P(M - q)] = rmerge<T>(xm, xk, t_mirror<T>(tq));
            };
            if (jt == 0) {
                const cx<T> x0 = line_f[P(0)], xM = line_f[P(M)];
                line_f[P(0)] = rmerge<T>(x0, xM, mkc<T>(1, 0));
                const cx<T> xh = line_f[P(HALF)];
                line_f[P(HALF)] = rmerge<T>(xh, xh, Wt[HALF]);
            } else {
                pair(jt);
            }
#pragma unroll
            for (int it = 1; it < 8; ++it) pair(jt + it * TL);
            __syncthreads();
        }
    }

    if constexpr (opb(OP) != OP_FWD) {
        // =============== INVERSE FFT + store (INV and MID)
        fft_tile<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W);
        compute_store_tail<T, LOGM, STRIDED, OP>(p, linfo, sm, 0, mid_store_scale<OP>(p));
    }
}

// ----------------------------------------------------------------------------
// Register path (M <= 512, i.e. TL <= 32 threads per line).  After the last
// radix-16 stage thread jt holds Z[jt + TL r] in registers; the partner of
// index k = jt + TL r is M - k = (TL - jt) + TL (15 - r), held by lane TL - jt
// of the same warp.  Post-processing, the MID scale and the inverse
// pre-processing then exchange the mirrored halves with warp shuffles instead
// of a shared-memory round trip, and the inverse FFT starts from registers.
template <typename T>
__device__ __forceinline__ cx<T> shfl_cx(cx<T> v, int src) {
    return mkc<T>(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// pz[r] = Z[M - (jt + TL r)] for r < 8 (jt = 0 uses its own registers)
template <typename T>
__device__ __forceinline__ void fetch_mirror(const cx<T>* v, cx<T>* pz, int jt, int partner) {
#pragma unroll
    for (int r = 0; r < 8; ++r) pz[r] = shfl_cx<T>(v[15 - r], partner);
    if (jt == 0) {
#pragma unroll
        for (int r = 1; r < 8; ++r) pz[r] = v[16 - r];
    }
}
// inverse of fetch_mirror: v[s], s >= 8, from the partner's pz (jt = 0: own)
// (v[8] of jt = 0 must be supplied by the caller: the self-paired HALF entry)
template <typename T>
__device__ __forceinline__ void return_mirror(cx<T>* v, const cx<T>* pz, int jt, int partner, cx<T> half0) {
#pragma unroll
    for (int s = 8; s < 16; ++s) v[s] = shfl_cx<T>(pz[15 - s], partner);
    if (jt == 0) {
        v[8] = half0;
#pragma unroll
        for (int s = 9; s < 16; ++s) v[s] = pz[16 - s];
    }
}

template <typename T, int LOGM, bool STRIDED, int OP>
__device__ __forceinline__ void compute_store_reg(const FftPass& p, const LineInfo* linfo, cx<T>* sm) {
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL, HALF = S::HALF;
    const int LS = line_stride<T, LOGM, STRIDED>(p);
    constexpr int n = 2 * M;
    const int tid = threadIdx.x;
    const int Lc = p.lines, logL = p.logLines;
    const void* __restrict__ W = p.wfft;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    const Geometry& g = p.g;
    const int lf = tid >> LOGTL;
    const int jt = tid & (TL - 1);
    const int lane = tid & 31;
    const int partner = (lane & ~(TL - 1)) | ((TL - jt) & (TL - 1));
    cx<T>* line_f = sm + lf * LS;
    cx<T> v[16], pz[8];

    if constexpr (opb(OP) == OP_FWD) {
        // CONTIG only: I/O mapping == line-major mapping
        fft_tile_to_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        const LineInfo L = linfo[lf];
        const int kind = fkind_of<OP>(p);
        const T om = (T)p.out_mult;
        if (kind == FK_CFFT) {
            if (!L.valid) return;
            cx<T>* po = reinterpret_cast<cx<T>*>(g.out) + L.out_off + (long long)jt * g.out_st;
            const long long step = (long long)TL * g.out_st;
#pragma unroll
            for (int r = 0; r < 16; ++r, po += step) *po = cscale<T>(v[r], om);
            return;
        }
        fetch_mirror<T>(v, pz, jt, partner);
        if (!L.valid) return;
        const long long os = g.out_st;
        if (kind == FK_RFFT) {
            cx<T>* const pb = reinterpret_cast<cx<T>*>(g.out) + L.out_off;
            const T omh = om * (T)0.5;
            QuadTw<T, kTwPowQ<T, OP>> qt(Wt, nullptr, jt, TL);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int q = jt + r * TL;
                cx<T> tq, wq_unused;
                qt.get(q, tq, wq_unused);
                if (r == 0 && jt == 0) {
                    const cx<T> z0 = v[0], zh = v[8];
                    pb[0] = mkc<T>((z0.x + z0.y) * om, 0);
                    pb[(long long)M * os] = mkc<T>((z0.x - z0.y) * om, 0);
                    pb[(long long)HALF * os] = cscale<T>(rsplit2<T>(zh, zh, Wt[HALF]), omh);
                } else {
                    pb[(long long)q * os] = cscale<T>(rsplit2<T>(v[r], pz[r], tq), omh);
                    pb[(long long)(M - q) * os] = cscale<T>(rsplit2<T>(pz[r], v[r], t_mirror<T>(tq)), omh);
                }
            }
        } else {
            const bool dst = kind == FK_DST2;
            T* const pb = reinterpret_cast<T*>(g.out) + L.out_off;
            const long long s1 = dst ? -os : os;
            T* const p0 = dst ? pb + (long long)(n - 1) * os : pb;
            QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int q = jt + r * TL;
                cx<T> tq, wq;
                qt.get(q, tq, wq);
                if (r == 0 && jt == 0) {
                    const cx<T> z0 = v[0], zh = v[8];
                    const cx<T> wM = Ww[M];
                    p0[0] = (T)2 * (z0.x + z0.y) * om;
                    p0[(long long)M * s1] = (T)2 * (z0.x - z0.y) * wM.x * om;
                    const cx<T> U = cmul<T>(Ww[HALF], rsplit2<T>(zh, zh, Wt[HALF]));
                    p0[(long long)HALF * s1] = U.x * om;
                    p0[(long long)(n - HALF) * s1] = -U.y * om;
                } else {
                    const cx<T> U1 = cmul<T>(wq, rsplit2<T>(v[r], pz[r], tq));
                    const cx<T> U2 = cmul<T>(w_mirror<T>(wq), rsplit2<T>(pz[r], v[r], t_mirror<T>(tq)));
                    p0[(long long)q * s1] = U1.x * om;
                    p0[(long long)(n - q) * s1] = -U1.y * om;
                    p0[(long long)(M - q) * s1] = U2.x * om;
                    p0[(long long)(M + q) * s1] = -U2.y * om;
                }
            }
        }
        return;
    } else {
        if constexpr (opb(OP) == OP_MID) {
            fft_tile_to_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
            const int kind = fkind_of<OP>(p);
            const Scaling& Sc = p.s;
            const LineInfo L = linfo[lf];
            const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
            const double cst = Sc.bscale * Sc.inv_np;
            if (kind == FK_CFFT) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int k = jt + r * TL;
                    if (r == 0 && jt == 0) {
                        if (cap) *Sc.dc_out = (double)v[0].x;
                        v[0] = cscale<T>(v[0], eig_factor<T>(Sc, L, 0));
                    } else {
                        v[r] = cscale<T>(v[r], eig_factor_nz<T>(Sc, L, k, cst));
                    }
                }
            } else {
                fetch_mirror<T>(v, pz, jt, partner);
                cx<T> half0 = mkc<T>(0, 0);
                if (kind == FK_RFFT) {
                    const double csth = cst * 0.5;
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int q = jt + r * TL;
                        if (r == 0 && jt == 0) {
                            const cx<T> z0 = v[0], zh = v[8];
                            T x0 = z0.x + z0.y, xM = z0.x - z0.y;
                            if (cap) *Sc.dc_out = (double)x0;
                            x0 *= eig_factor<T>(Sc, L, 0);
                            xM *= eig_factor<T>(Sc, L, M);
                            v[0] = mkc<T>(x0 + xM, x0 - xM);
                            const cx<T> xh = cscale<T>(rsplit<T>(zh, zh, Wt[HALF]), eig_factor<T>(Sc, L, HALF));
                            half0 = rmerge<T>(xh, xh, Wt[HALF]);
                        } else {
                            const cx<T> tq = Wt[q], tm = t_mirror<T>(tq);
                            const cx<T> xk = cscale<T>(rsplit2<T>(v[r], pz[r], tq), eig_factor_nz<T>(Sc, L, q, csth));
                            const cx<T> xm = cscale<T>(rsplit2<T>(pz[r], v[r], tm), eig_factor_nz<T>(Sc, L, M - q, csth));
                            v[r] = rmerge<T>(xk, xm, tq);
                            pz[r] = rmerge<T>(xm, xk, tm);
                        }
                    }
                } else {
                    const bool dst = kind == FK_DST2;
#define KPHYS(K) (dst ? (n - 1 - (K)) : (K))
                    const cx<T>* __restrict__ Wb = reinterpret_cast<const cx<T>*>(p.wb);
                    const double* __restrict__ lt = Sc.lam_t;
                    const double C = line_lam_sum(L);
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int q = jt + r * TL;
                        if (r == 0 && jt == 0) {
                            const cx<T> z0 = v[0], zh = v[8];
                            const cx<T> wM = Ww[M];
                            T X0 = (T)2 * (z0.x + z0.y);
                            T XM = (T)2 * (z0.x - z0.y) * wM.x;
                            if (cap && !dst) *Sc.dc_out = (double)X0;
                            X0 *= eig_recip<T>(lt, KPHYS(0), C);
                            XM *= eig_recip<T>(lt, KPHYS(M), C);
                            const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                            v[0] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                            const cx<T> wh = Ww[HALF], th = Wt[HALF];
                            const cx<T> U = cmul<T>(wh, rsplit<T>(zh, zh, th));
                            const T Xa = (T)2 * U.x * eig_recip<T>(lt, KPHYS(HALF), C);
                            const T Xb = (T)-2 * U.y * eig_recip<T>(lt, KPHYS(n - HALF), C);
                            const cx<T> Vh = cmulc<T>(mkc<T>(Xa, -Xb), wh);
                            half0 = rmerge<T>(Vh, Vh, th);
                        } else {
                            T f0, f1, f2, f3;
                            eig_quad<T>(Sc.lam_pair, q, M, C, f0, f1, f2, f3);
                            mid_quad<T>(v[r], pz[r], Ww[q], Wb[q], f0, f1, f2, f3);
                        }
                    }
#undef KPHYS
                }
                return_mirror<T>(v, pz, jt, partner, half0);
            }
        } else {
            // OP_INV, real kinds: pre-processing from the placed spectrum
            const int ik = ikind_of<OP>(p);
            cx<T> half0 = mkc<T>(0, 0);
            if (ik == IK_IRFFT) {
                QuadTw<T, kTwPowQ<T, OP>> qt(Wt, nullptr, jt, TL);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int q = jt + r * TL;
                    cx<T> tq, wq_unused;
                    qt.get(q, tq, wq_unused);
                    if (r == 0 && jt == 0) {
                        const cx<T> x0 = line_f[P(0)], xM = line_f[P(M)], xh = line_f[P(HALF)];
                        v[0] = rmerge<T>(x0, xM, mkc<T>(1, 0));
                        half0 = rmerge<T>(xh, xh, Wt[HALF]);
                    } else {
                        const cx<T> xk = line_f[P(q)], xm = line_f[P(M - q)];
                        v[r] = rmerge<T>(xk, xm, tq);
                        pz[r] = rmerge<T>(xm, xk, t_mirror<T>(tq));
                    }
                }
            } else {
                const T* zr = reinterpret_cast<const T*>(line_f);
                QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int q = jt + r * TL;
                    cx<T> tq0, wq0;
                    qt.get(q, tq0, wq0);
                    if (r == 0 && jt == 0) {
                        const T X0 = zr[PR(0)], XM = zr[PR(M)];
                        const cx<T> wM = Ww[M];
                        const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                        v[0] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                        const cx<T> wh = Ww[HALF], th = Wt[HALF];
                        const cx<T> Vh = cmulc<T>(mkc<T>(zr[PR(HALF)], -zr[PR(n - HALF)]), wh);
                        half0 = rmerge<T>(Vh, Vh, th);
                    } else {
                        const cx<T> wq = wq0, wm = w_mirror<T>(wq);
                        const cx<T> tq = tq0, tm = t_mirror<T>(tq);
                        const cx<T> Vk = cmulc<T>(mkc<T>(zr[PR(q)], -zr[PR(n - q)]), wq);
                        const cx<T> Vm = cmulc<T>(mkc<T>(zr[PR(M - q)], -zr[PR(M + q)]), wm);
                        v[r] = rmerge<T>(Vk, Vm, tq);
                        pz[r] = rmerge<T>(Vm, Vk, tm);
                    }
                }
            }
            return_mirror<T>(v, pz, jt, partner, half0);
        }
        // inverse FFT from registers (its first write is preceded by a barrier,
        // so the pre-processing reads above are complete)
        fft_tile_from_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        compute_store_tail<T, LOGM, STRIDED, OP>(p, linfo, sm, 0, mid_store_scale<OP>(p));
    }
}

// ----------------------------------------------------------------------------
// general path: one tile per CTA, loads straight from HBM
template <typename T, int LOGM, bool STRIDED, int OP>
__device__ __forceinline__ void fft_pass_tile(const FftPass& p) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using S = Shape<LOGM>;
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw + linfo_bytes(p.lines));
    setup_lines<STRIDED, OP>(p, blockIdx.x, linfo);
    __syncthreads();
    const int tid = threadIdx.x;
    const int lio = STRIDED ? (tid & (p.lines - 1)) : (tid >> S::LOGTL);
    const int bio = STRIDED ? (tid >> p.logLines) : (tid & (S::TL - 1));
    const LineInfo Lio = linfo[lio];
    cx<T>* line_io = sm + lio * line_stride<T, LOGM, STRIDED>(p);
    bool bad = place_tile<T, LOGM, STRIDED, OP>(p, Lio, line_io, bio);
    bad |= place_nyquist<T, LOGM, OP>(p, Lio, line_io, bio);
    if (bad) *p.nonfinite = 1;
    __syncthreads();
    if constexpr (S::TL <= 32 && !(opb(OP) == OP_FWD && STRIDED)) {
        if ((opb(OP) != OP_INV || ikind_of<OP>(p) != IK_ICFFT) && !is_r1<OP>(p)) {
            compute_store_reg<T, LOGM, STRIDED, OP>(p, linfo, sm);
            return;
        }
    }
    compute_store<T, LOGM, STRIDED, OP>(p, linfo, sm);   // (DCT-I / DST-I always take this path)
}

// Strided tiles: up to 512 threads, 128 registers (capping them spills the MID).
template <typename T, int LOGM, bool STRIDED, int OP>
__global__ void __launch_bounds__(512) fft_pass_kernel(const FftPass p) {
    fft_pass_tile<T, LOGM, STRIDED, OP>(p);
}

// Strided complex pass (MID, or forward / inverse complex FFT) whose I/O tile is
// twice as wide as one compute pass: the loads and stores cover 2W lines (twice
// the row segment: 64-B rows for fp32 2048-point lines instead of 32-B), the
// transform runs on W lines at a time with all 512 threads.  (c5: the axis-0
// MID at a 16.8 MB row stride is bound by DRAM transactions -- 16-B rows took
// it from 50 to 97 ms, 64-B rows from 50 to 40 ms.)
template <typename T, int LOGM, int OP>
__global__ void __launch_bounds__(512) fft_pass_wide(const FftPass p) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using S = Shape<LOGM>;
    constexpr int TL = S::TL, LOGTL = S::LOGTL;
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw + linfo_bytes(p.lines));
    setup_lines<true, OP>(p, blockIdx.x, linfo);
    __syncthreads();
    const int tid = threadIdx.x;
    const int LS = line_stride<T, LOGM, true>(p);
    const int lio = tid & (p.lines - 1);
    const int bio = tid >> p.logLines;   // row blocks [0, TL/2) of the first half
    const LineInfo Lio = linfo[lio];
    cx<T>* line_io = sm + lio * LS;
    bool bad = false;
#pragma unroll 1
    for (int f = 0; f < 2; ++f) bad |= place_tile<T, LOGM, true, OP>(p, Lio, line_io, bio + f * (TL / 2));
    if (bad) *p.nonfinite = 1;
    __syncthreads();
    const void* __restrict__ W = p.wfft;
    const int jt = tid & (TL - 1);
#pragma unroll 1
    for (int f = 0; f < 2; ++f) {
        const int lf = (tid >> LOGTL) + f * (p.lines >> 1);
        cx<T>* line_f = sm + lf * LS;
        if constexpr (opb(OP) == OP_MID) {
            const Scaling& Sc = p.s;
            const double cst = Sc.bscale * Sc.inv_np;
            const LineInfo L = linfo[lf];
            const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
            cx<T> v[16];
            fft_tile_to_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
            if (jt == 0) {
                if (cap) *Sc.dc_out = (double)v[0].x;
                v[0] = cscale<T>(v[0], eig_factor<T>(Sc, L, 0));
            } else {
                v[0] = cscale<T>(v[0], eig_factor_nz<T>(Sc, L, jt, cst));
            }
#pragma unroll
            for (int it = 1; it < 16; ++it) v[it] = cscale<T>(v[it], eig_factor_nz<T>(Sc, L, jt + it * TL, cst));
            fft_tile_from_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        } else {
            fft_tile<opb(OP) == OP_INV, T, LOGM, kTwPow<T, OP>>(line_f, jt, W);
        }
    }
    if constexpr (opb(OP) == OP_FWD) {
        // natural-order complex spectrum: row k = 16 b + i at 17 b + i
        if (!Lio.valid) return;
        const T om = (T)p.out_mult;
        const long long os = p.g.out_st;
#pragma unroll 1
        for (int f = 0; f < 2; ++f) {
            const int b = bio + f * (TL / 2);
            cx<T>* po = reinterpret_cast<cx<T>*>(p.g.out) + Lio.out_off + (long long)(16 * b) * os;
#pragma unroll
            for (int it = 0; it < 16; ++it, po += os) *po = cscale<T>(line_io[17 * b + it], om);
        }
    } else {
#pragma unroll 1
        for (int f = 0; f < 2; ++f) compute_store_tail<T, LOGM, true, OP>(p, linfo, sm, f * (TL / 2));
    }
}
#define FP_FFT_WIDE(NAME, T, L)                                                     \
    namespace fpb {                                                                 \
    FftKernelFn NAME(int op) {                                                      \
        return op == OP_MID ? fft_pass_wide<T, L, mid_op(FK_CFFT)>                  \
             : op == OP_FWD ? fft_pass_wide<T, L, OP_FWD> : fft_pass_wide<T, L, OP_INV>; \
    }                                                                               \
    }

// Long fp32 strided forward / inverse lines: at <= 64 registers two 512-thread
// CTAs fit per SM (70 would allow one).
#ifndef FP_WIDE_F32_REGS
#define FP_WIDE_F32_REGS 64
#endif
#ifndef FP_WIDE_F32_MID
#define FP_WIDE_F32_MID 0   // the MID too (variant builds; it spills at 64)
#endif
template <typename T, int LOGM, int OP>
__global__ void __maxnreg__(FP_WIDE_F32_REGS) fft_pass_wide_f32(const FftPass p) {
    fft_pass_tile<T, LOGM, true, OP>(p);
}

// Contiguous tiles trade registers for residency: capped at 72 (fp32) / 96 (fp64)
// they run 5-7 CTAs/SM instead of 4 (c5 line passes 16.5 -> 14.4 ms; c3 -2 %).
#ifndef FP_CONTIG_REGS_F32
#define FP_CONTIG_REGS_F32 72
#endif
#ifndef FP_CONTIG_REGS_F64
#define FP_CONTIG_REGS_F64 96
#endif
template <typename T> struct ContigRegs { static constexpr int v = sizeof(T) == 4 ? FP_CONTIG_REGS_F32 : FP_CONTIG_REGS_F64; };
template <typename T, int LOGM, int OP>
__global__ void __maxnreg__(ContigRegs<T>::v) fft_pass_contig(const FftPass p) {
    fft_pass_tile<T, LOGM, false, OP>(p);
}

// ----------------------------------------------------------------------------
// Pipelined STRIDED path: persistent CTAs, two transform tiles.  The loads of
// tile i+1 are cp.async copies of single elements (4/8/16 bytes) straight into
// their padded slots of the second tile -- the Makhoul / half-FFT placement is
// just the destination address -- while tile i is transformed and stored.
// (DST kinds need a sign flip on load and the first pass needs the
// non-finite check: both stay on fft_pass_kernel.)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_elem(void* dst, const void* src) {
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <typename T, int LOGM, int OP>
__device__ __forceinline__ void issue_tile_async(const FftPass& p, const LineInfo* linfo, cx<T>* sm) {
    using S = Shape<LOGM>;
    constexpr int M = S::M;
    const int LS = line_stride<T, LOGM, true>(p);
    constexpr int n = 2 * M;
    const int tid = threadIdx.x;
    const int lio = tid & (p.lines - 1);
    const int b = tid >> p.logLines;
    const LineInfo L = linfo[lio];
    if (!L.valid) return;
    const Geometry& g = p.g;
    cx<T>* line = sm + lio * LS;
    T* zr = reinterpret_cast<T*>(line);
    const long long st = g.in_st;
    const bool blk = blocked(g);
    auto row_off = [&](int j) -> long long { return blk ? blk_row(g, j, st, g.in_st_hi) : (long long)j * st; };
    const bool cin = complex_input<OP>(p);
    if (cin) {
        const cx<T>* src = reinterpret_cast<const cx<T>*>(g.in) + L.in_off;
#pragma unroll
        for (int it = 0; it < 16; ++it)
            cp_async_elem<sizeof(cx<T>)>(line + 17 * b + it, src + row_off(16 * b + it));
        if (opb(OP) == OP_INV && ikind_of<OP>(p) == IK_IRFFT && b == 0)
            cp_async_elem<sizeof(cx<T>)>(line + P(M), src + (long long)M * st);
    } else {
        const T* src = reinterpret_cast<const T*>(g.in) + L.in_off;
        const RowBlk rb(b, n);
        if (opb(OP) == OP_INV) {             // DCT-III: real spectrum in the PR layout
#pragma unroll
            for (int it = 0; it < 32; ++it) cp_async_elem<sizeof(T)>(zr + rb.pr + it, src + (long long)(32 * b + it) * st);
        } else if (fkind_of<OP>(p) == FK_RFFT) {
#pragma unroll
            for (int it = 0; it < 32; ++it) cp_async_elem<sizeof(T)>(zr + rb.r34 + it, src + row_off(32 * b + it));
        } else {                        // DCT-II: Makhoul reordering
#pragma unroll
            for (int it = 0; it < 32; ++it) cp_async_elem<sizeof(T)>(zr + rb.makhoul(it), src + row_off(32 * b + it));
        }
    }
}

template <typename T, int LOGM, int OP>
__global__ void __launch_bounds__(512) fft_pass_spipe(const FftPass p) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using S = Shape<LOGM>;
    const unsigned lib = (unsigned)linfo_bytes(p.lines);
    const unsigned zb = (unsigned)p.lines * (unsigned)line_stride<T, LOGM, true>(p) * (unsigned)sizeof(cx<T>);
    // buffer k: line table at smem_raw + k*lib, tile at smem_raw + 2*lib + k*zb
    int tile = blockIdx.x;
    if (tile >= p.tiles) return;
    setup_lines<true, OP>(p, tile, reinterpret_cast<LineInfo*>(smem_raw));
    __syncthreads();
    issue_tile_async<T, LOGM, OP>(p, reinterpret_cast<LineInfo*>(smem_raw), reinterpret_cast<cx<T>*>(smem_raw + 2 * lib));
    cp_async_commit_group();
    for (unsigned k = 0; tile < p.tiles; tile += gridDim.x, k ^= 1u) {
        const int next = tile + gridDim.x;
        LineInfo* lc = reinterpret_cast<LineInfo*>(smem_raw + k * lib);
        LineInfo* ln = reinterpret_cast<LineInfo*>(smem_raw + (k ^ 1u) * lib);
        cx<T>* zc = reinterpret_cast<cx<T>*>(smem_raw + 2 * lib + k * zb);
        cx<T>* zn = reinterpret_cast<cx<T>*>(smem_raw + 2 * lib + (k ^ 1u) * zb);
        if (next < p.tiles) setup_lines<true, OP>(p, next, ln);
        __syncthreads();   // ln written; zn free (the previous tile's compute is done)
        if (next < p.tiles) issue_tile_async<T, LOGM, OP>(p, ln, zn);
        cp_async_commit_group();
        cp_async_wait_prev();  // this thread's copies of `tile` have landed
        __syncthreads();       // ... and everybody's
        if constexpr (S::TL <= 32 && opb(OP) != OP_FWD) {
            if (opb(OP) != OP_INV || ikind_of<OP>(p) != IK_ICFFT) {
                compute_store_reg<T, LOGM, true, OP>(p, lc, zc);
                continue;
            }
        }
        compute_store<T, LOGM, true, OP>(p, lc, zc);
    }
}

inline bool wide_f32_enabled() {
    static const bool on = [] { const char* v = std::getenv("FP_WIDE_F32"); return !(v && *v == '0'); }();
    return on;
}
// strided entry point of (T, L, OPV): the 64-register one for long fp32 lines
template <typename T, int L, int OPV>
inline FftKernelFn strided_fn() {
    if constexpr (sizeof(T) == 4 && L >= 9 && (opb(OPV) != OP_MID || FP_WIDE_F32_MID))
        if (wide_f32_enabled()) return fft_pass_wide_f32<T, L, OPV>;
    return fft_pass_kernel<T, L, true, OPV>;
}
template <typename T, int L, int OPV>
inline FftKernelFn spipe_fn(bool strided) {
    if constexpr (opb(OPV) == OP_MID || L < 9) return nullptr;   // the MID step is not pipelined; nor short lines
    else return strided ? (FftKernelFn)fft_pass_spipe<T, L, OPV> : (FftKernelFn) nullptr;
}

}  // namespace fpb

// (an earlier persistent variant that staged raw rows through TMA/cp.async
// buffers and then re-placed them was slower -- its staging tiles cut residency
// to 1-2 CTAs/SM; fft_pass_spipe copies straight into the transform tile)
#define FP_FFT_PIPE_FN(T, L, s, OPV) spipe_fn<T, L, OPV>(s)

#define FP_FFT_PICK(NAME, T, LO, HI)                                                                  \
    namespace fpb {                                                                                   \
    template <int L, int OPV> static FftKernelFn NAME##_one(bool s, bool pipe) {                      \
        if (pipe) return FP_FFT_PIPE_FN(T, L, s, OPV);                                                \
        return s ? strided_fn<T, L, OPV>() : fft_pass_contig<T, L, OPV>;                              \
    }                                                                                                 \
    template <int L> static FftKernelFn NAME##_mid(bool s, bool pipe, int kind) {                     \
        if (pipe || !s || kind < 0) return NAME##_one<L, OP_MID>(s, pipe);                            \
        switch (kind) {                                                                               \
            case FK_DCT2: return strided_fn<T, L, mid_op(FK_DCT2)>();                        \
            case FK_DST2: return strided_fn<T, L, mid_op(FK_DST2)>();                        \
            case FK_RFFT: return strided_fn<T, L, mid_op(FK_RFFT)>();                        \
            case FK_DCT1: case FK_DST1: /* regular grids: the runtime-kind MID (build time) */     \
                return NAME##_one<L, OP_MID>(s, pipe);                                                \
            default: /* fp64 complex: the specialised build spills (c4 MID +7 %) */                  \
                if constexpr (sizeof(T) == 8) return NAME##_one<L, OP_MID>(s, pipe);                  \
                else return strided_fn<T, L, mid_op(FK_CFFT)>();                             \
        }                                                                                             \
    }                                                                                                 \
    template <int L> static FftKernelFn NAME##_rec(int logM, bool s, int op, bool pipe, int kind) {   \
        if constexpr (L > HI) { return nullptr; }                                                     \
        else {                                                                                        \
            if (logM != L) return NAME##_rec<L + 1>(logM, s, op, pipe, kind);                         \
            return op == OP_FWD ? NAME##_one<L, OP_FWD>(s, pipe)                                      \
                 : op == OP_INV ? NAME##_one<L, OP_INV>(s, pipe) : NAME##_mid<L>(s, pipe, kind);      \
        }                                                                                             \
    }                                                                                                 \
    FftKernelFn NAME(int logM, bool s, int op, bool pipe, int kind) {                                 \
        return NAME##_rec<LO>(logM, s, op, pipe, kind);                                               \
    }                                                                                                 \
    }
