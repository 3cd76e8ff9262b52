// fp_tma.cuh -- TMA-staged strided passes of the FFT line engine (fp64 DCT / DST
// lines, 16 adjacent columns = 128-B rows per tile, M <= 512: c3's y and x passes).
//
// The regular strided kernel moves every element through the LSU twice on the
// way in (LDG into registers, STS into the padded tile at its Makhoul position)
// and twice on the way out (LDS, STG); ncu put those passes at 68-70 % of the LSU
// data pipe (profiles/r02/ncu_full_c3_strided_v2.md).  Here one thread issues
// cp.async.bulk.tensor copies that land the tile in shared memory without the
// LSU, and the first FFT stage reads its butterfly inputs straight out of the
// staged rows (the Makhoul / half-FFT permutation folded into that read); the
// last inverse stage leaves its outputs in registers, which are written in the
// staged row layout and stored with cp.async.bulk.tensor.
//
// Staging layouts (SWIZZLE_128B: 16-B chunk c of row r at chunk c ^ (r & 7), so
// 16 lanes reading one column of 16 consecutive rows hit 8 distinct chunks):
//   PHASE   real rows y = 4t + phi in sub-tile phi, row t (TMA traversal stride 4):
//           the Makhoul half-FFT pairs z_m = (v_2m, v_2m+1) are rows (4m, 4m+2) for
//           m < M/2 and (2n-1-4m, 2n-3-4m) for m >= M/2 -- phases (0, 2) resp.
//           (3, 1) at the same t -- so consecutive m are consecutive t;
//   NATURAL rows in order (spectra: DCT-II outputs, DCT-III inputs).
// The staging area aliases the padded FFT tile: every stage reads all of its
// inputs before a barrier and only then writes.
#pragma once
#include <cuda.h>

#include "fp_fft.cuh"

namespace fpb {

__device__ __forceinline__ unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(smem_addr(bar)), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_addr(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)) : "memory");
}
// L2 prefetch of one box (no shared-memory destination, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(src)) : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// element (row r, column c) of a 1024-B aligned staging region of 128-B rows (fp64)
__device__ __forceinline__ int stg_off(int r, int c) { return r * 128 + ((((c >> 1) ^ r) & 7) << 4) + ((c & 1) << 3); }

template <int N>   // real line length n; PHASE sub-tile phi starts at phi * (n/4) rows
__device__ __forceinline__ double& stg_phase(unsigned char* stg, int phi, int t, int c) {
    return *reinterpret_cast<double*>(stg + phi * (N / 4) * 128 + stg_off(t, c));
}
__device__ __forceinline__ double& stg_nat(unsigned char* stg, int r, int c) {
    return *reinterpret_cast<double*>(stg + stg_off(r, c));
}

// one tile's coordinates: column block start, a index
struct TmaTile {
    int c0, ia;
};
__device__ __forceinline__ TmaTile tma_tile(const FftPass& p) {
    TmaTile t;
    t.ia = blockIdx.x / p.nbt;
    t.c0 = (blockIdx.x % p.nbt) * p.lines;
    return t;
}
// TMA coordinates (dim 0 = columns; the transform axis is dim p.tm_tdim, the a axis the other)
__device__ __forceinline__ void tma_coords(const FftPass& p, const TmaTile& tt, int row, int* c1, int* c2) {
    if (p.tm_tdim == 1) { *c1 = row; *c2 = tt.ia; }
    else { *c1 = tt.ia; *c2 = row; }
}

// issue the loads of one tile: PHASE (4 phases x n/256 boxes of 64 rows) or NATURAL (n/256 boxes of 256 rows)
template <int N>
__device__ __forceinline__ void tma_issue_load(const FftPass& p, const TmaTile& tt, unsigned char* stg, uint64_t* bar,
                                               bool phase) {
    mbar_expect_tx(bar, (unsigned)N * 128u);
    int c1, c2;
    if (phase) {
#pragma unroll
        for (int phi = 0; phi < 4; ++phi)
#pragma unroll
            for (int h = 0; h < N / 256; ++h) {
                tma_coords(p, tt, phi + 256 * h, &c1, &c2);
                tma_load_3d(stg + (phi * (N / 4) + 64 * h) * 128, &p.tm_in, tt.c0, c1, c2, bar);
            }
    } else {
#pragma unroll
        for (int h = 0; h < N / 256; ++h) {
            tma_coords(p, tt, 256 * h, &c1, &c2);
            tma_load_3d(stg + 256 * h * 128, &p.tm_in, tt.c0, c1, c2, bar);
        }
    }
}
// L2 prefetch of the tile `pf_tiles` ahead (the tile a later CTA on this SM will load: its TMA
// load then hits L2 instead of waiting ~2 us on HBM with the CTA's registers and shared memory idle)
template <int N>
__device__ __forceinline__ void tma_issue_prefetch(const FftPass& p) {
    if (p.pf_tiles <= 0) return;
    const int t = (int)blockIdx.x + p.pf_tiles;
    if (t >= p.tiles) return;
    TmaTile tt;
    tt.ia = t / p.nbt;
    tt.c0 = (t % p.nbt) * p.lines;
    int c1, c2;
    // always as NATURAL boxes of 256 consecutive rows through tm_aux (element stride 1 over the
    // input): a prefetch through the PHASE map (traversal stride 4) was measured to cost the
    // forward pass 20 % -- it appears to fetch the rows between the strided ones as well
#pragma unroll
    for (int h = 0; h < N / 256; ++h) {
        tma_coords(p, tt, 256 * h, &c1, &c2);
        tma_prefetch_3d(&p.tm_aux, tt.c0, c1, c2);
    }
}
template <int N>
__device__ __forceinline__ void tma_issue_store(const FftPass& p, const TmaTile& tt, const unsigned char* stg, bool phase) {
    int c1, c2;
    if (phase) {
#pragma unroll
        for (int phi = 0; phi < 4; ++phi)
#pragma unroll
            for (int h = 0; h < N / 256; ++h) {
                tma_coords(p, tt, phi + 256 * h, &c1, &c2);
                tma_store_3d(&p.tm_out, tt.c0, c1, c2, stg + (phi * (N / 4) + 64 * h) * 128);
            }
    } else {
#pragma unroll
        for (int h = 0; h < N / 256; ++h) {
            tma_coords(p, tt, 256 * h, &c1, &c2);
            tma_store_3d(&p.tm_out, tt.c0, c1, c2, stg + 256 * h * 128);
        }
    }
    tma_store_commit_wait();
}

// all stages, the first from registers vio[s] = z[jt + TL s], the last into them
template <bool INV, typename T, int LOGM, bool TWP>
__device__ __forceinline__ void fft_tile_reg_reg(cx<T>* line, int jt, const void* __restrict__ W, cx<T>* v) {
    constexpr int REM = LOGM & 3;
    if constexpr (REM == 0) stockham_stage<16, 0, INV, T, LOGM, true, false, TWP>(line, jt, W, v);
    if constexpr (REM == 1) stockham_stage<2, 0, INV, T, LOGM, true>(line, jt, W, v);
    if constexpr (REM == 2) stockham_stage<4, 0, INV, T, LOGM, true>(line, jt, W, v);
    if constexpr (REM == 3) stockham_stage<8, 0, INV, T, LOGM, true>(line, jt, W, v);
    constexpr int FIRST16 = REM == 0 ? 4 : REM;
    radix16_stages_upto<FIRST16, LOGM - 4, INV, T, LOGM, TWP>(line, jt, W);
    stockham_stage<16, LOGM - 4, INV, T, LOGM, false, true, TWP>(line, jt, W, v);
}

// Makhoul half-FFT pairs of line lf from the PHASE staging: v[s] = z_{jt + TL s}
template <int LOGM>
__device__ __forceinline__ void read_makhoul(unsigned char* stg, int lf, int jt, bool dst, cx<double>* v) {
    constexpr int M = 1 << LOGM, TL = M / 16, n = 2 * M;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int m = jt + TL * s;
        double a, b;
        if (s < 8) {   // m < M/2: rows 4m, 4m + 2
            a = stg_phase<n>(stg, 0, m, lf);
            b = stg_phase<n>(stg, 2, m, lf);
        } else {       // rows 2n-1-4m, 2n-3-4m (odd: DST-II's sign flip)
            const int t = n / 2 - 1 - m;
            a = stg_phase<n>(stg, 3, t, lf);
            b = stg_phase<n>(stg, 1, t, lf);
            if (dst) { a = -a; b = -b; }
        }
        v[s] = mkc<double>(a, b);
    }
}
// the first pass's non-finite check (solver.py:201-202) of line lf: this thread's 2M/TL
// staged values of its column (every row of a line is covered by its TL threads)
template <int LOGM>
__device__ __forceinline__ bool staged_nonfinite(unsigned char* stg, int lf, int jt) {
    constexpr int M = 1 << LOGM, TL = M / 16, n = 2 * M;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < n / TL; ++i) bad |= !finite_t(*reinterpret_cast<const double*>(stg + stg_off(jt + TL * i, lf)));
    return bad;
}

// ... and back: the inverse's time-domain pairs z_m = (v_2m, v_2m+1) to the x rows
template <int LOGM>
__device__ __forceinline__ void write_makhoul(unsigned char* stg, int lf, int jt, bool dst, double om, const cx<double>* v) {
    constexpr int M = 1 << LOGM, TL = M / 16, n = 2 * M;
    const double oo = dst ? -om : om;   // DST-III: odd rows negated
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int m = jt + TL * s;
        if (s < 8) {
            stg_phase<n>(stg, 0, m, lf) = v[s].x * om;
            stg_phase<n>(stg, 2, m, lf) = v[s].y * om;
        } else {
            const int t = n / 2 - 1 - m;
            stg_phase<n>(stg, 3, t, lf) = v[s].x * oo;
            stg_phase<n>(stg, 1, t, lf) = v[s].y * oo;
        }
    }
}

// smem layout of a TMA tile: [line table][pad to 1024][max(padded tile, staging)][mbarrier]
template <int LOGM>
__host__ __device__ constexpr size_t tma_stage_bytes() { return (size_t)(2 << LOGM) * 128; }
// Register-path kernels at M = 256 interleave the two lines of a warp (lane = 2 jt + line
// parity): a half-warp's 8-byte staging accesses then cover 8 rows x 2 adjacent columns =
// sixteen distinct 8-byte slots of the swizzled 128-B row instead of 16 rows of one column
// (rows t and t + 8 share a chunk: a 2-way conflict on every staged read and write, 27 % of
// the MID's shared-memory wavefronts, profiles/r02/ncu_full_c3_v6_raw.csv).  The FFT
// exchanges stay conflict-free with a line stride = 4 (mod 8): a quarter-warp's 16-byte
// accesses are 4 consecutive jt x 2 lines -> chunks (jt + 4 b) mod 8.
constexpr int kTmaAltLS = 276;
__host__ __device__ inline size_t tma_region_bytes(const FftPass& p, size_t stage) {
    const int ls = (p.logM == 8 && p.ls < kTmaAltLS) ? kTmaAltLS : p.ls;
    const size_t tile = (size_t)p.lines * ls * 16;
    return tile > stage ? tile : stage;
}
__host__ __device__ inline size_t tma_smem_bytes(const FftPass& p, size_t stage) {
    return linfo_bytes(p.lines) + 1024 + tma_region_bytes(p, stage) + 16;
}

// OP: OP_FWD (DCT-II / DST-II lines), OP_INV (DCT-III / DST-III), or the kind-specialised MID (DCT-II / DST-II)
// SMEM: the step between the forward and inverse FFTs goes through the shared-memory
// tile instead of registers + warp shuffles (fewer registers -> 3 CTAs per SM):
//   forward: post-process from the spectrum in shared memory, row stores to HBM;
//   inverse: pre-processed spectrum written to the tile, then the inverse FFT;
//   MID:     forward FFT into the tile, the folded 1/lam step in place per quad, inverse FFT
// (register paths: two resident CTAs, <= 128 registers -- an explicit minimum of 1 lets
// ptxas take 220+ and drops to one CTA per SM; shared-memory variants: three CTAs, 80
// registers -- the forward fits with 8 B of spill, the MID / inverse spill more and
// measured slower than their register paths, profiles/r02/ab_tma_variants.txt)
template <int LOGM, int OP, bool SMEM = false>
__global__ void __launch_bounds__(256, SMEM ? 3 : 2) fft_pass_tma(const __grid_constant__ FftPass p) {
    pdl_wait();
    using T = double;
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL, HALF = S::HALF, n = 2 * M;
    constexpr size_t STG = tma_stage_bytes<LOGM>();
    extern __shared__ __align__(16) unsigned char smem_raw[];   // (the staging base is aligned to 1024 below)
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    // 1024-B aligned staging (SWIZZLE_128B); offset arithmetic on the __shared__ array keeps
    // the compiler on LDS/STS (an integer round trip of the address would turn every tile
    // access into a generic LD/ST)
    unsigned char* const b0 = smem_raw + linfo_bytes(p.lines);
    unsigned char* stg = b0 + ((1024u - (smem_addr(b0) & 1023u)) & 1023u);
    cx<T>* sm = reinterpret_cast<cx<T>*>(stg);
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + tma_region_bytes(p, STG));
    const int tid = threadIdx.x;
    const TmaTile tt = tma_tile(p);
    constexpr bool kFwdIn = opb(OP) != OP_INV;
    if (tid == 0) {
        mbar_init(bar, 1);
        tma_issue_load<n>(p, tt, stg, bar, kFwdIn);
        tma_issue_prefetch<n>(p);
    }
    setup_lines<true, OP>(p, blockIdx.x, linfo);
    __syncthreads();

    constexpr bool ALT = !SMEM && LOGM == 8;   // two interleaved lines per warp (see kTmaAltLS)
    const int lane = tid & 31;
    const int lf = ALT ? (((tid >> 5) << 1) | (lane & 1)) : (tid >> LOGTL);
    const int jt = ALT ? (lane >> 1) : (tid & (TL - 1));
    const int partner = ALT ? ((((TL - jt) & (TL - 1)) << 1) | (lane & 1)) : ((lane & ~(TL - 1)) | ((TL - jt) & (TL - 1)));
    const int LS = ALT ? kTmaAltLS : line_stride<T, LOGM, true>(p);
    cx<T>* line_f = sm + lf * LS;
    const void* __restrict__ W = p.wfft;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    const LineInfo L = linfo[lf];
    cx<T> v[16], pz[8];
    mbar_wait(bar, 0);

    if constexpr (opb(OP) == OP_FWD && SMEM) {
        read_makhoul<LOGM>(stg, lf, jt, p.fkind == FK_DST2, v);
        if (p.nonfinite && L.valid && staged_nonfinite<LOGM>(stg, lf, jt)) *p.nonfinite = 1;
        fft_tile_from_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        const int lio = tid & (p.lines - 1), bio = tid >> p.logLines;
        fwd_strided_post<T, LOGM, OP>(p, linfo[lio], sm + lio * LS, bio);
        return;
    } else if constexpr (opb(OP) == OP_FWD) {
        const bool dst = p.fkind == FK_DST2;
        read_makhoul<LOGM>(stg, lf, jt, dst, v);
        if (p.nonfinite && L.valid && staged_nonfinite<LOGM>(stg, lf, jt)) *p.nonfinite = 1;
        fft_tile_reg_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        fetch_mirror<T>(v, pz, jt, partner);
        __syncthreads();   // every thread is done with the tile: the staging may be overwritten
        // DCT-II quads {q, n-q, M-q, M+q} into NATURAL rows (DST-II: row n-1-k)
        const T om = (T)p.out_mult;
        auto row = [&](int k) { return dst ? n - 1 - k : k; };
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq;
            qt.get(q, tq, wq);
            if (r == 0 && jt == 0) {
                const cx<T> z0 = v[0], zh = v[8];
                const cx<T> wM = Ww[M];
                stg_nat(stg, row(0), lf) = (T)2 * (z0.x + z0.y) * om;
                stg_nat(stg, row(M), lf) = (T)2 * (z0.x - z0.y) * wM.x * om;
                const cx<T> U = cmul<T>(Ww[HALF], rsplit2<T>(zh, zh, Wt[HALF]));
                stg_nat(stg, row(HALF), lf) = U.x * om;
                stg_nat(stg, row(n - HALF), lf) = -U.y * om;
            } else {
                const cx<T> U1 = cmul<T>(wq, rsplit2<T>(v[r], pz[r], tq));
                const cx<T> U2 = cmul<T>(w_mirror<T>(wq), rsplit2<T>(pz[r], v[r], t_mirror<T>(tq)));
                stg_nat(stg, row(q), lf) = U1.x * om;
                stg_nat(stg, row(n - q), lf) = -U1.y * om;
                stg_nat(stg, row(M - q), lf) = U2.x * om;
                stg_nat(stg, row(M + q), lf) = -U2.y * om;
            }
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) tma_issue_store<n>(p, tt, stg, false);
        return;
    } else if constexpr (opb(OP) == OP_INV && SMEM) {
        const bool dst = p.ikind == IK_DST3;
        auto X = [&](int k) { return stg_nat(stg, dst ? n - 1 - k : k, lf); };
        // all spectrum values of this thread's quads first (the tile aliases the staging)
        T xa[8], xb[8], xc[8], xd[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            if (r == 0) {   // (jt == 0: X_0, X_M, X_HALF, X_{n-HALF})
                xa[0] = X(jt == 0 ? 0 : q);
                xb[0] = X(jt == 0 ? M : n - q);
                xc[0] = X(jt == 0 ? HALF : M - q);
                xd[0] = X(jt == 0 ? n - HALF : M + q);
            } else {
                xa[r] = X(q); xb[r] = X(n - q); xc[r] = X(M - q); xd[r] = X(M + q);
            }
        }
        if (p.nonfinite && L.valid && staged_nonfinite<LOGM>(stg, lf, jt)) *p.nonfinite = 1;
        __syncthreads();
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq;
            qt.get(q, tq, wq);
            if (r == 0 && jt == 0) {
                const cx<T> wM = Ww[M];
                const cx<T> VM = cmulc<T>(mkc<T>(xb[0], -xb[0]), wM);
                line_f[P(0)] = rmerge<T>(mkc<T>(xa[0], 0), VM, mkc<T>(1, 0));
                const cx<T> wh = Ww[HALF], th = Wt[HALF];
                const cx<T> Vh = cmulc<T>(mkc<T>(xc[0], -xd[0]), wh);
                line_f[P(HALF)] = rmerge<T>(Vh, Vh, th);
            } else {
                const cx<T> wm = w_mirror<T>(wq), tm = t_mirror<T>(tq);
                const cx<T> Vk = cmulc<T>(mkc<T>(xa[r], -xb[r]), wq);
                const cx<T> Vm = cmulc<T>(mkc<T>(xc[r], -xd[r]), wm);
                line_f[P(q)] = rmerge<T>(Vk, Vm, tq);
                line_f[P(M - q)] = rmerge<T>(Vm, Vk, tm);
            }
        }
        __syncthreads();
        fft_tile_to_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        __syncthreads();
        write_makhoul<LOGM>(stg, lf, jt, dst, p.out_mult, v);
        fence_async_smem();
        __syncthreads();
        if (tid == 0) tma_issue_store<n>(p, tt, stg, true);
        return;
    } else if constexpr (opb(OP) == OP_INV) {
        // DCT-III / DST-III pre-processing straight from the NATURAL staging (DST-III: X reversed)
        const bool dst = p.ikind == IK_DST3;
        auto X = [&](int k) { return stg_nat(stg, dst ? n - 1 - k : k, lf); };
        cx<T> half0 = mkc<T>(0, 0);
        if (p.nonfinite && L.valid && staged_nonfinite<LOGM>(stg, lf, jt)) *p.nonfinite = 1;
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq;
            qt.get(q, tq, wq);
            if (r == 0 && jt == 0) {
                const T X0 = X(0), XM = X(M), Xh = X(HALF), Xnh = X(n - HALF);
                const cx<T> wM = Ww[M];
                const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                v[0] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                const cx<T> wh = Ww[HALF], th = Wt[HALF];
                const cx<T> Vh = cmulc<T>(mkc<T>(Xh, -Xnh), wh);
                half0 = rmerge<T>(Vh, Vh, th);
            } else {
                const T a = X(q), b = X(n - q), c = X(M - q), d = X(M + q);
                const cx<T> wm = w_mirror<T>(wq), tm = t_mirror<T>(tq);
                const cx<T> Vk = cmulc<T>(mkc<T>(a, -b), wq);
                const cx<T> Vm = cmulc<T>(mkc<T>(c, -d), wm);
                v[r] = rmerge<T>(Vk, Vm, tq);
                pz[r] = rmerge<T>(Vm, Vk, tm);
            }
        }
        return_mirror<T>(v, pz, jt, partner, half0);
        fft_tile_reg_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        __syncthreads();
        write_makhoul<LOGM>(stg, lf, jt, dst, p.out_mult, v);
        fence_async_smem();
        __syncthreads();
        if (tid == 0) tma_issue_store<n>(p, tt, stg, true);
        return;
    } else if constexpr (SMEM) {
        // MID through the tile: forward FFT (first stage from the staging) into shared memory,
        // the folded 1/lam step in place per quad (each quad's two slots belong to one thread),
        // inverse FFT with its last stage into registers
        const int kind = fkind_of<OP>(p);
        const bool dst = kind == FK_DST2;
        read_makhoul<LOGM>(stg, lf, jt, dst, v);
        if (p.nonfinite && L.valid && staged_nonfinite<LOGM>(stg, lf, jt)) *p.nonfinite = 1;
        fft_tile_from_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        const Scaling& Sc = p.s;
        const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
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
        __syncthreads();
        fft_tile_to_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        __syncthreads();
        write_makhoul<LOGM>(stg, lf, jt, dst, p.out_mult * Sc.bscale * Sc.inv_np, v);
        fence_async_smem();
        __syncthreads();
        if (tid == 0) tma_issue_store<n>(p, tt, stg, true);
    } else {
        // MID: forward, null capture, folded 1/lam step, inverse -- all in registers but the FFT stages
        const int kind = fkind_of<OP>(p);
        const bool dst = kind == FK_DST2;
        read_makhoul<LOGM>(stg, lf, jt, dst, v);
        if (p.nonfinite && L.valid && staged_nonfinite<LOGM>(stg, lf, jt)) *p.nonfinite = 1;
        fft_tile_reg_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        const Scaling& Sc = p.s;
        const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
        fetch_mirror<T>(v, pz, jt, partner);
        cx<T> half0 = mkc<T>(0, 0);
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
        return_mirror<T>(v, pz, jt, partner, half0);
        fft_tile_reg_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        __syncthreads();
        write_makhoul<LOGM>(stg, lf, jt, dst, p.out_mult * Sc.bscale * Sc.inv_np, v);
        fence_async_smem();
        __syncthreads();
        if (tid == 0) tma_issue_store<n>(p, tt, stg, true);
    }
}

// ----------------------------------------------------------------------------
// Real-FFT lines (periodic axis transformed as a real FFT on a strided axis: c4's y
// passes): n = 2M = 1024 real points, 8 adjacent columns (64-B rows), TL = 32.
//   forward: real rows in PAIR staging -- rows y = 2t + phi in sub-tile phi, row t
//            (traversal stride 2), so z_m = (x_2m, x_2m+1) is row m of both sub-tiles --
//            -> FFT -> untangle -> complex half spectrum X_0..X_M in NATURAL rows of
//            8 complex (128 B) -> TMA store;
//   inverse: the half spectrum from NATURAL complex rows -> tangle -> inverse FFT ->
//            the real pairs back into PAIR staging -> TMA store.
// 64-B rows (SWIZZLE_64B): 16-B chunk c of row r at chunk c ^ ((r >> 1) & 3)
__device__ __forceinline__ int stg_off64(int r, int byte) {
    return r * 64 + (((((byte >> 4) ^ (r >> 1)) & 3)) << 4) + (byte & 15);
}
template <int N>   // PAIR sub-tile phi (n/2 rows of 64 B) starts at phi * (n/2) * 64
__device__ __forceinline__ double& stg_pair(unsigned char* stg, int phi, int t, int c) {
    return *reinterpret_cast<double*>(stg + phi * (N / 2) * 64 + stg_off64(t, c * 8));
}
__device__ __forceinline__ cx<double>& stg_cnat(unsigned char* stg, int r, int c) {   // 8 complex per row
    return *reinterpret_cast<cx<double>*>(stg + r * 128 + (((c ^ r) & 7) << 4));
}

template <int LOGM, int OP>
__global__ void __launch_bounds__(256, 2) fft_pass_tma_r(const __grid_constant__ FftPass p) {
    pdl_wait();
    using T = double;
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL, HALF = S::HALF, n = 2 * M;
    constexpr bool kFwd = opb(OP) == OP_FWD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    unsigned char* const b0 = smem_raw + linfo_bytes(p.lines);
    unsigned char* stg = b0 + ((1024u - (smem_addr(b0) & 1023u)) & 1023u);
    cx<T>* sm = reinterpret_cast<cx<T>*>(stg);
    const size_t tile = (size_t)p.lines * p.ls * 16;
    const size_t cstg = (size_t)(M + 8) * 128;
    const size_t region = tile > cstg ? tile : cstg;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + region);
    const int tid = threadIdx.x;
    const TmaTile tt = tma_tile(p);
    int c1, c2;
    if (tid == 0) {
        mbar_init(bar, 1);
        if constexpr (kFwd) {   // PAIR staging: 2 phases x n/512 boxes of 128 rows (traversal stride 2)
            mbar_expect_tx(bar, (unsigned)n * 64u);
#pragma unroll
            for (int phi = 0; phi < 2; ++phi)
#pragma unroll
                for (int h = 0; h < n / 256; ++h) {
                    tma_coords(p, tt, phi + 256 * h, &c1, &c2);
                    tma_load_3d(stg + (phi * (n / 2) + 128 * h) * 64, &p.tm_in, tt.c0, c1, c2, bar);
                }
            const int tpf = (int)blockIdx.x + p.pf_tiles;   // L2 prefetch of a later tile's real rows
            if (p.pf_tiles > 0 && tpf < p.tiles) {
                TmaTile tp;
                tp.ia = tpf / p.nbt;
                tp.c0 = (tpf % p.nbt) * p.lines;
#pragma unroll
                for (int phi = 0; phi < 2; ++phi)
#pragma unroll
                    for (int h = 0; h < n / 256; ++h) {
                        tma_coords(p, tp, phi + 256 * h, &c1, &c2);
                        tma_prefetch_3d(&p.tm_in, tp.c0, c1, c2);
                    }
            }
        } else {                // NATURAL complex rows 0..M: boxes of 256 rows + one of 8 (tm_aux)
            mbar_expect_tx(bar, (unsigned)(M + 8) * 128u);
#pragma unroll
            for (int h = 0; h < M / 256; ++h) {
                tma_coords(p, tt, 256 * h, &c1, &c2);
                tma_load_3d(stg + 256 * h * 128, &p.tm_in, 2 * tt.c0, c1, c2, bar);
            }
            tma_coords(p, tt, M, &c1, &c2);
            tma_load_3d(stg + M * 128, &p.tm_aux, 2 * tt.c0, c1, c2, bar);
            // L2 prefetch of the half spectrum of the tile one resident wave ahead
            const int tpf = (int)blockIdx.x + p.pf_tiles;
            if (p.pf_tiles > 0 && tpf < p.tiles) {
                TmaTile tp;
                tp.ia = tpf / p.nbt;
                tp.c0 = (tpf % p.nbt) * p.lines;
#pragma unroll
                for (int h = 0; h < M / 256; ++h) {
                    tma_coords(p, tp, 256 * h, &c1, &c2);
                    tma_prefetch_3d(&p.tm_in, 2 * tp.c0, c1, c2);
                }
                tma_coords(p, tp, M, &c1, &c2);
                tma_prefetch_3d(&p.tm_aux, 2 * tp.c0, c1, c2);
            }
        }
    }
    setup_lines<true, OP>(p, blockIdx.x, linfo);
    __syncthreads();
    const int lf = tid >> LOGTL, jt = tid & (TL - 1);
    const int lane = tid & 31;
    const int partner = (lane & ~(TL - 1)) | ((TL - jt) & (TL - 1));
    const int LS = line_stride<T, LOGM, true>(p);
    cx<T>* line_f = sm + lf * LS;
    const void* __restrict__ W = p.wfft;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const LineInfo L = linfo[lf];
    const T om = (T)p.out_mult;
    cx<T> v[16], pz[8];
    mbar_wait(bar, 0);
    if constexpr (kFwd) {
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            const int m = jt + TL * s;
            v[s] = mkc<T>(stg_pair<n>(stg, 0, m, lf), stg_pair<n>(stg, 1, m, lf));
        }
        if (p.nonfinite && L.valid) {
            bool bad = false;
#pragma unroll
            for (int s = 0; s < 16; ++s) bad |= !(finite_t(v[s].x) && finite_t(v[s].y));
            if (bad) *p.nonfinite = 1;
        }
        fft_tile_reg_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        fetch_mirror<T>(v, pz, jt, partner);
        __syncthreads();   // the complex staging overwrites the tile
        const T omh = om * (T)0.5;
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, nullptr, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq_unused;
            qt.get(q, tq, wq_unused);
            if (r == 0 && jt == 0) {
                const cx<T> z0 = v[0], zh = v[8];
                stg_cnat(stg, 0, lf) = mkc<T>((z0.x + z0.y) * om, 0);
                stg_cnat(stg, M, lf) = mkc<T>((z0.x - z0.y) * om, 0);
                stg_cnat(stg, HALF, lf) = cscale<T>(rsplit2<T>(zh, zh, Wt[HALF]), omh);
            } else {
                stg_cnat(stg, q, lf) = cscale<T>(rsplit2<T>(v[r], pz[r], tq), omh);
                stg_cnat(stg, M - q, lf) = cscale<T>(rsplit2<T>(pz[r], v[r], t_mirror<T>(tq)), omh);
            }
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int h = 0; h < M / 256; ++h) {
                tma_coords(p, tt, 256 * h, &c1, &c2);
                tma_store_3d(&p.tm_out, 2 * tt.c0, c1, c2, stg + 256 * h * 128);
            }
            tma_coords(p, tt, M, &c1, &c2);   // row M (the 8-row box is clipped to the tensor)
            tma_store_3d(&p.tm_aux, 2 * tt.c0, c1, c2, stg + M * 128);
            tma_store_commit_wait();
        }
    } else {
        cx<T> half0 = mkc<T>(0, 0);
        if (p.nonfinite && L.valid) {
            bool bad = false;
            for (int k = jt; k <= M; k += TL) {
                const cx<T> x = stg_cnat(stg, k, lf);
                bad |= !(finite_t(x.x) && finite_t(x.y));
            }
            if (bad) *p.nonfinite = 1;
        }
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, nullptr, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq_unused;
            qt.get(q, tq, wq_unused);
            if (r == 0 && jt == 0) {
                const cx<T> x0 = stg_cnat(stg, 0, lf), xM = stg_cnat(stg, M, lf), xh = stg_cnat(stg, HALF, lf);
                v[0] = rmerge<T>(x0, xM, mkc<T>(1, 0));
                half0 = rmerge<T>(xh, xh, Wt[HALF]);
            } else {
                const cx<T> xk = stg_cnat(stg, q, lf), xm = stg_cnat(stg, M - q, lf);
                v[r] = rmerge<T>(xk, xm, tq);
                pz[r] = rmerge<T>(xm, xk, t_mirror<T>(tq));
            }
        }
        return_mirror<T>(v, pz, jt, partner, half0);
        fft_tile_reg_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        __syncthreads();
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            const int m = jt + TL * s;
            stg_pair<n>(stg, 0, m, lf) = v[s].x * om;
            stg_pair<n>(stg, 1, m, lf) = v[s].y * om;
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int phi = 0; phi < 2; ++phi)
#pragma unroll
                for (int h = 0; h < n / 256; ++h) {
                    tma_coords(p, tt, phi + 256 * h, &c1, &c2);
                    tma_store_3d(&p.tm_out, tt.c0, c1, c2, stg + (phi * (n / 2) + 128 * h) * 64);
                }
            tma_store_commit_wait();
        }
    }
}

// ----------------------------------------------------------------------------
// Complex lines (the MID over a complex state: c4's x axis after the real FFT along y):
// M = 1024 complex fp64 points, 4 adjacent columns (64-B rows of 4 complex), TL = 64.
// NATURAL staging (row k = z_k; SWIZZLE_64B: eight consecutive rows of one column fall
// in eight distinct 16-B bank groups); the first forward stage reads its butterfly
// inputs from the staged rows, the eigenvalue divide is pointwise on the registers the
// last forward stage leaves, and the last inverse stage's outputs go back to the rows.
__device__ __forceinline__ cx<double>& stg_c64(unsigned char* stg, int r, int c) {   // 4 complex per row
    return *reinterpret_cast<cx<double>*>(stg + stg_off64(r, c * 16));
}

template <int LOGM>
__global__ void __launch_bounds__(256, 2) fft_pass_tma_c(const __grid_constant__ FftPass p) {
    pdl_wait();
    using T = double;
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL;
    constexpr int OP = mid_op(FK_CFFT);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    unsigned char* const b0 = smem_raw + linfo_bytes(p.lines);
    unsigned char* stg = b0 + ((1024u - (smem_addr(b0) & 1023u)) & 1023u);
    cx<T>* sm = reinterpret_cast<cx<T>*>(stg);
    const size_t tile = (size_t)p.lines * p.ls * 16, cstg = (size_t)M * 64;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + (tile > cstg ? tile : cstg));
    const int tid = threadIdx.x;
    const TmaTile tt = tma_tile(p);
    int c1, c2;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (unsigned)M * 64u);
#pragma unroll
        for (int h = 0; h < M / 256; ++h) {
            tma_coords(p, tt, 256 * h, &c1, &c2);
            tma_load_3d(stg + 256 * h * 64, &p.tm_in, 2 * tt.c0, c1, c2, bar);
        }
    }
    setup_lines<true, OP>(p, blockIdx.x, linfo);
    __syncthreads();
    const int lf = tid >> LOGTL, jt = tid & (TL - 1);
    const int LS = line_stride<T, LOGM, true>(p);
    cx<T>* line_f = sm + lf * LS;
    const void* __restrict__ W = p.wfft;
    const LineInfo L = linfo[lf];
    cx<T> v[16];
    mbar_wait(bar, 0);
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = stg_c64(stg, jt + TL * s, lf);
    if (p.nonfinite && L.valid) {
        bool bad = false;
#pragma unroll
        for (int s = 0; s < 16; ++s) bad |= !(finite_t(v[s].x) && finite_t(v[s].y));
        if (bad) *p.nonfinite = 1;
    }
    fft_tile_reg_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
    const Scaling& Sc = p.s;
    const bool cap = Sc.singular && Sc.dc_out && L.null_line && L.valid;
    const double cst = Sc.bscale * Sc.inv_np;
    if (jt == 0) {
        if (cap) *Sc.dc_out = (double)v[0].x;
        v[0] = cscale<T>(v[0], eig_factor<T>(Sc, L, 0));
    } else {
        v[0] = cscale<T>(v[0], eig_factor_nz<T>(Sc, L, jt, cst));
    }
#pragma unroll
    for (int it = 1; it < 16; ++it) v[it] = cscale<T>(v[it], eig_factor_nz<T>(Sc, L, jt + it * TL, cst));
    fft_tile_reg_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
    __syncthreads();
    const T om = (T)p.out_mult;
#pragma unroll
    for (int s = 0; s < 16; ++s) stg_c64(stg, jt + TL * s, lf) = cscale<T>(v[s], om);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int h = 0; h < M / 256; ++h) {
            tma_coords(p, tt, 256 * h, &c1, &c2);
            tma_store_3d(&p.tm_out, 2 * tt.c0, c1, c2, stg + 256 * h * 64);
        }
        tma_store_commit_wait();
    }
}

// ----------------------------------------------------------------------------
// Contiguous DCT / DST lines (c3's z passes): L = 2 lines of n = 2M = 512 fp64 per CTA.
// A 4D tensor map views each line as n/16 rows of 128 B; the CTA's box lands UNSWIZZLED as
// [line][row][16 doubles] = the line in natural order, element k of line l at l*n*8 + 8k.
// The spectrum side (DCT-II outputs, DCT-III inputs: rows q, n-q, M-q, M+q of consecutive
// threads) is conflict-free 8-byte accesses at base + immediate.  The time-domain side reads
// 32 contiguous bytes per half-FFT index m -- x_4m .. x_4m+3 as two 16-byte accesses: the even
// pair is z_m, the odd pair (x_4m+3, x_4m+1) is z_{M-1-m}, which the thread 15 - jt of the
// same line holds in slot 15 - s -- and exchanges the odd pairs with one warp shuffle each.
// (A 128-B-swizzled staging needed ~5 integer instructions of address arithmetic per access:
// 40 % of the kernel's instructions at 70 % issue utilisation.)
template <int N>
__device__ __forceinline__ double& stg_lin(unsigned char* stg, int l, int k) {
    return *reinterpret_cast<double*>(stg + l * (N * 8) + k * 8);
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(smem_addr(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3, const void* src) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(src)) : "memory");
}

template <int LOGM, int OP>   // OP_FWD (DCT-II / DST-II) or OP_INV (DCT-III / DST-III)
__global__ void __maxnreg__(128) fft_pass_tma_z(const __grid_constant__ FftPass p) {
    pdl_wait();
    using T = double;
    using S = Shape<LOGM>;
    constexpr int M = S::M, LOGTL = S::LOGTL, TL = S::TL, HALF = S::HALF, n = 2 * M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    unsigned char* const b0 = smem_raw + linfo_bytes(p.lines);
    unsigned char* stg = b0 + ((1024u - (smem_addr(b0) & 1023u)) & 1023u);
    cx<T>* sm = reinterpret_cast<cx<T>*>(stg);
    const size_t tile = (size_t)p.lines * S::LS * 16, sbytes = (size_t)p.lines * n * 8;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + (tile > sbytes ? tile : sbytes));
    const int tid = threadIdx.x;
    // (tma_prepare_z admits only line counts below 2^31: 32-bit divides)
    const unsigned l0 = blockIdx.x * (unsigned)p.lines;
    const int ia = (int)(l0 / (unsigned)p.g.nb), ib0 = (int)(l0 - (unsigned)ia * (unsigned)p.g.nb);
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (unsigned)sbytes);
        tma_load_4d(stg, &p.tm_in, 0, 0, ib0, ia, bar);
    }
    setup_lines<false, OP>(p, blockIdx.x, linfo);
    __syncthreads();
    const int lf = tid >> LOGTL, jt = tid & (TL - 1);
    const int lane = tid & 31;
    const int partner = (lane & ~(TL - 1)) | ((TL - jt) & (TL - 1));
    static_assert(TL == 16, "two 512-point lines per warp");
    const int partner2 = (lane & ~(TL - 1)) | (TL - 1 - jt);   // holds z_{M-1-m} in slot 15 - s
    cx<T>* line_f = sm + lf * S::LS;
    const void* __restrict__ W = p.wfft;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    const LineInfo L = linfo[lf];
    const T om = (T)p.out_mult;
    cx<T> v[16], pz[8];
    mbar_wait(bar, 0);
    if constexpr (opb(OP) == OP_INV) {
        if (p.nonfinite && L.valid) {
            bool bad = false;
#pragma unroll
            for (int i = 0; i < n / TL; ++i) bad |= !finite_t(stg_lin<n>(stg, lf, jt + TL * i));
            if (bad) *p.nonfinite = 1;
        }
    }
    if constexpr (opb(OP) == OP_FWD) {
        const bool dst = p.fkind == FK_DST2;
        {
            cx<T> odd[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const double2* c = reinterpret_cast<const double2*>(stg + lf * (n * 8) + 32 * (jt + TL * s));
                const double2 c0 = c[0], c1 = c[1];
                v[s] = mkc<T>(c0.x, c1.x);
                odd[s] = mkc<T>(c1.y, c0.y);
            }
#pragma unroll
            for (int s = 8; s < 16; ++s) {
                v[s] = shfl_cx<T>(odd[15 - s], partner2);
                if (dst) v[s] = mkc<T>(-v[s].x, -v[s].y);
            }
        }
        // the first pass's non-finite check (solver.py:201-202): the line's 16 threads hold every
        // element of it exactly once in v[]; 0 * x is NaN for x = NaN / +-Inf, so one fused
        // multiply-add per value and one test replace a second read of the staged line
        if (p.nonfinite && L.valid) {
            T acc = (T)0;
#pragma unroll
            for (int s = 0; s < 16; ++s) acc = fma(v[s].x, (T)0, fma(v[s].y, (T)0, acc));
            if (acc != (T)0) *p.nonfinite = 1;
        }
        fft_tile_reg_reg<false, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        fetch_mirror<T>(v, pz, jt, partner);
        __syncthreads();
        auto row = [&](int k) { return dst ? n - 1 - k : k; };
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq;
            qt.get(q, tq, wq);
            if (r == 0 && jt == 0) {
                const cx<T> z0 = v[0], zh = v[8];
                const cx<T> wM = Ww[M];
                stg_lin<n>(stg, lf, row(0)) = (T)2 * (z0.x + z0.y) * om;
                stg_lin<n>(stg, lf, row(M)) = (T)2 * (z0.x - z0.y) * wM.x * om;
                const cx<T> U = cmul<T>(Ww[HALF], rsplit2<T>(zh, zh, Wt[HALF]));
                stg_lin<n>(stg, lf, row(HALF)) = U.x * om;
                stg_lin<n>(stg, lf, row(n - HALF)) = -U.y * om;
            } else {
                const cx<T> U1 = cmul<T>(wq, rsplit2<T>(v[r], pz[r], tq));
                const cx<T> U2 = cmul<T>(w_mirror<T>(wq), rsplit2<T>(pz[r], v[r], t_mirror<T>(tq)));
                stg_lin<n>(stg, lf, row(q)) = U1.x * om;
                stg_lin<n>(stg, lf, row(n - q)) = -U1.y * om;
                stg_lin<n>(stg, lf, row(M - q)) = U2.x * om;
                stg_lin<n>(stg, lf, row(M + q)) = -U2.y * om;
            }
        }
    } else {
        const bool dst = p.ikind == IK_DST3;
        auto X = [&](int k) { return stg_lin<n>(stg, lf, dst ? n - 1 - k : k); };
        cx<T> half0 = mkc<T>(0, 0);
        QuadTw<T, kTwPowQ<T, OP>> qt(Wt, Ww, jt, TL);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = jt + r * TL;
            cx<T> tq, wq;
            qt.get(q, tq, wq);
            if (r == 0 && jt == 0) {
                const T X0 = X(0), XM = X(M), Xh = X(HALF), Xnh = X(n - HALF);
                const cx<T> wM = Ww[M];
                const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                v[0] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                const cx<T> wh = Ww[HALF], th = Wt[HALF];
                const cx<T> Vh = cmulc<T>(mkc<T>(Xh, -Xnh), wh);
                half0 = rmerge<T>(Vh, Vh, th);
            } else {
                const T a = X(q), b = X(n - q), c = X(M - q), d = X(M + q);
                const cx<T> wm = w_mirror<T>(wq), tm = t_mirror<T>(tq);
                const cx<T> Vk = cmulc<T>(mkc<T>(a, -b), wq);
                const cx<T> Vm = cmulc<T>(mkc<T>(c, -d), wm);
                v[r] = rmerge<T>(Vk, Vm, tq);
                pz[r] = rmerge<T>(Vm, Vk, tm);
            }
        }
        return_mirror<T>(v, pz, jt, partner, half0);
        fft_tile_reg_reg<true, T, LOGM, kTwPow<T, OP>>(line_f, jt, W, v);
        __syncthreads();
        const double oo = dst ? -om : om;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const cx<T> po = shfl_cx<T>(v[15 - s], partner2);   // (x_4m+3, x_4m+1) of this thread's m
            double2* c = reinterpret_cast<double2*>(stg + lf * (n * 8) + 32 * (jt + TL * s));
            c[0] = make_double2(v[s].x * om, po.y * oo);
            c[1] = make_double2(v[s].y * om, po.x * oo);
        }
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
        tma_store_4d(&p.tm_out, 0, 0, ib0, ia, stg);
        tma_store_commit_wait();
    }
}

}  // namespace fpb
