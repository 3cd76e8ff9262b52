// fp_fft.cuh -- the FFT line-engine pass kernel (see fp_kernels.cu header for
// the algorithm).  Instantiated per (precision, log2 FFT length, family) in the
// fp_fft_*.cu translation units, which are compiled in parallel.
#pragma once
#include "fp_common.cuh"

namespace fpb {

using FftKernelFn = void (*)(const FftPass);

// the FFT pass kernel: compile-time FFT length M = 2^LOGM and line family.
//
// Thread mappings (nth = lines * M/16 threads, TL = M/16):
//   line-major  (FFT stages, MID step):  line = tid / TL, jt = tid % TL
//   I/O mapping (global loads/stores):   CONTIG = line-major (lanes walk along a
//     line), STRIDED = column-major (lanes walk across the W adjacent lines so
//     each row segment of W elements is one coalesced access).
// Every per-thread loop has a compile-time trip count, and all of a thread's
// global loads are issued before the first shared-memory store.

template <typename T, int LOGM, bool STRIDED, int OP>
__global__ void __launch_bounds__(512) fft_pass_kernel(const FftPass p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int M = 1 << LOGM;
    constexpr int LOGTL = LOGM - 4;
    constexpr int TL = 1 << LOGTL;
    constexpr int HALF = M / 2;
    constexpr int LS = ((M + M / 16 + 1) & 1) ? (M + M / 16 + 1) : (M + M / 16 + 2);
    LineInfo* linfo = reinterpret_cast<LineInfo*>(smem_raw);
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw + linfo_bytes(p.lines));

    const int tid = threadIdx.x;
    const int Lc = p.lines, logL = p.logLines;
    const int n = p.n;
    const void* __restrict__ W = p.wfft;
    const cx<T>* __restrict__ Wt = reinterpret_cast<const cx<T>*>(p.wt);
    const cx<T>* __restrict__ Ww = reinterpret_cast<const cx<T>*>(p.ww);
    const Geometry& g = p.g;

    // ---- per-line setup
    if (tid < Lc) {
        LineInfo L;
        int ia, ib;
        bool valid;
        if (!STRIDED) {
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
        if (OP == OP_MID) {
            const bool ha = p.s.lam_a != nullptr, hb = p.s.lam_b != nullptr;
            const double la = ha ? p.s.lam_a[ia] : 0.0;
            const double lb = hb ? p.s.lam_b[ib] : 0.0;
            if (ha && p.s.pos_a < p.s.pos_t) before += la;
            if (hb && p.s.pos_b < p.s.pos_t) before += lb;
            if (ha && p.s.pos_a > p.s.pos_t) { a1 = la; nafter = 1; }
            if (hb && p.s.pos_b > p.s.pos_t) { if (nafter == 0) a1 = lb; else a2 = lb; ++nafter; }
        }
        L.before = before; L.after1 = a1; L.after2 = a2; L.nafter = nafter; L.pad = 0;
        linfo[tid] = L;
    }
    __syncthreads();

    const int lf = tid >> LOGTL;          // line-major mapping
    const int jt = tid & (TL - 1);
    const int lio = STRIDED ? (tid & (Lc - 1)) : lf;   // I/O mapping
    const int bio = STRIDED ? (tid >> logL) : jt;
    cx<T>* line_f = sm + lf * LS;
    cx<T>* line_io = sm + lio * LS;
    T* zr_io = reinterpret_cast<T*>(line_io);
    const LineInfo Lio = linfo[lio];
    constexpr bool fwd_in = OP != OP_INV;
    bool bad = false;

    // =============== LOAD (batched: 16 complex / 32 real values per thread in flight)
    {
        cx<T> v[16];
        if (fwd_in && p.fkind != FK_CFFT) {
            const int kind = p.fkind;
            if (!STRIDED) {
                // pairs (x_j, x_{j+1}), j = 2 (bio + TL it)
                if (Lio.valid) {
                    if (p.vec_in) {
                        const cx<T>* src = reinterpret_cast<const cx<T>*>(reinterpret_cast<const T*>(g.in) + Lio.in_off) + bio;
#pragma unroll
                        for (int it = 0; it < 16; ++it) v[it] = src[it * TL];
                    } else {
#pragma unroll
                        for (int it = 0; it < 16; ++it) {
                            const long long off = Lio.in_off + (long long)(2 * (bio + it * TL)) * g.in_st;
                            v[it] = mkc<T>(ld_real<T>(g.in, g.in_type, off), ld_real<T>(g.in, g.in_type, off + g.in_st));
                        }
                    }
                } else {
#pragma unroll
                    for (int it = 0; it < 16; ++it) v[it] = mkc<T>(0, 0);
                }
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int pi = bio + it * TL;
                    T x0 = v[it].x, x1 = v[it].y;
                    if (p.nonfinite) bad |= !(finite_t(x0) && finite_t(x1));
                    if (kind == FK_RFFT) {
                        line_io[P(pi)] = mkc<T>(x0, x1);
                    } else {
                        if (kind == FK_DST2) x1 = -x1;
                        const int pa = pi, pb = n - 1 - pi;  // Makhoul: v_pi = x_j, v_{n-1-pi} = x_{j+1}
                        zr_io[2 * P(pa >> 1) + (pa & 1)] = x0;
                        zr_io[2 * P(pb >> 1) + (pb & 1)] = x1;
                    }
                }
            } else {
                // rows j = bio + TL it, it < 32 (n = 2M rows)
                T xr[32];
                if (Lio.valid) {
                    const long long st = g.in_st;
                    const long long off0 = Lio.in_off + (long long)bio * st;
#pragma unroll
                    for (int it = 0; it < 32; ++it) xr[it] = ld_real<T>(g.in, g.in_type, off0 + (long long)(it * TL) * st);
                } else {
#pragma unroll
                    for (int it = 0; it < 32; ++it) xr[it] = 0;
                }
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int j = bio + it * TL;
                    T x = xr[it];
                    if (p.nonfinite) bad |= !finite_t(x);
                    int pv;
                    if (kind == FK_RFFT) pv = j;
                    else {
                        pv = (j & 1) ? (n - 1 - (j >> 1)) : (j >> 1);
                        if (kind == FK_DST2 && (j & 1)) x = -x;
                    }
                    zr_io[2 * P(pv >> 1) + (pv & 1)] = x;
                }
            }
        } else if (fwd_in || p.ikind == IK_ICFFT || p.ikind == IK_IRFFT) {
            // complex lines in natural order (CFFT forward, ICFFT / IRFFT inverse)
            if (Lio.valid) {
                const long long st = g.in_st;
                const long long off0 = Lio.in_off + (long long)bio * st;
#pragma unroll
                for (int it = 0; it < 16; ++it) v[it] = ld_cx<T>(g.in, g.in_type, off0 + (long long)(it * TL) * st);
            } else {
#pragma unroll
                for (int it = 0; it < 16; ++it) v[it] = mkc<T>(0, 0);
            }
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                if (p.nonfinite) bad |= !(finite_t(v[it].x) && finite_t(v[it].y));
                line_io[P(bio + it * TL)] = v[it];
            }
            if (!fwd_in && p.ikind == IK_IRFFT && bio == 0) {
                // the Nyquist entry k = M of the half spectrum
                cx<T> xm = mkc<T>(0, 0);
                if (Lio.valid) xm = ld_cx<T>(g.in, g.in_type, Lio.in_off + (long long)M * g.in_st);
                if (p.nonfinite) bad |= !(finite_t(xm.x) && finite_t(xm.y));
                line_io[P(M)] = xm;
            }
        } else {
            // DCT-III / DST-III: real spectrum of n = 2M entries
            const bool dst = p.ikind == IK_DST3;
            if (!STRIDED && p.vec_in) {
                if (Lio.valid) {
                    const cx<T>* src = reinterpret_cast<const cx<T>*>(reinterpret_cast<const T*>(g.in) + Lio.in_off) + bio;
#pragma unroll
                    for (int it = 0; it < 16; ++it) v[it] = src[it * TL];
                } else {
#pragma unroll
                    for (int it = 0; it < 16; ++it) v[it] = mkc<T>(0, 0);
                }
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int k = 2 * (bio + it * TL);
                    if (p.nonfinite) bad |= !(finite_t(v[it].x) && finite_t(v[it].y));
                    zr_io[PR(dst ? n - 1 - k : k)] = v[it].x;
                    zr_io[PR(dst ? n - 2 - k : k + 1)] = v[it].y;
                }
            } else {
                // generic: CONTIG rows k = 2(bio + TL it) + {0,1}; STRIDED rows k = bio + TL it
                T xr[32];
                const long long st = g.in_st;
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int k = STRIDED ? (bio + it * TL) : (2 * (bio + (it >> 1) * TL) + (it & 1));
                    xr[it] = Lio.valid ? ld_real<T>(g.in, g.in_type, Lio.in_off + (long long)k * st) : (T)0;
                }
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int k = STRIDED ? (bio + it * TL) : (2 * (bio + (it >> 1) * TL) + (it & 1));
                    if (p.nonfinite) bad |= !finite_t(xr[it]);
                    zr_io[PR(dst ? n - 1 - k : k)] = xr[it];
                }
            }
        }
    }
    if (bad) *p.nonfinite = 1;
    __syncthreads();

    // =============== FORWARD FFT (+ post / mid)
    if constexpr (fwd_in) {
        fft_tile<false, T, LOGM>(line_f, jt, W);

        if constexpr (OP == OP_FWD) {
            const int kind = p.fkind;
            const T om = (T)p.out_mult;
            if (!Lio.valid) return;
            const long long ob = Lio.out_off;
            const long long os = g.out_st;
            if (kind == FK_CFFT) {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int k = bio + it * TL;
                    st_cx<T>(g.out, g.out_type, ob + (long long)k * os, cscale<T>(line_io[P(k)], om));
                }
            } else if (kind == FK_RFFT) {
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int q = bio + it * TL;
                    if (q == 0) {
                        const cx<T> z0 = line_io[P(0)];
                        st_cx<T>(g.out, g.out_type, ob, mkc<T>((z0.x + z0.y) * om, 0));
                        st_cx<T>(g.out, g.out_type, ob + (long long)M * os, mkc<T>((z0.x - z0.y) * om, 0));
                        const cx<T> zh = line_io[P(HALF)];
                        st_cx<T>(g.out, g.out_type, ob + (long long)HALF * os, cscale<T>(rsplit<T>(zh, zh, Wt[HALF]), om));
                    } else {
                        const cx<T> zk = line_io[P(q)], zm = line_io[P(M - q)];
                        const cx<T> tq = Wt[q];
                        st_cx<T>(g.out, g.out_type, ob + (long long)q * os, cscale<T>(rsplit<T>(zk, zm, tq), om));
                        st_cx<T>(g.out, g.out_type, ob + (long long)(M - q) * os, cscale<T>(rsplit<T>(zm, zk, t_mirror<T>(tq)), om));
                    }
                }
            } else {
                const bool dst = kind == FK_DST2;
#define EMIT(K, X) st_real<T>(g.out, g.out_type, ob + (long long)(dst ? (n - 1 - (K)) : (K)) * os, (X) * om)
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int q = bio + it * TL;
                    if (q == 0) {
                        const cx<T> z0 = line_io[P(0)];
                        const cx<T> wM = Ww[M];
                        EMIT(0, (T)2 * (z0.x + z0.y));
                        EMIT(M, (T)2 * (z0.x - z0.y) * wM.x);
                        const cx<T> zh = line_io[P(HALF)];
                        const cx<T> U = cmul<T>(Ww[HALF], rsplit<T>(zh, zh, Wt[HALF]));
                        EMIT(HALF, (T)2 * U.x);
                        EMIT(n - HALF, (T)-2 * U.y);
                    } else {
                        const cx<T> zk = line_io[P(q)], zm = line_io[P(M - q)];
                        const cx<T> tq = Wt[q], wq = Ww[q];
                        const cx<T> U1 = cmul<T>(wq, rsplit<T>(zk, zm, tq));
                        const cx<T> U2 = cmul<T>(w_mirror<T>(wq), rsplit<T>(zm, zk, t_mirror<T>(tq)));
                        EMIT(q, (T)2 * U1.x);
                        EMIT(n - q, (T)-2 * U1.y);
                        EMIT(M - q, (T)2 * U2.x);
                        EMIT(M + q, (T)-2 * U2.y);
                    }
                }
#undef EMIT
            }
            return;
        }

        // ---- OP_MID: post -> capture -> scale -> pre, in place on each quad/pair
        {
            const int kind = p.fkind;
            const Scaling& S = p.s;
            const LineInfo L = linfo[lf];
            const bool cap = S.singular && S.dc_out && L.null_line && L.valid;
            if (kind == FK_CFFT) {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int k = jt + it * TL;
                    const cx<T> X = line_f[P(k)];
                    if (cap && k == 0) *S.dc_out = (double)X.x;
                    line_f[P(k)] = cscale<T>(X, eig_factor<T>(S, L, k));
                }
            } else if (kind == FK_RFFT) {
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int q = jt + it * TL;
                    if (q == 0) {
                        const cx<T> z0 = line_f[P(0)];
                        T x0 = z0.x + z0.y, xM = z0.x - z0.y;
                        if (cap) *S.dc_out = (double)x0;
                        x0 *= eig_factor<T>(S, L, 0);
                        xM *= eig_factor<T>(S, L, M);
                        line_f[P(0)] = mkc<T>(x0 + xM, x0 - xM);
                        const cx<T> zh = line_f[P(HALF)];
                        const cx<T> xh = cscale<T>(rsplit<T>(zh, zh, Wt[HALF]), eig_factor<T>(S, L, HALF));
                        line_f[P(HALF)] = rmerge<T>(xh, xh, Wt[HALF]);
                    } else {
                        const cx<T> zk = line_f[P(q)], zm = line_f[P(M - q)];
                        const cx<T> tq = Wt[q], tm = t_mirror<T>(tq);
                        const cx<T> xk = cscale<T>(rsplit<T>(zk, zm, tq), eig_factor<T>(S, L, q));
                        const cx<T> xm = cscale<T>(rsplit<T>(zm, zk, tm), eig_factor<T>(S, L, M - q));
                        line_f[P(q)] = rmerge<T>(xk, xm, tq);
                        line_f[P(M - q)] = rmerge<T>(xm, xk, tm);
                    }
                }
            } else {
                const bool dst = kind == FK_DST2;
#define KPHYS(K) (dst ? (n - 1 - (K)) : (K))
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int q = jt + it * TL;
                    if (q == 0) {
                        const cx<T> z0 = line_f[P(0)];
                        const cx<T> wM = Ww[M];
                        T X0 = (T)2 * (z0.x + z0.y);
                        T XM = (T)2 * (z0.x - z0.y) * wM.x;
                        if (cap && !dst) *S.dc_out = (double)X0;
                        X0 *= eig_factor<T>(S, L, KPHYS(0));
                        XM *= eig_factor<T>(S, L, KPHYS(M));
                        const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                        line_f[P(0)] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                        const cx<T> zh = line_f[P(HALF)];
                        const cx<T> wh = Ww[HALF], th = Wt[HALF];
                        const cx<T> U = cmul<T>(wh, rsplit<T>(zh, zh, th));
                        const T Xa = (T)2 * U.x * eig_factor<T>(S, L, KPHYS(HALF));
                        const T Xb = (T)-2 * U.y * eig_factor<T>(S, L, KPHYS(n - HALF));
                        const cx<T> Vh = cmulc<T>(mkc<T>(Xa, -Xb), wh);
                        line_f[P(HALF)] = rmerge<T>(Vh, Vh, th);
                    } else {
                        const cx<T> zk = line_f[P(q)], zm = line_f[P(M - q)];
                        const cx<T> tq = Wt[q], tm = t_mirror<T>(tq);
                        const cx<T> wq = Ww[q], wm = w_mirror<T>(wq);
                        const cx<T> U1 = cmul<T>(wq, rsplit<T>(zk, zm, tq));
                        const cx<T> U2 = cmul<T>(wm, rsplit<T>(zm, zk, tm));
                        const T Xq = (T)2 * U1.x * eig_factor<T>(S, L, KPHYS(q));
                        const T Xnq = (T)-2 * U1.y * eig_factor<T>(S, L, KPHYS(n - q));
                        const T Xmq = (T)2 * U2.x * eig_factor<T>(S, L, KPHYS(M - q));
                        const T Xpq = (T)-2 * U2.y * eig_factor<T>(S, L, KPHYS(M + q));
                        const cx<T> Vk = cmulc<T>(mkc<T>(Xq, -Xnq), wq);
                        const cx<T> Vm = cmulc<T>(mkc<T>(Xmq, -Xpq), wm);
                        line_f[P(q)] = rmerge<T>(Vk, Vm, tq);
                        line_f[P(M - q)] = rmerge<T>(Vm, Vk, tm);
                    }
                }
#undef KPHYS
            }
            __syncthreads();
        }
    } else {
        // =============== INVERSE pre-processing (line-major mapping)
        const int ik = p.ikind;
        if (ik == IK_DCT3 || ik == IK_DST3) {
            // two-phase: the real-valued view overlaps the complex slots
            const T* zr = reinterpret_cast<const T*>(line_f);
            cx<T> hold[16];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int q = jt + it * TL;
                if (q == 0) {
                    const T X0 = zr[PR(0)], XM = zr[PR(M)];
                    const cx<T> wM = Ww[M];
                    const cx<T> VM = cmulc<T>(mkc<T>(XM, -XM), wM);
                    hold[2 * it] = rmerge<T>(mkc<T>(X0, 0), VM, mkc<T>(1, 0));
                    const cx<T> wh = Ww[HALF], th = Wt[HALF];
                    const cx<T> Vh = cmulc<T>(mkc<T>(zr[PR(HALF)], -zr[PR(n - HALF)]), wh);
                    hold[2 * it + 1] = rmerge<T>(Vh, Vh, th);
                } else {
                    const cx<T> wq = Ww[q], wm = w_mirror<T>(wq);
                    const cx<T> tq = Wt[q], tm = t_mirror<T>(tq);
                    const cx<T> Vk = cmulc<T>(mkc<T>(zr[PR(q)], -zr[PR(n - q)]), wq);
                    const cx<T> Vm = cmulc<T>(mkc<T>(zr[PR(M - q)], -zr[PR(M + q)]), wm);
                    hold[2 * it] = rmerge<T>(Vk, Vm, tq);
                    hold[2 * it + 1] = rmerge<T>(Vm, Vk, tm);
                }
            }
            __syncthreads();
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int q = jt + it * TL;
                line_f[P(q)] = hold[2 * it];
                line_f[P(q == 0 ? HALF : M - q)] = hold[2 * it + 1];
            }
            __syncthreads();
        } else if (ik == IK_IRFFT) {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int q = jt + it * TL;
                if (q == 0) {
                    const cx<T> x0 = line_f[P(0)], xM = line_f[P(M)];
                    line_f[P(0)] = rmerge<T>(x0, xM, mkc<T>(1, 0));
                    const cx<T> xh = line_f[P(HALF)];
                    line_f[P(HALF)] = rmerge<T>(xh, xh, Wt[HALF]);
                } else {
                    const cx<T> xk = line_f[P(q)], xm = line_f[P(M - q)];
                    line_f[P(q)] = rmerge<T>(xk, xm, Wt[q]);
                    line_f[P(M - q)] = rmerge<T>(xm, xk, t_mirror<T>(Wt[q]));
                }
            }
            __syncthreads();
        }
    }

    // =============== INVERSE FFT + store (INV and MID)
    if constexpr (OP == OP_FWD) return; else {
    fft_tile<true, T, LOGM>(line_f, jt, W);
    if (!Lio.valid) return;
    {
        const int ik = p.ikind;
        const T om = (T)p.out_mult;
        const long long ob = Lio.out_off;
        const long long os = g.out_st;
        if (ik == IK_ICFFT) {
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                const int k = bio + it * TL;
                st_cx<T>(g.out, g.out_type, ob + (long long)k * os, cscale<T>(line_io[P(k)], om));
            }
        } else {
            const bool dct = ik != IK_IRFFT;
            const bool dst = ik == IK_DST3;
            if (!STRIDED) {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int m = bio + it * TL;   // output pair (x_{2m}, x_{2m+1})
                    T x0, x1;
                    if (dct) {
                        const int pa = m, pb = n - 1 - m;
                        x0 = zr_io[2 * P(pa >> 1) + (pa & 1)];
                        x1 = zr_io[2 * P(pb >> 1) + (pb & 1)];
                        if (dst) x1 = -x1;
                    } else {
                        const cx<T> v = line_io[P(m)];
                        x0 = v.x; x1 = v.y;
                    }
                    x0 *= om; x1 *= om;
                    const long long off = ob + (long long)(2 * m) * os;
                    if (p.vec_out) {
                        *reinterpret_cast<cx<T>*>(reinterpret_cast<T*>(g.out) + off) = mkc<T>(x0, x1);
                    } else {
                        st_real<T>(g.out, g.out_type, off, x0);
                        st_real<T>(g.out, g.out_type, off + os, x1);
                    }
                }
            } else {
#pragma unroll
                for (int it = 0; it < 32; ++it) {
                    const int j = bio + it * TL;
                    const int pv = dct ? ((j & 1) ? (n - 1 - (j >> 1)) : (j >> 1)) : j;
                    T x = zr_io[2 * P(pv >> 1) + (pv & 1)];
                    if (dst && (j & 1)) x = -x;
                    st_real<T>(g.out, g.out_type, ob + (long long)j * os, x * om);
                }
            }
        }
    }
    }
}

}  // namespace fpb

#define FP_FFT_PICK(NAME, T, LO, HI)                                                   \
    namespace fpb {                                                                    \
    template <int L, int OPV> static FftKernelFn NAME##_one(bool s) {                  \
        return s ? fft_pass_kernel<T, L, true, OPV> : fft_pass_kernel<T, L, false, OPV>; \
    }                                                                                  \
    template <int L> static FftKernelFn NAME##_rec(int logM, bool s, int op) {         \
        if constexpr (L > HI) { return nullptr; }                                      \
        else {                                                                         \
            if (logM != L) return NAME##_rec<L + 1>(logM, s, op);                      \
            return op == OP_FWD ? NAME##_one<L, OP_FWD>(s)                             \
                 : op == OP_INV ? NAME##_one<L, OP_INV>(s) : NAME##_one<L, OP_MID>(s); \
        }                                                                              \
    }                                                                                  \
    FftKernelFn NAME(int logM, bool s, int op) { return NAME##_rec<LO>(logM, s, op); } \
    }
