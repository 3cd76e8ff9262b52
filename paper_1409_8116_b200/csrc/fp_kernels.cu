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
//   for every other (kind, n) the reference supports (odd n, tiny n, ...):
//   a register-tiled product for lines of 64+ points, a simple one for short
//   lines.  Both tile-exclusive (a CTA owns complete lines), so in-place safe.
#include <cstdlib>
#include <type_traits>

#include "fp_attr.h"
#include "fp_common.cuh"

namespace fpb {

using FftKernelFn = void (*)(const FftPass);
FftKernelFn pick_fft_d_l4(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_d_l6(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_d_l8(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_d_l9(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_d_l11(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_d_l12(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_f_l4(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_f_l6(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_f_l8(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_f_l9(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_f_l11(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_fft_f_l12(int logM, bool strided, int op, bool pipe, int kind);
FftKernelFn pick_wide_f_l11(int op);
FftKernelFn pick_wide_f_l12(int op);
static FftKernelFn pick_wide(int logM, bool f32, int op) {
    if (!f32) return nullptr;
    return logM == 11 ? pick_wide_f_l11(op) : (logM == 12 ? pick_wide_f_l12(op) : nullptr);
}

// ----------------------------------------------------------------------------
// projection step (flow.py:114-139): the divergence as a stand-alone rhs (used when
// the first pass cannot produce it, e.g. a dense-engine z axis) and the corrector
template <typename T>
__global__ void __launch_bounds__(256) divergence_kernel(const Producer q, T* rhs) {
    const long long total = (long long)q.nx * q.nz;
    const T sx = (T)q.sx, sz = (T)q.sz;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < total; e += (long long)gridDim.x * 256) {
        const int i = (int)(e / q.nz), j = (int)(e - (long long)i * q.nz);
        const int ip = (i + 1 == q.nx) ? 0 : i + 1;
        const int jp = (q.w_periodic && j + 1 == q.nz) ? 0 : j + 1;
        const T* u = reinterpret_cast<const T*>(q.u);
        const T* w = reinterpret_cast<const T*>(q.w);
        const T du = __ldg(u + ip * q.us0 + j * q.us1) - __ldg(u + i * q.us0 + j * q.us1);
        const T dw = __ldg(w + i * q.ws0 + jp * q.ws1) - __ldg(w + i * q.ws0 + j * q.ws1);
        rhs[e] = du * sx + dw * sz;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) correct_kernel(const CorrectPass c) {
    const int nwz = c.w_periodic ? c.nz : c.nz + 1;
    const long long nu = (long long)c.nx * c.nz, nw = (long long)c.nx * nwz;
    const T* phi = reinterpret_cast<const T*>(c.phi);
    const T cx = (T)c.cx, cz = (T)c.cz;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < nu + nw; e += (long long)gridDim.x * 256) {
        if (e < nu) {
            const int i = (int)(e / c.nz), j = (int)(e - (long long)i * c.nz);
            const int im = (i == 0) ? c.nx - 1 : i - 1;
            const T ph = __ldg(phi + e);
            reinterpret_cast<T*>(c.u_out)[e] =
                __ldg(reinterpret_cast<const T*>(c.u_in) + e) - cx * (ph - __ldg(phi + (long long)im * c.nz + j));
            if (c.p) reinterpret_cast<T*>(c.p)[e] += ph;
        } else {
            const long long f = e - nu;
            const int i = (int)(f / nwz), j = (int)(f - (long long)i * nwz);
            T g = 0;   // wall faces: zero gradient (Neumann pressure), w stays pinned
            if (c.w_periodic) {
                const int jm = (j == 0) ? c.nz - 1 : j - 1;
                g = __ldg(phi + (long long)i * c.nz + j) - __ldg(phi + (long long)i * c.nz + jm);
            } else if (j > 0 && j < c.nz) {
                g = __ldg(phi + (long long)i * c.nz + j) - __ldg(phi + (long long)i * c.nz + j - 1);
            }
            reinterpret_cast<T*>(c.w_out)[f] = __ldg(reinterpret_cast<const T*>(c.w_in) + f) - cz * g;
        }
    }
}

cudaError_t launch_divergence(const Producer& q, void* rhs, bool f32, cudaStream_t st) {
    long long blocks = ((long long)q.nx * q.nz + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (f32) divergence_kernel<float><<<(int)blocks, 256, 0, st>>>(q, (float*)rhs);
    else divergence_kernel<double><<<(int)blocks, 256, 0, st>>>(q, (double*)rhs);
    return cudaGetLastError();
}

cudaError_t launch_correct(const CorrectPass& c, bool f32, cudaStream_t st) {
    long long blocks = ((long long)c.nx * (2LL * c.nz + 1) + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (f32) correct_kernel<float><<<(int)blocks, 256, 0, st>>>(c);
    else correct_kernel<double><<<(int)blocks, 256, 0, st>>>(c);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// dense engine, long lines: the same product as a register-tiled GEMM.  The CTA
// still owns LT complete lines (staged in shared memory first, so in-place
// passes stay safe); the matrix streams through a padded [JT][KT] shared tile,
// and every thread accumulates KB outputs for all LT lines (the line values are
// warp-wide broadcast reads).  The matrix is read once per LT lines instead of
// once per line.
template <typename T, int CLS, int LT>
__global__ void __launch_bounds__(256) dense_tile_kernel(const DensePass p) {
    constexpr bool CIN = CLS == DC_C2C || CLS == DC_C2R;
    constexpr bool CMAT = CLS != DC_R2R;
    constexpr bool COUT = CLS == DC_C2C || CLS == DC_R2C;
    constexpr int KB = 2, JT = 8, KT = 256 * KB, AS = KT + 1;   // odd row stride: conflict-free staging
    using XE = typename std::conditional<CIN, cx<T>, T>::type;
    using ME = typename std::conditional<CMAT, cx<T>, T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nin = p.n_in, nout = p.n_out;
    XE* xs = reinterpret_cast<XE*>(smem_raw);
    ME* as = reinterpret_cast<ME*>(smem_raw + (((size_t)LT * nin * sizeof(XE) + 15) & ~(size_t)15));
    const Geometry& g = p.g;
    const int tid = threadIdx.x;
    const long long nlines = (long long)g.na * g.nb;
    const long long l0 = (long long)blockIdx.x * LT;
    int nonfinite = 0;
    for (int idx = tid; idx < LT * nin; idx += 256) {
        const int li = idx / nin, j = idx - li * nin;
        const long long l = l0 + li;
        XE v;
        if constexpr (CIN) v = mkc<T>(0, 0); else v = (T)0;
        if (l < nlines) {
            const long long off = (l / g.nb) * g.in_sa + (l % g.nb) * g.in_sb + (long long)j * g.in_st;
            if constexpr (CIN) {
                v = ld_cx<T>(g.in, g.in_type, off);
                if (p.nonfinite && !(finite_t(v.x) && finite_t(v.y))) nonfinite = 1;
            } else {
                v = ld_real<T>(g.in, g.in_type, off);
                if (p.nonfinite && !finite_t(v)) nonfinite = 1;
            }
        }
        xs[idx] = v;
    }
    if (nonfinite) *p.nonfinite = 1;
    const ME* mat = reinterpret_cast<const ME*>(p.mat);
    const T om = (T)p.out_mult;
    for (int k0 = 0; k0 < nout; k0 += KT) {
        T ar[LT][KB], ai[LT][KB];
#pragma unroll
        for (int l = 0; l < LT; ++l)
#pragma unroll
            for (int b = 0; b < KB; ++b) ar[l][b] = ai[l][b] = (T)0;
        for (int j0 = 0; j0 < nin; j0 += JT) {
            __syncthreads();   // (first round: the staged lines; later: the previous matrix tile is consumed)
            for (int idx = tid; idx < KT * JT; idx += 256) {
                const int kk = idx / JT, jj = idx - kk * JT;
                const int k = k0 + kk, j = j0 + jj;
                ME m;
                if constexpr (CMAT) m = mkc<T>(0, 0); else m = (T)0;
                if (k < nout && j < nin) m = __ldg(&mat[(long long)k * nin + j]);
                as[jj * AS + kk] = m;
            }
            __syncthreads();
            const int jn = min(JT, nin - j0);
            for (int jj = 0; jj < jn; ++jj) {
                ME a[KB];
#pragma unroll
                for (int b = 0; b < KB; ++b) a[b] = as[jj * AS + tid + 256 * b];
#pragma unroll
                for (int l = 0; l < LT; ++l) {
                    const XE x = xs[l * nin + j0 + jj];
#pragma unroll
                    for (int b = 0; b < KB; ++b) {
                        if constexpr (CLS == DC_R2R) {
                            ar[l][b] = fma(a[b], x, ar[l][b]);
                        } else if constexpr (CLS == DC_R2C) {
                            ar[l][b] = fma(a[b].x, x, ar[l][b]);
                            ai[l][b] = fma(a[b].y, x, ai[l][b]);
                        } else if constexpr (CLS == DC_C2C) {
                            ar[l][b] = fma(a[b].x, x.x, fma(-a[b].y, x.y, ar[l][b]));
                            ai[l][b] = fma(a[b].x, x.y, fma(a[b].y, x.x, ai[l][b]));
                        } else {   // C2R: Re(sum m_j X_j)
                            ar[l][b] = fma(a[b].x, x.x, fma(-a[b].y, x.y, ar[l][b]));
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int l = 0; l < LT; ++l) {
            const long long ll = l0 + l;
            if (ll >= nlines) break;
            const long long ob = (ll / g.nb) * g.out_sa + (ll % g.nb) * g.out_sb;
#pragma unroll
            for (int b = 0; b < KB; ++b) {
                const int k = k0 + tid + 256 * b;
                if (k >= nout) continue;
                const long long off = ob + (long long)k * g.out_st;
                if constexpr (COUT) st_cx<T>(g.out, g.out_type, off, mkc<T>(ar[l][b] * om, ai[l][b] * om));
                else st_real<T>(g.out, g.out_type, off, ar[l][b] * om);
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
        double f;
        if (p.ovr) {
            // dense _inv_lam override (solver.py:221 `work *= _inv_lam`): the table already
            // carries bscale / lambda and its zeros; only the DFT normalisation is added
            f = (double)reinterpret_cast<const T*>(p.ovr)[idx] * p.inv_np;
        } else {
            double lam = 0.0;
            for (int a = 0; a < p.ndim; ++a) lam += p.lam[a][ks[3 - p.ndim + a]];
            f = lam != 0.0 ? (p.bscale / lam) * p.inv_np : 0.0;
        }
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
    if (threadIdx.x == 0) {
        if (p.sum_out) *p.sum_out = s;          // distributed: local sum only
        else p.partials[nparts] = s / total;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) mean_sub_kernel(const MeanPass p, int nparts) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    T* d = reinterpret_cast<T*>(p.data);
    const T m = p.mean_in ? (T)(*p.mean_in * p.inv_total) : (T)p.partials[nparts];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long off = mean_offset<T>(p, i);
        d[off] = d[off] - m;
    }
}

// ----------------------------------------------------------------------------
// dtype cast of a strided rhs into a dense plan-typed array (solver.py:213's
// np.array(rhs, dtype=work_dtype)); only when the caller's rhs dtype differs
// from the plan precision -- the FFT passes then read plan-typed operands only.
template <typename Ti, typename To>
__global__ void __launch_bounds__(256) cast_kernel(const Ti* __restrict__ in, CastPass p, To* __restrict__ out) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long k2 = i % p.ext[2];
        const long long r = i / p.ext[2];
        const long long k1 = r % p.ext[1];
        const long long k0 = r / p.ext[1];
        out[i] = (To)__ldg(in + k0 * p.st[0] + k1 * p.st[1] + k2 * p.st[2]);
    }
}

cudaError_t launch_cast(const void* in, int in_type, const CastPass& p, void* out, int out_type, cudaStream_t st) {
    const long long total = (long long)p.ext[0] * p.ext[1] * p.ext[2];
    long long blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks < 1) blocks = 1;
    if (in_type == ET_F32 && out_type == ET_F64)
        cast_kernel<float, double><<<(int)blocks, 256, 0, st>>>((const float*)in, p, (double*)out);
    else if (in_type == ET_F64 && out_type == ET_F32)
        cast_kernel<double, float><<<(int)blocks, 256, 0, st>>>((const double*)in, p, (float*)out);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// launchers (host)
// Line stride of a strided tile (complex elements, >= M + M/16 + 1).  With
// TL >= 32 each warp owns one line, so only the strided placement / store
// pattern  lio * LS + 17 b + i  (lio = tid % W, b = tid / W) constrains it:
// E elements fill one 128-byte wavefront (E = 16 for complex fp32, 8 for
// complex fp64), and LS = E/W (mod E) maps the E threads of a wavefront onto
// distinct banks.  Real operands (and short lines) keep the odd stride.
int strided_line_stride(const FftPass& p, bool f32) {
    const int base = p.M + p.M / 16 + 1;
    const int odd = base | 1;
    if (p.family != FAM_STRIDED || p.logM < 9) return odd;
    const bool cin = (p.op == OP_INV) ? (p.ikind == IK_ICFFT || p.ikind == IK_IRFFT) : (p.fkind == FK_CFFT);
    const int E = f32 ? 16 : 8;
    if (!cin || p.lines > E) return odd;
    const int want = (E / p.lines) % E;
    int ls = base;
    while (ls % E != want) ++ls;
    return ls;
}

size_t fft_pass_smem_bytes(const FftPass& p, int real_bytes) {
    return linfo_bytes(p.lines) + (size_t)p.lines * p.ls * 2 * real_bytes;
}

template <typename T>
static FftKernelFn pick_fft(int logM, bool strided, int op, bool pipe, int kind = -1) {
    // kind >= 0 selects the MID specialised on that line kind (strided, non-pipelined)
    using PickFn = FftKernelFn (*)(int, bool, int, bool, int);
    static const PickFn d[14] = {nullptr, nullptr, nullptr, nullptr, pick_fft_d_l4, pick_fft_d_l4, pick_fft_d_l6,
                                 pick_fft_d_l6, pick_fft_d_l8, pick_fft_d_l9, pick_fft_d_l9, pick_fft_d_l11,
                                 pick_fft_d_l12, pick_fft_d_l12};
    static const PickFn f[14] = {nullptr, nullptr, nullptr, nullptr, pick_fft_f_l4, pick_fft_f_l4, pick_fft_f_l6,
                                 pick_fft_f_l6, pick_fft_f_l8, pick_fft_f_l9, pick_fft_f_l9, pick_fft_f_l11,
                                 pick_fft_f_l12, pick_fft_f_l12};
    if (logM < 4 || logM > 13) return nullptr;
    return (sizeof(T) == 8 ? d : f)[logM](logM, strided, op, pipe, kind);
}

// Opt in to the full 227 KB per CTA.  The L1/shared carveout stays the driver's
// choice: forcing max-shared (FP_CARVEOUT=100, experiments only) measured 33 %
// slower on c3 -- the twiddle / eigenvalue tables live in L1.
static cudaError_t allow_smem(const void* fn) {
    if (!fn) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    const char* v = getenv("FP_CARVEOUT");   // percent, or unset = driver default
    if (!v || !*v) return cudaSuccess;
    return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(v));
}

static cudaError_t set_smem_attr_all() {
    cudaError_t e;
    for (int l = 4; l <= 13; ++l)
        for (int s = 0; s < 2; ++s)
            for (int op = 0; op < 3; ++op)
                for (int pp = 0; pp < 2; ++pp) {
                    for (int kind = -1; kind < (op == OP_MID ? 4 : 0); ++kind) {   // (kinds 4, 5 use the runtime MID)
                        if ((e = allow_smem((const void*)pick_fft<double>(l, s, op, pp, kind))) != cudaSuccess) return e;
                        if ((e = allow_smem((const void*)pick_fft<float>(l, s, op, pp, kind))) != cudaSuccess) return e;
                    }
                }
    for (int l = 11; l <= 12; ++l)
        for (int op = 0; op < 3; ++op)
            if ((e = allow_smem((const void*)pick_wide(l, true, op))) != cudaSuccess) return e;
    if ((e = allow_smem((const void*)dense_pass_kernel<double>)) != cudaSuccess) return e;
    if ((e = allow_smem((const void*)dense_pass_kernel<float>)) != cudaSuccess) return e;
    return cudaSuccess;
}
// (once per device: the opt-in belongs to the device context)
static cudaError_t set_smem_attr() {
    static PerDeviceOnce once;
    return once.run(set_smem_attr_all);
}

static int env_flag(const char* name, int dflt) {
    const char* v = getenv(name);
    if (!v || !*v) return dflt;
    return atoi(v);
}

cudaError_t launch_fft_tma(const FftPass& p, cudaStream_t st);

cudaError_t launch_fft_pass(const FftPass& p, bool f32, cudaStream_t st) {
    if (p.tma) return launch_fft_tma(p, st);   // TMA-staged strided pass (fp_tma.cu)
    cudaError_t e = set_smem_attr();
    if (e != cudaSuccess) return e;
    const int threads = p.lines << (p.logM - 4);
    const bool strided = p.family == FAM_STRIDED;
    const int rb = f32 ? 4 : 8;
    // pipelined strided path for long lines (FP_SPIPE=0 disables; FP_SPIPE_MINLOG sets
    // the shortest line): forward / inverse passes on a typed operand, no DST, not
    // the first pass, and only when two tiles of the planned width fit (measured:
    // halving the width or pipelining the fp64-heavy MID step loses)
    static const int use_spipe = env_flag("FP_SPIPE", 1);
    static const int spipe_min = env_flag("FP_SPIPE_MINLOG", 9);   // (instantiated from 9 up)
    const bool cin = (p.op == OP_INV) ? (p.ikind == IK_ICFFT || p.ikind == IK_IRFFT) : (p.fkind == FK_CFFT);
    const int want = cin ? (f32 ? ET_C64 : ET_C128) : (f32 ? ET_F32 : ET_F64);
    const bool dst = (p.op != OP_INV && p.fkind == FK_DST2) || (p.op != OP_FWD && p.ikind == IK_DST3);
    const size_t psmem = 2 * linfo_bytes(p.lines) + 2 * (size_t)p.lines * p.ls * 2 * rb;
    const bool r1 = (p.op == OP_INV ? p.ikind : p.fkind) >= FK_DCT1;   // DCT-I / DST-I: own placement
    if (use_spipe && strided && p.op != OP_MID && p.sub != 2 && p.logM >= spipe_min && !dst && !r1 && p.nonfinite == nullptr &&
        p.g.in_type == want && psmem <= 227 * 1024) {
        FftKernelFn fn = f32 ? pick_fft<float>(p.logM, true, p.op, true) : pick_fft<double>(p.logM, true, p.op, true);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // ... and only where the regular kernel is held to one CTA per SM (with two
        // or more resident CTAs their load / compute phases already overlap)
        FftKernelFn reg = f32 ? pick_fft<float>(p.logM, true, p.op, false) : pick_fft<double>(p.logM, true, p.op, false);
        int reg_per_sm = 0;
        if (reg) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&reg_per_sm, (const void*)reg, threads,
                                                              fft_pass_smem_bytes(p, rb));
        if (fn && reg_per_sm == 1 &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, threads, psmem) == cudaSuccess &&
            per_sm > 0) {
            long long grid = (long long)sms * per_sm;
            if (grid > p.tiles) grid = p.tiles;
            return launch_pass(fn, dim3((unsigned)grid), dim3(threads), psmem, st, p);
        }
    }
    const size_t smem = fft_pass_smem_bytes(p, rb);
    if (p.sub == 2) {
        FftKernelFn w = pick_wide(p.logM, f32, p.op);
        if (!w || !strided) return cudaErrorInvalidValue;
        return launch_pass(w, dim3(p.tiles), dim3(threads / 2), smem, st, p);
    }
    static const int mid_spec = env_flag("FP_MID_KIND_KERNELS", 1);   // 0: one MID kernel for all kinds (A/B)
    const int kind = (p.op == OP_MID && mid_spec) ? p.fkind : -1;
    FftKernelFn fn = f32 ? pick_fft<float>(p.logM, strided, p.op, false, kind)
                         : pick_fft<double>(p.logM, strided, p.op, false, kind);
    if (!fn) return cudaErrorInvalidValue;
    return launch_pass(fn, dim3(p.tiles), dim3(threads), smem, st, p);
}

template <typename T, int CLS, int LT>
static cudaError_t launch_dense_tile_lt(const DensePass& p, size_t smem, long long tiles, cudaStream_t st) {
    cudaError_t e = ensure_smem_attr((const void*)dense_tile_kernel<T, CLS, LT>);
    if (e != cudaSuccess) return e;
    dense_tile_kernel<T, CLS, LT><<<(unsigned)tiles, 256, smem, st>>>(p);
    return cudaGetLastError();
}

template <typename T, int CLS>
static cudaError_t launch_dense_tile(const DensePass& p, cudaStream_t st) {
    const bool cin = CLS == DC_C2C || CLS == DC_C2R;
    const size_t xe = (cin ? 2 : 1) * sizeof(T), me = (CLS != DC_R2R ? 2 : 1) * sizeof(T);
    const size_t as_bytes = (size_t)8 * (512 + 1) * me;
    const long long nlines = (long long)p.g.na * p.g.nb;
    int lt = 8;   // lines per CTA: as many as fit next to the matrix tile
    while (lt > 1 && (((size_t)lt * p.n_in * xe + 15) & ~(size_t)15) + as_bytes > 200 * 1024) lt >>= 1;
    while (lt > 1 && lt / 2 >= nlines) lt >>= 1;
    const size_t smem = (((size_t)lt * p.n_in * xe + 15) & ~(size_t)15) + as_bytes;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    const long long tiles = (nlines + lt - 1) / lt;
    switch (lt) {
        case 8: return launch_dense_tile_lt<T, CLS, 8>(p, smem, tiles, st);
        case 4: return launch_dense_tile_lt<T, CLS, 4>(p, smem, tiles, st);
        case 2: return launch_dense_tile_lt<T, CLS, 2>(p, smem, tiles, st);
        default: return launch_dense_tile_lt<T, CLS, 1>(p, smem, tiles, st);
    }
}

template <typename T>
static cudaError_t launch_dense_tile_cls(const DensePass& p, cudaStream_t st) {
    switch (p.cls) {
        case DC_R2R: return launch_dense_tile<T, DC_R2R>(p, st);
        case DC_R2C: return launch_dense_tile<T, DC_R2C>(p, st);
        case DC_C2C: return launch_dense_tile<T, DC_C2C>(p, st);
        default: return launch_dense_tile<T, DC_C2R>(p, st);
    }
}

cudaError_t launch_dense_pass(const DensePass& p, bool f32, cudaStream_t st) {
    cudaError_t e = set_smem_attr();
    if (e != cudaSuccess) return e;
    static const int tile_min = [] { const char* v = getenv("FP_DENSE_TILE_MIN"); return (v && *v) ? atoi(v) : 64; }();
    if (p.n_in >= tile_min) return f32 ? launch_dense_tile_cls<float>(p, st) : launch_dense_tile_cls<double>(p, st);
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
    const bool reduce = p.mean_in == nullptr, sub = p.sum_out == nullptr;
    if (f32) {
        if (reduce) mean_partial_kernel<float><<<nb, 256, 0, st>>>(p);
        if (reduce) mean_final_kernel<float><<<1, 256, 0, st>>>(p, nb);
        if (sub) mean_sub_kernel<float><<<nb, 256, 0, st>>>(p, nb);
    } else {
        if (reduce) mean_partial_kernel<double><<<nb, 256, 0, st>>>(p);
        if (reduce) mean_final_kernel<double><<<1, 256, 0, st>>>(p, nb);
        if (sub) mean_sub_kernel<double><<<nb, 256, 0, st>>>(p, nb);
    }
    return cudaGetLastError();
}

}  // namespace fpb
