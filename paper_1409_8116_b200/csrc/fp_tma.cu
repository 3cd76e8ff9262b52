// fp_tma.cu -- instances and host side of the TMA-staged strided passes (fp_tma.cuh):
// eligibility, the tensor maps (cuTensorMapEncodeTiled through the runtime's driver
// entry point; no libcuda link), and the launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "fp_attr.h"
#include "fp_tma.cuh"

namespace fpb {

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeFn) nullptr;
        return (EncodeFn)f;
    }();
    return fn;
}

bool tma_enabled() {
    static const bool on = [] { const char* v = std::getenv("FP_TMA"); return !(v && *v == '0'); }();
    return on;
}

// 3D map over (columns b [stride 1], transform axis, a axis) of an fp64 array (complex:
// two doubles per column); dims 1 / 2 ordered by stride (tdim = the transform axis' dim).
// Box: `cols` doubles x `rows` rows traversed at `estride` (PHASE / PAIR staging: 4 / 2).
bool encode(CUtensorMap* map, const void* base, long long ncols, long long nt, long long na, long long st_bytes,
            long long sa_bytes, int cols, int rows, int estride, CUtensorMapSwizzle swz, int* tdim) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const bool t_first = st_bytes <= sa_bytes || na <= 1;
    cuuint64_t dims[3] = {(cuuint64_t)ncols, (cuuint64_t)(t_first ? nt : na), (cuuint64_t)(t_first ? na : nt)};
    cuuint64_t strides[2] = {(cuuint64_t)(t_first ? st_bytes : sa_bytes), (cuuint64_t)(t_first ? sa_bytes : st_bytes)};
    if (na <= 1) strides[1] = strides[0] * (cuuint64_t)nt;   // (a dummy axis: any consistent stride)
    cuuint32_t box[3] = {(cuuint32_t)cols, 1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const int td = t_first ? 1 : 2;
    box[td] = (cuuint32_t)rows;
    es[td] = (cuuint32_t)estride;
    *tdim = td;
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool encode_real(CUtensorMap* map, const void* base, long long nb, long long nt, long long na, long long st,
                 long long sa, bool phase, int* tdim) {
    return encode(map, base, nb, nt, na, st * 8, sa * 8, 16, 256, phase ? 4 : 1, CU_TENSOR_MAP_SWIZZLE_128B, tdim);
}

// per-op variant (FP_TMA_FWD / FP_TMA_INV / FP_TMA_MID): 0 = regular kernel, 1 = the
// between-FFT step in registers + warp shuffles, 2 = through the shared-memory tile
// (fewer registers, more resident CTAs)
int env_mode(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}
int tma_mode(int op) {
    static const int m[3] = {env_mode("FP_TMA_FWD", 2), env_mode("FP_TMA_INV", 1), env_mode("FP_TMA_MID", 1)};
    return m[op];
}

template <int LOGM>
FftKernelFn tma_kernel(const FftPass& p) {
    const bool sm = tma_mode(p.op) == 2;
    if (p.op == OP_FWD) return sm ? fft_pass_tma<LOGM, OP_FWD, true> : fft_pass_tma<LOGM, OP_FWD>;
    if (p.op == OP_INV) return sm ? fft_pass_tma<LOGM, OP_INV, true> : fft_pass_tma<LOGM, OP_INV>;
    if (p.fkind == FK_DST2) return sm ? fft_pass_tma<LOGM, mid_op(FK_DST2), true> : fft_pass_tma<LOGM, mid_op(FK_DST2)>;
    return sm ? fft_pass_tma<LOGM, mid_op(FK_DCT2), true> : fft_pass_tma<LOGM, mid_op(FK_DCT2)>;
}

int sm_count_cached() {
    static int cnt[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    int& c = cnt[dev & 63];
    if (c == 0) {
        int v = 0;
        c = (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) ? v : 148;
    }
    return c;
}

// L2 prefetch distance (FP_TMA_PF_FWD / _INV / _MID, in tiles per SM; defaults 0 / 2 / 0): a CTA
// prefetches the input of tile blockIdx.x + distance x #SMs into L2.  At two CTAs per SM a
// distance of 2 is one resident wave ahead: the tile the CTA that replaces this one will load.
// Measured on c3 (profiles/r02/ab_l2_prefetch.txt): the inverse pass (two CTAs per SM, exposed
// load latency) gains 10 %; the forward pass (three CTAs per SM, already at 94 % of the copy
// bandwidth) and the MID lose at every distance.
int pf_distance(int op) {
    // (percent of the SM count)
    static const int w[3] = {env_mode("FP_TMA_PF_FWD", 100), env_mode("FP_TMA_PF_INV", 100), env_mode("FP_TMA_PF_MID", 0)};   // PassOp order
    return w[op] > 0 ? (w[op] * sm_count_cached() + 50) / 100 : 0;
}

FftKernelFn tma_kernel_for(const FftPass& p) {
    switch (p.logM) {
        case 7: return tma_kernel<7>(p);
        case 8: return tma_kernel<8>(p);
        default: return nullptr;
    }
}

}  // namespace

// fills p.tm_in / p.tm_out and sets p.tma when the pass runs on the TMA kernel:
// fp64 DCT-II / DST-II forward, DCT-III / DST-III inverse, or their MID, strided
// over 16 adjacent columns (128-B rows) of plan-typed operands with 16-B aligned
// rows, M = 128 or 256 (one 128-B row segment per line per tile)
// real-FFT passes (c4's y axis): fp64, M = 512, 8 columns (64-B real rows, 128-B complex rows)
static bool tma_prepare_rfft(FftPass& p) {
    const Geometry& g = p.g;
    const bool fwd = p.op == OP_FWD && p.fkind == FK_RFFT;
    const bool inv = p.op == OP_INV && p.ikind == IK_IRFFT;
    if (!(fwd || inv) || p.lines != 8 || p.logM != 9) return false;
    if (g.blk_lg > 0 || g.row_tab || g.pair_b || g.a_lim > 0 || g.b_lim > 0 || p.prod.active) return false;
    const int rt = fwd ? g.in_type : g.out_type, ct = fwd ? g.out_type : g.in_type;
    if (rt != ET_F64 || ct != ET_C128) return false;
    if ((g.nb > 1 && (g.in_sb != 1 || g.out_sb != 1)) || g.nb < 1) return false;
    const long long rst = fwd ? g.in_st : g.out_st, rsa = fwd ? g.in_sa : g.out_sa;   // real operand (doubles)
    const long long cst = fwd ? g.out_st : g.in_st, csa = fwd ? g.out_sa : g.in_sa;   // complex operand (complex)
    if ((rst * 8) % 16 || (g.na > 1 && (rsa * 8) % 16)) return false;
    if (((uintptr_t)g.in % 16) || ((uintptr_t)g.out % 16)) return false;
    const void* rbase = fwd ? g.in : g.out;
    const void* cbase = fwd ? g.out : g.in;
    const long long M = p.M;
    int td_r = 0, td_c = 0, td_a = 0;
    CUtensorMap* rmap = fwd ? &p.tm_in : &p.tm_out;
    CUtensorMap* cmap = fwd ? &p.tm_out : &p.tm_in;
    if (!encode(rmap, rbase, g.nb, 2 * M, g.na, rst * 8, rsa * 8, 8, 256, 2, CU_TENSOR_MAP_SWIZZLE_64B, &td_r)) return false;
    if (!encode(cmap, cbase, 2 * g.nb, M + 1, g.na, cst * 16, csa * 16, 16, 256, 1, CU_TENSOR_MAP_SWIZZLE_128B, &td_c)) return false;
    if (!encode(&p.tm_aux, cbase, 2 * g.nb, M + 1, g.na, cst * 16, csa * 16, 16, 8, 1, CU_TENSOR_MAP_SWIZZLE_128B, &td_a)) return false;
    if (td_r != td_c || td_c != td_a) return false;
    p.tm_tdim = td_r;
    p.tma = 2;
    return true;
}

// complex-line MID (c4's x axis): fp64, M = 1024, 4 columns (64-B rows)
static bool tma_prepare_cmid(FftPass& p) {
    const Geometry& g = p.g;
    if (p.op != OP_MID || p.fkind != FK_CFFT || p.lines != 4 || p.logM != 10 || p.sub == 2) return false;
    if (g.blk_lg > 0 || g.row_tab || g.pair_b || g.a_lim > 0 || g.b_lim > 0 || p.prod.active) return false;
    if (g.in_type != ET_C128 || g.out_type != ET_C128) return false;
    if ((g.nb > 1 && (g.in_sb != 1 || g.out_sb != 1)) || g.nb < 1) return false;
    if (((uintptr_t)g.in % 16) || ((uintptr_t)g.out % 16)) return false;
    int td_i = 0, td_o = 0;
    if (!encode(&p.tm_in, g.in, 2 * g.nb, p.M, g.na, g.in_st * 16, g.in_sa * 16, 8, 256, 1, CU_TENSOR_MAP_SWIZZLE_64B, &td_i)) return false;
    if (!encode(&p.tm_out, g.out, 2 * g.nb, p.M, g.na, g.out_st * 16, g.out_sa * 16, 8, 256, 1, CU_TENSOR_MAP_SWIZZLE_64B, &td_o)) return false;
    if (td_i != td_o) return false;
    p.tm_tdim = td_i;
    p.tma = 3;
    return true;
}

// contiguous DCT / DST lines (c3's z passes): fp64, n = 512, 2 lines per CTA
static bool encode_lines(CUtensorMap* map, const void* base, long long n, long long nb, long long na, long long sb,
                         long long sa, int lines) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {16, (cuuint64_t)(n / 16), (cuuint64_t)nb, (cuuint64_t)(na < 1 ? 1 : na)};
    cuuint64_t strides[3] = {128, (cuuint64_t)(sb * 8), (cuuint64_t)(na > 1 ? sa * 8 : sb * 8 * nb)};
    cuuint32_t box[4] = {16, (cuuint32_t)(n / 16), (cuuint32_t)lines, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool tma_prepare_z(FftPass& p) {
    const Geometry& g = p.g;
    const bool fwd = p.op == OP_FWD && (p.fkind == FK_DCT2 || p.fkind == FK_DST2);
    const bool inv = p.op == OP_INV && (p.ikind == IK_DCT3 || p.ikind == IK_DST3);
    if (!(fwd || inv) || p.logM != 8 || p.lines != 2 || p.family != FAM_CONTIG) return false;
    if (g.blk_lg > 0 || g.row_tab || g.pair_b || g.a_lim > 0 || g.b_lim > 0 || p.prod.active) return false;
    if (g.in_type != ET_F64 || g.out_type != ET_F64 || g.in_st != 1 || g.out_st != 1) return false;
    if (g.nb % p.lines || (long long)g.na * g.nb > 0x7fffffffLL) return false;
    auto ok16 = [](long long s) { return (s * 8) % 16 == 0; };
    if ((g.nb > 1 && (!ok16(g.in_sb) || !ok16(g.out_sb))) || (g.na > 1 && (!ok16(g.in_sa) || !ok16(g.out_sa)))) return false;
    if (((uintptr_t)g.in % 16) || ((uintptr_t)g.out % 16)) return false;
    const long long n = 2LL * p.M;
    if (!encode_lines(&p.tm_in, g.in, n, g.nb, g.na, g.in_sb, g.in_sa, p.lines)) return false;
    if (!encode_lines(&p.tm_out, g.out, n, g.nb, g.na, g.out_sb, g.out_sa, p.lines)) return false;
    p.tma = 5;
    return true;
}

bool tma_prepare(FftPass& p, bool f32) {
    p.tma = 0;
    static const bool z_on = env_mode("FP_TMA_Z", 1) != 0;
    if (tma_enabled() && !f32 && z_on && tma_prepare_z(p)) return true;
    static const bool cmid_on = env_mode("FP_TMA_CMID", 1) != 0;
    if (tma_enabled() && !f32 && p.family == FAM_STRIDED && cmid_on && tma_prepare_cmid(p)) return true;
    static const bool rfft_on = env_mode("FP_TMA_RFFT", 1) != 0;
    if (tma_enabled() && !f32 && p.family == FAM_STRIDED && rfft_on && tma_prepare_rfft(p)) return true;
    if (!tma_enabled() || f32 || p.family != FAM_STRIDED || p.lines != 16 || (p.logM != 7 && p.logM != 8)) return false;
    if (tma_mode(p.op) == 0) return false;
    const bool real_fwd = p.fkind == FK_DCT2 || p.fkind == FK_DST2;
    const bool real_inv = p.ikind == IK_DCT3 || p.ikind == IK_DST3;
    if ((p.op == OP_FWD && !real_fwd) || (p.op == OP_INV && !real_inv) || (p.op == OP_MID && !real_fwd)) return false;
    const Geometry& g = p.g;
    if (g.blk_lg > 0 || g.row_tab || g.pair_b || g.a_lim > 0 || g.b_lim > 0 || p.prod.active) return false;
    if (g.in_type != ET_F64 || g.out_type != ET_F64) return false;
    if ((g.nb > 1 && (g.in_sb != 1 || g.out_sb != 1)) || g.nb < 1) return false;
    auto ok16 = [](long long s) { return (s * 8) % 16 == 0; };
    if (!ok16(g.in_st) || !ok16(g.out_st) || (g.na > 1 && (!ok16(g.in_sa) || !ok16(g.out_sa)))) return false;
    if (((uintptr_t)g.in % 16) || ((uintptr_t)g.out % 16)) return false;
    const long long nreal = 2LL * p.M;
    int td_in = 0, td_out = 0;
    const bool phase_in = p.op != OP_INV, phase_out = p.op != OP_FWD;
    if (!encode_real(&p.tm_in, g.in, g.nb, nreal, g.na, g.in_st, g.in_sa, phase_in, &td_in)) return false;
    if (!encode_real(&p.tm_out, g.out, g.nb, nreal, g.na, g.out_st, g.out_sa, phase_out, &td_out)) return false;
    if (td_in != td_out) return false;
    int td_aux = 0;   // NATURAL view of the input for the L2 prefetch of a later tile
    if (!encode_real(&p.tm_aux, g.in, g.nb, nreal, g.na, g.in_st, g.in_sa, false, &td_aux) || td_aux != td_in) return false;
    p.tm_tdim = td_in;
    p.tma = 1;
    return true;
}

cudaError_t launch_fft_tma(const FftPass& p, cudaStream_t st) {
    if (p.tma == 5) {   // contiguous DCT / DST lines
        FftKernelFn fn = p.op == OP_FWD ? fft_pass_tma_z<8, OP_FWD> : fft_pass_tma_z<8, OP_INV>;
        const size_t tile = (size_t)p.lines * Shape<8>::LS * 16, sb = (size_t)p.lines * 2 * p.M * 8;
        const size_t smem = linfo_bytes(p.lines) + 1024 + (tile > sb ? tile : sb) + 16;
        const cudaError_t e = ensure_smem_attr((const void*)fn);
        if (e != cudaSuccess) return e;
        return launch_pass(fn, dim3(p.tiles), dim3(p.lines << (p.logM - 4)), smem, st, p);
    }
    if (p.tma == 3) {   // complex-line MID
        FftKernelFn fn = fft_pass_tma_c<10>;
        const size_t tile = (size_t)p.lines * p.ls * 16, cstg = (size_t)p.M * 64;
        const size_t smem = linfo_bytes(p.lines) + 1024 + (tile > cstg ? tile : cstg) + 16;
        const cudaError_t e = ensure_smem_attr((const void*)fn);
        if (e != cudaSuccess) return e;
        return launch_pass(fn, dim3(p.tiles), dim3(p.lines << (p.logM - 4)), smem, st, p);
    }
    if (p.tma == 2) {   // real-FFT lines
        FftKernelFn fn = p.op == OP_FWD ? fft_pass_tma_r<9, OP_FWD> : fft_pass_tma_r<9, OP_INV>;
        const size_t tile = (size_t)p.lines * p.ls * 16, cstg = (size_t)(p.M + 8) * 128;
        const size_t smem = linfo_bytes(p.lines) + 1024 + (tile > cstg ? tile : cstg) + 16;
        const cudaError_t e = ensure_smem_attr((const void*)fn);
        if (e != cudaSuccess) return e;
        FftPass q = p;
        q.pf_tiles = pf_distance(p.op);
        return launch_pass(fn, dim3(p.tiles), dim3(p.lines << (p.logM - 4)), smem, st, q);
    }
    FftKernelFn fn = tma_kernel_for(p);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = tma_smem_bytes(p, (size_t)(2 * p.M) * 128);
    const cudaError_t e = ensure_smem_attr((const void*)fn);
    if (e != cudaSuccess) return e;
    const int threads = p.lines << (p.logM - 4);
    FftPass q = p;
    q.pf_tiles = pf_distance(p.op);
    return launch_pass(fn, dim3(p.tiles), dim3(threads), smem, st, q);
}

}  // namespace fpb
