// fp_types.h -- pass descriptors shared by the host planner (fp_plan.cu) and
// the sm_100a kernels (fp_kernels.cu).
//
// One Poisson solve is a short list of PASSES over HBM.  A pass transforms
// every line along one axis `t` of a (up to) 3D array; the lines are indexed by
// the two other axes `a` (outer) and `b` (inner).  Three pass ops exist:
//   FWD  forward 1D transform            (solver.py:234-240 for one axis)
//   INV  inverse 1D transform            (solver.py:242-249 for one axis)
//   MID  forward -> eigenvalue scale -> inverse along the last forward axis,
//        with null-mode capture (solver.py:216-223), all on one on-chip tile.
#pragma once
#include <cuda.h>   // CUtensorMap (type only; the maps are encoded through the runtime's driver entry point)
#include <stdint.h>

namespace fpb {

enum PassOp { OP_FWD = 0, OP_INV = 1, OP_MID = 2 };

// Forward / inverse line kinds of the FFT engine (power-of-two lengths).
// DCT2/DST2/RFFT are real-to-real/-complex transforms built around a
// half-length complex FFT (Makhoul reordering + real-FFT untangling).
// DCT-I / DST-I (regular grids, n = 2^k +- 1) run as the half-length real FFT of the
// even / odd extension (2M reals, M = n - 1 or n + 1); a pair's two kinds share a value
enum FwdKind { FK_DCT2 = 0, FK_DST2 = 1, FK_RFFT = 2, FK_CFFT = 3, FK_DCT1 = 4, FK_DST1 = 5 };
enum InvKind { IK_DCT3 = 0, IK_DST3 = 1, IK_IRFFT = 2, IK_ICFFT = 3, IK_DCT1 = 4, IK_DST1 = 5 };

// Dense (direct-summation) engine classes, any length, any kind.
enum DenseClass { DC_R2R = 0, DC_R2C = 1, DC_C2C = 2, DC_C2R = 3 };

// Line-to-thread family: CONTIG = lines are contiguous rows (transform axis is
// the unit-stride axis); STRIDED = lines are columns, W adjacent columns per
// tile so every row segment is a coalesced run.
enum Family { FAM_CONTIG = 0, FAM_STRIDED = 1 };

// element types (match FP_F64.. in the public header)
enum ElemType { ET_F64 = 0, ET_F32 = 1, ET_C128 = 2, ET_C64 = 3 };

struct Geometry {
    int na, nb;                 // extents of the line-index axes (a outer, b inner)
    long long in_st, in_sa, in_sb;    // strides (elements of in_type)
    long long out_st, out_sa, out_sb; // strides (elements of out_type)
    const void* in;
    void* out;
    int in_type, out_type;
    // distributed exchange layout (slab decomposition):
    // element j of a line at (j >> blk_lg) * st_hi + (j & (2^blk_lg - 1)) * st
    // when blk_lg > 0 (the all-to-all's source-rank blocks along axis 0;
    // zero-initialized geometry = plain stride)
    int blk_lg;
    long long in_st_hi, out_st_hi;
    // uneven slabs / any rank count: element j of a line at row_tab[j] (elements;
    // the same table for in and out -- the distributed MID runs in place)
    const long long* row_tab;
    // real view of a complex state (distributed MID of a wall axis 0 after a periodic
    // axis made the state complex): line ib is part (ib & 1) of complex column ib >> 1;
    // strides are in reals, sb steps complex columns, a_/b_ offsets and limits count
    // complex columns
    int pair_b;
    // global index of the line axes = local + off; lines with global >= lim
    // (lim > 0) are padding (not loaded, not stored, no eigenvalue lookup)
    int a_off, a_lim, b_off, b_lim;
};

// Eigenvalue scaling of the middle pass (solver.py:151-159,221).  The factor
// for spectral index (k_t, k_a, k_b) is  bscale / lam  with
// lam = sum over axes in AXIS ORDER of the per-axis tables (eigenvalues.py:104-108),
// and 0 where lam == 0 (the null mode, solver.py:157-158).
struct Scaling {
    const double* lam_t;        // table along the transform axis (n_t entries)
    const double* lam_a;        // table along axis a (nullptr => 0)
    const double* lam_b;        // table along axis b (nullptr => 0)
    int pos_t, pos_a, pos_b;    // axis ids (summation order); -1 = absent axis
    double bscale;              // prod backward_scale (transforms.py:88-96)
    double inv_np;              // 1 / prod n_periodic (solver.py:238-239)
    int singular;
    double* dc_out;             // raw null-mode coefficient sink (or nullptr)
    // folded DCT-II / DST-II MID: (lam_t[KPHYS(q)], lam_t[KPHYS(n-q)]) for q = 0..M, fp64
    // pairs, so one 16-B load serves a quad's (q, n-q) and another its (M-q, M+q)
    const double* lam_pair;
};

// rhs producer of a 2D projection step (flow.py:114-122, 290): the first pass
// computes  rhs[i][j] = ((u[i+1][j] - u[i][j]) / dx + (w[i][j+1] - w[i][j]) / dz) / scale
// (i periodic along axis 0; w has nz + 1 faces with walls, nz when periodic in z)
// from the face arrays while it loads its lines, instead of reading an rhs array
struct Producer {
    const void* u;              // x-faces (nx, nz), plan-typed
    const void* w;              // z-faces (nx, nz) or (nx, nz + 1)
    long long us0, us1, ws0, ws1;   // element strides
    double sx, sz;              // 1 / (dx * scale), 1 / (dz * scale)
    int nx, nz, w_periodic, active;
};

struct FftPass {
    int op, fkind, ikind, family;
    int n;                      // real line length (or complex length for CFFT)
    int M, logM;                // complex FFT length
    int lines;                  // lines per tile (W for STRIDED; pow2)
    int logLines;
    int ls;                     // shared-memory line stride in complex elements
    int tiles;                  // grid size
    int nbt;                    // STRIDED: tiles along b
    int vec_in, vec_out;        // 16-byte vector path allowed (contiguous pairs)
    Geometry g;
    Scaling s;
    const void* wfft;           // M roots  e^{-2 pi i k/M}          (Real2)
    const void* wt;             // M+1 roots e^{-2 pi i k/n}  (real kinds)
    const void* ww;             // M+1 roots e^{-i pi k/(2n)} (DCT/DST)
    const void* wb;             // M+1 roots e^{-5 i pi k/(2n)} = w_k t_k (DCT/DST MID; else nullptr)
    int* nonfinite;             // first pass only
    double out_mult;            // extra output scale (DFT 1/n in TransformPlan)
    Producer prod;              // first pass of a fused projection step (active = 0 otherwise)
    int sub;                    // STRIDED MID: compute sub-tiles per I/O tile (0/1 = one; 2 = the
                                // tile is twice as wide as one 512-thread compute pass)
    // TMA-staged strided pass (fp_tma.cu): tensor maps of the in / out arrays, filled at
    // solve time by tma_prepare; tm_tdim = the map dimension of the transform axis
    int tma, tm_tdim;
    int pf_tiles;               // TMA kernels: L2-prefetch tile blockIdx.x + pf_tiles while this tile computes (0 = off)
    CUtensorMap tm_in, tm_out;
    CUtensorMap tm_aux;         // real-FFT passes: 8-row boxes of the complex half spectrum (row M)
};

struct DensePass {
    int cls;                    // DenseClass
    int n_in, n_out;
    int lines;                  // lines per CTA
    int tiles;
    int in_ls, out_ls;          // smem line strides (reals)
    Geometry g;
    const void* mat;            // [n_out][n_in] Real (R2R) or Real2 (others)
    int* nonfinite;
    double out_mult;
};

// Mixed-radix engine (any n whose FFT length factors into primes <= 61): one
// in-place decimation-in-time FFT of length N per line in shared memory, input
// placed in mixed-radix digit-reversed order.  kind = public FP_* transform id,
// or MR_RFFT / MR_IRFFT (real-input DFT -> half spectrum and back).
//   DFT / IDFT / RFFT / IRFFT: N = n;  DCT2 / DST2 / DCT3 / DST3: N = n (Makhoul
//   reordering + quarter-wave twiddle, any parity);  DCT1: N = 2(n-1) (even
//   extension);  DST1: N = 2(n+1) (odd extension).
constexpr int MR_RFFT = 100, MR_IRFFT = 101;
constexpr int kMrMaxStages = 24;
constexpr int kMrMaxPrime = 61;
struct MrPass {
    int kind;
    int n;                      // line length
    int n_in, n_out;            // elements read / written per line
    int N;                      // complex FFT length
    int inv;                    // FFT direction: 1 = e^{+2 pi i jk/N}
    int cin, cout;              // complex operands
    int nf;                     // stages
    int fac[kMrMaxStages];      // radix per stage (stage 0 first)
    int lines, log_lines;       // lines per CTA (power of two)
    int tiles;
    Geometry g;
    const void* root;           // N roots e^{-2 pi i k/N} (plan precision, complex)
    const void* wq;             // n+1 roots e^{-i pi k/(2n)} (II / III kinds)
    const int* perm;            // digit-reversed position of input index j (N)
    int* nonfinite;
    double out_mult;
    // MID (forward -> eigenvalue scale -> inverse on the tile): ikind = the
    // pair's inverse transform; n_in follows kind, n_out follows ikind
    int mid, ikind;
    Scaling s;
    int half;                   // even n, DCT/DST II-III or real FFT: complex FFT of length N = n/2
    const void* wt;             // half: n/2 + 1 roots e^{-2 pi i k/n}
};

// Bluestein (chirp-z) engine (fp_blue.cu): any line length, any kind -- the axes
// neither the FFT nor the mixed-radix engine takes (a prime factor above 61, or
// lines longer than a CTA's shared memory).  One pass = per chunk of lines:
// gather (recipe x pre-chirp, zero pad to L) -> FFT_L -> x filter spectrum ->
// inverse FFT_L -> emit (post-chirp x output recipe); FFT_L on the FFT engine.
struct BluePass {
    int kind;                   // public FP_* kind, or MR_RFFT / MR_IRFFT
    int n;                      // line length
    int n_out;                  // outputs per line
    int N;                      // DFT length of the recipe: n, 2(n-1) (DCT-I), 2(n+1) (DST-I)
    int L;                      // cyclic convolution length (power of two >= 2N - 1, >= 16)
    int inv;                    // DFT sign of the recipe: 1 = e^{+2 pi i jk/N}
    Geometry g;
    const void* chirp;          // N entries c_m = e^{i pi m^2/N} (plan precision, complex)
    const void* wq;             // n+1 entries e^{-i pi k/(2n)} (II / III kinds; else nullptr)
    int* nonfinite;
    double out_mult;
};

// the projection corrector (flow.py:125-139, 292-295):
//   u -= scale * (phi[i][j] - phi[i-1][j]) / dx,  w -= scale * (phi[i][j] - phi[i][j-1]) / dz
// (wall faces keep w), optionally p += phi; dense C-order (nx, nz) / (nx, nz[+1]) arrays
struct CorrectPass {
    const void* phi;
    const void* u_in;
    const void* w_in;
    void* u_out;
    void* w_out;
    void* p;                    // nullable
    double cx, cz;              // scale / dx, scale / dz
    int nx, nz, w_periodic;
};

struct ScalePass {              // stand-alone eigenvalue scale (dense middle)
    int ndim;
    int ext[3];                 // spectral extents
    long long st[3];            // strides (elements)
    void* data;
    int type;
    const double* lam[3];
    double bscale;
    double inv_np;
    int singular;
    double* dc_out;
    const void* ovr;            // NULL, or the caller's dense factor table (plan precision, C order over ext)
};

struct MeanPass {               // subtract the arithmetic mean (DCT-I plans)
    int ext[3];
    long long st[3];
    void* data;                 // real, plan precision
    double* partials;           // kMeanParts + 1 doubles of workspace
    // distributed plans (slab decomposition): the mean is global --
    //   sum_out != nullptr: only the local sum, into *sum_out (then all-reduced by the caller)
    //   mean_in != nullptr: only the subtraction of (*mean_in) * inv_total
    double* sum_out;
    const double* mean_in;
    double inv_total;
};
constexpr int kMeanParts = 1184;  // 8 x 148 SMs

struct CastPass {               // strided rhs -> dense plan-typed copy
    int ext[3];
    long long st[3];
};

}  // namespace fpb
