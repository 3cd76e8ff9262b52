// fp_plan.cu -- plan construction, pass scheduling and the C ABI
// (include/fastpoisson_b200.h).
//
// Reference behaviour mirrored here:
//   SolverConfig validation          solver.py:73-91, grid.py:64-78
//   pair table / backward scales     transforms.py:88-125
//   eigenvalue tables                eigenvalues.py:51-83
//   null-mode bookkeeping            solver.py:56-62,177-181,218-220
//   solve pipeline                   solver.py:191-249
// The pipeline is re-planned for HBM: real axes first (contiguous axis first),
// then the periodic axes (the first one as a real FFT -> half spectrum), and
// the LAST forward axis runs as one fused MID pass (forward, scale, inverse).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fastpoisson_b200.h"
#include "fp_tables.h"
#include "fp_types.h"

namespace fpb {
cudaError_t launch_fft_pass(const FftPass& p, bool f32, cudaStream_t st);
cudaError_t launch_dense_pass(const DensePass& p, bool f32, cudaStream_t st);
cudaError_t launch_mr_pass(const MrPass& p, bool f32, cudaStream_t st);
size_t mr_smem_bytes(const MrPass& p, bool f32);
cudaError_t launch_scale_pass(const ScalePass& p, bool f32, cudaStream_t st);
cudaError_t launch_mean_pass(const MeanPass& p, bool f32, cudaStream_t st);
cudaError_t launch_cast(const void* in, int in_type, const CastPass& p, void* out, int out_type, cudaStream_t st);
size_t fft_pass_smem_bytes(const FftPass& p, int real_bytes);
int strided_line_stride(const FftPass& p, bool f32);
cudaError_t launch_divergence(const Producer& q, void* rhs, bool f32, cudaStream_t st);
cudaError_t launch_correct(const CorrectPass& c, bool f32, cudaStream_t st);
bool tma_prepare(FftPass& p, bool f32);
cudaError_t launch_blue_gather(const BluePass& p, void* S, long long l0, long long cl, bool f32, cudaStream_t st);
cudaError_t launch_blue_emit(const BluePass& p, const void* S, long long l0, long long cl, bool f32, cudaStream_t st);
cudaError_t launch_blue_mul(void* S, const void* bhat, long long cl, int L, bool f32, cudaStream_t st);
cudaError_t launch_blue_twiddle(void* S, long long cl, int L1, int L2, int inv, bool f32, cudaStream_t st);
cudaError_t launch_blue_filter(void* S, const void* chirp, int N, int L, int conj, bool f32, cudaStream_t st);
cudaError_t launch_blue_scale(void* dst, const void* S, int L, double s, bool f32, cudaStream_t st);
}  // namespace fpb

using namespace fpb;

static thread_local std::string g_err;
static fp_status fail(fp_status st, const std::string& msg) {
    g_err = msg;
    return st;
}
#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(FP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

namespace {

enum Buf { B_RHS = 0, B_OUT = 1, B_RS = 2, B_CW = 3, B_X = 4 };  // B_X: caller's exchange buffer (distributed)
enum Engine { EN_FFT = 0, EN_DENSE = 1, EN_SCALE = 2, EN_MR = 3, EN_BLUE = 4 };
enum Layout { LY_REAL = 0, LY_CPLX = 1 };  // state of the data in the buffer

struct DevTables {
    void* wfft = nullptr;
    void* wt = nullptr;
    void* ww = nullptr;
    void* wb = nullptr;     // folded DCT-II / DST-II MID twiddle (fp_tables.h mid_table)
    void* lam2 = nullptr;   // folded MID eigenvalue pairs (Scaling::lam_pair)
    void* mat_f = nullptr;  // dense forward
    void* mat_b = nullptr;  // dense backward
    int fwd_nout = 0, fwd_nin = 0, bwd_nout = 0, bwd_nin = 0;
    bool fwd_cpx = false, bwd_cpx = false;
    // mixed-radix engine (fp_mr.cu): one FFT length for both directions of a pair
    bool mr = false;
    int mrN = 0;
    bool mr_half = false;   // half-length recipes (even n, II/III kinds and the real FFT)
    void* mr_wt = nullptr;
    int fwd_kind = 0, bwd_kind = 0;
    std::vector<int> fac;
    void* mr_root = nullptr;
    void* mr_wq = nullptr;
    void* mr_perm = nullptr;
    // Bluestein engine (fp_blue.cu): one DFT length N and one convolution length L
    // (= L1 x L2 four-step when L exceeds the FFT engine's 8192 points) per pair
    bool blue = false;
    int bN = 0, bL = 0, bL1 = 1, bL2 = 0;
    void* b_chirp = nullptr;
    void* b_wq = nullptr;
    void* b_bhat_m = nullptr;   // FFT_L of the chirp filter / L (DFT sign -)
    void* b_bhat_p = nullptr;   // ... of its conjugate (sign +)
    void* b_w1 = nullptr;       // FFT-engine stage twiddles for M = L1 (four-step only)
    void* b_w2 = nullptr;       // ... for M = L2 (= L without the four-step)
};

struct PassT {
    int engine;
    int phase;           // 0 forward, 1 diagonal, 2 backward
    int t;               // transform axis (-1 for scale)
    int in_buf, out_buf;
    int in_layout, out_layout;
    FftPass fp;
    DensePass dp;
    MrPass mp;
    ScalePass sp;
    BluePass bp;
    int a, b;            // other axes (-1 = dummy)
    bool dist_mid;       // MID over the all-to-all receive layout (blocked axis 0)
};

// strides per axis for a buffer state (elements)
struct Strides {
    long long s[3];
};

}  // namespace

struct fp_plan {
    int device = 0;
    fp_config cfg{};
    int ndim = 0;
    bool f32 = false;
    bool singular = false;
    bool mixed = false;
    int periodic_mask = 0;
    int r_axis = -1;          // periodic axis transformed as real FFT (half spectrum)
    int middle = -1;
    int fft_mask = 0;
    long long n[3] = {1, 1, 1};
    long long cext[3] = {1, 1, 1};   // complex-state extents (r axis = n/2+1)
    long long cpitch_last = 1;       // padded contiguous extent of the complex buffer
    bool need_cw = false, need_rs = false;
    bool mean_fix = false;           // exact arithmetic-mean removal (DCT-I axes)
    // slab decomposition along axis 0
    int nranks = 1, rank = 0;
    long long a0 = 0;                // planes of this rank
    long long A = 0;                 // plane pitch of the exchange blocks (max planes per rank)
    bool wall0_cpx = false;          // wall axis 0 after a complex local state: real-view MID
    const long long* row_tab = nullptr;   // uneven slabs / non-power-of-two pitch: MID row table
    long long E1 = 0, B = 0;         // exchanged extent of axis 1 (padded to P) and per-peer block
    long long e1 = 0, e2 = 1;        // true extents of axes 1, 2 in the exchanged state
    bool x_cpx = false;              // exchanged state complex?
    long long xs[3] = {0, 0, 0};     // exchange-buffer strides (send layout: axis 1 outermost)
    double bscale = 1.0;
    double np_prod = 1.0;
    double null_scale = 1.0;
    size_t blue_bytes = 0;           // Bluestein scratch (workspace), max over the passes
    std::vector<PassT> passes;
    std::vector<PassT> passes_ovr;   // middle axis split around a dense _inv_lam scale (override solves)
    bool need_cw_ovr = false;
    DevTables tab[3];
    double* d_lam[3] = {nullptr, nullptr, nullptr};       // per-axis eigenvalue tables
    double* d_lam_pad[3] = {nullptr, nullptr, nullptr};   // the same, from the leading pad entry
    std::vector<void*> allocs;
    ~fp_plan() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (void* p : allocs) cudaFree(p);
        cudaSetDevice(prev);
    }
};

struct fp_transform {
    int device = 0;
    int kind = 0;
    long long n = 0;
    bool f32 = false;
    bool fft = false;
    int M = 0;
    DevTables tab;
    std::vector<void*> allocs;
    ~fp_transform() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (void* p : allocs) cudaFree(p);
        cudaSetDevice(prev);
    }
};

namespace {

// NVTX ranges (header-only NVTX v3; no-ops unless a profiler is attached): one per
// solve / phase call and one per pass, named after the pass (ncu --nvtx filters on them)
struct NvtxRange {
    explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    const int x = std::atoi(v);
    return x > 0 ? x : dflt;
}

int ilog2(long long x) { int l = 0; while ((1LL << l) < x) ++l; return l; }

// upload a long double table rounded to the plan precision (complex pairs or reals)
template <typename AllocT>
fp_status upload(AllocT& allocs, const std::vector<double>& v, bool f32, void** out) {
    *out = nullptr;
    if (v.empty()) return FP_OK;
    const size_t cnt = v.size();
    void* d = nullptr;
    if (f32) {
        std::vector<float> h(cnt);
        for (size_t i = 0; i < cnt; ++i) h[i] = (float)v[i];
        CUDA_TRY(cudaMalloc(&d, cnt * sizeof(float)));
        allocs.push_back(d);
        CUDA_TRY(cudaMemcpy(d, h.data(), cnt * sizeof(float), cudaMemcpyHostToDevice));
    } else {
        CUDA_TRY(cudaMalloc(&d, cnt * sizeof(double)));
        allocs.push_back(d);
        CUDA_TRY(cudaMemcpy(d, v.data(), cnt * sizeof(double), cudaMemcpyHostToDevice));
    }
    *out = d;
    return FP_OK;
}
template <typename AllocT>
fp_status upload(AllocT& allocs, const std::vector<long double>& v, bool f32, void** out) {
    *out = nullptr;
    if (v.empty()) return FP_OK;
    const size_t cnt = v.size();
    void* d = nullptr;
    if (f32) {
        std::vector<float> h(cnt);
        for (size_t i = 0; i < cnt; ++i) h[i] = (float)v[i];
        CUDA_TRY(cudaMalloc(&d, cnt * sizeof(float)));
        allocs.push_back(d);
        CUDA_TRY(cudaMemcpy(d, h.data(), cnt * sizeof(float), cudaMemcpyHostToDevice));
    } else {
        std::vector<double> h(cnt);
        for (size_t i = 0; i < cnt; ++i) h[i] = (double)v[i];
        CUDA_TRY(cudaMalloc(&d, cnt * sizeof(double)));
        allocs.push_back(d);
        CUDA_TRY(cudaMemcpy(d, h.data(), cnt * sizeof(double), cudaMemcpyHostToDevice));
    }
    *out = d;
    return FP_OK;
}

template <typename AllocT>
fp_status upload_ints(AllocT& allocs, const std::vector<int>& v, void** out) {
    *out = nullptr;
    void* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, v.size() * sizeof(int)));
    allocs.push_back(d);
    CUDA_TRY(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    *out = d;
    return FP_OK;
}

// complex FFT length of a mixed-radix line of transform `kind` (FP_* id, or
// MR_RFFT / MR_IRFFT); 0 if the length has no mixed-radix plan in this build
// complex FFT length of the half-length recipe (0: none): n/2 for even-n II/III
// kinds and the real FFT; n - 1 / n + 1 (half the type-I extension) for DCT-I / DST-I
long long mr_half_length(int kind, long long n) {
    static const bool on = [] { const char* v = std::getenv("FP_MR_HALF"); return !(v && *v == '0'); }();
    if (!on) return 0;
    long long h = 0;
    if (kind == FP_DCT2 || kind == FP_DST2 || kind == FP_DCT3 || kind == FP_DST3 || kind == MR_RFFT || kind == MR_IRFFT)
        h = (n % 2 == 0) ? n / 2 : 0;
    else if (kind == FP_DCT1) h = n - 1;
    else if (kind == FP_DST1) h = n + 1;
    if (h < 8 || mr_factors(h, kMrMaxPrime).empty()) return 0;
    return h;
}
bool mr_half_kind(int kind, long long n) { return mr_half_length(kind, n) > 0; }

long long mr_length(int kind, long long n, bool f32) {
    static const bool on = [] { const char* v = std::getenv("FP_MR"); return !(v && *v == '0'); }();
    if (!on || n < 16) return 0;   // short lines: the dense engine
    long long N = n;
    if (kind == FP_DCT1) N = 2 * (n - 1);
    if (kind == FP_DST1) N = 2 * (n + 1);
    if (mr_half_kind(kind, n)) N = mr_half_length(kind, n);
    if (mr_factors(N, kMrMaxPrime).empty()) return 0;
    const size_t line = (size_t)(N + (N - 1) / 16 + 1) * (f32 ? 8 : 16);
    if (line > 200 * 1024) return 0;
    return N;
}

// does one line of the fused MID (tile + spectrum buffer) fit a CTA?
bool mr_mid_fits(const DevTables& T, long long n, bool f32) {
    MrPass p{};
    p.kind = T.fwd_kind;
    p.n = (int)n;
    p.N = T.mrN;
    p.lines = 1;
    p.mid = 1;
    p.half = T.mr_half ? 1 : 0;
    return mr_smem_bytes(p, f32) <= 200 * 1024;
}

// upload the root / quarter-wave / permutation tables of a mixed-radix axis
template <typename AllocT>
fp_status mr_setup(AllocT& allocs, DevTables& T, int kind, long long n, bool f32) {
    const long long N = mr_length(kind, n, f32);
    if (N == 0) return FP_OK;
    T.fac = mr_factors(N, kMrMaxPrime);
    if ((int)T.fac.size() > kMrMaxStages) return FP_OK;
    T.mrN = (int)N;
    T.mr_half = mr_half_kind(kind, n);
    std::vector<long double> r;
    root_table(N, N, r);
    fp_status st;
    if ((st = upload(allocs, r, f32, &T.mr_root)) != FP_OK) return st;
    root_table(4 * n, n + 1, r);   // e^{-i pi k/(2n)}
    if ((st = upload(allocs, r, f32, &T.mr_wq)) != FP_OK) return st;
    if (T.mr_half) {
        // e^{-2 pi i k/(2N)}, k <= N: the real-FFT untangle of the packed line (2N reals)
        root_table(2 * N, N + 1, r);
        if ((st = upload(allocs, r, f32, &T.mr_wt)) != FP_OK) return st;
    }
    if ((st = upload_ints(allocs, mr_perm((int)N, T.fac), &T.mr_perm)) != FP_OK) return st;
    T.mr = true;
    return FP_OK;
}

// a mixed-radix pass of transform `kind` over lines of length n (geometry filled at solve time)
MrPass mr_pass(const DevTables& T, int kind, long long n, long long na, long long nb, bool f32, bool strided,
               int mid_ikind = -1) {
    MrPass p{};
    p.kind = kind;
    p.mid = mid_ikind >= 0;
    p.ikind = p.mid ? mid_ikind : 0;
    p.n = (int)n;
    p.N = T.mrN;
    p.inv = (kind == FP_IDFT || kind == FP_DCT3 || kind == FP_DST3 || kind == MR_IRFFT) ? 1 : 0;
    p.cin = (kind == FP_DFT || kind == FP_IDFT || kind == MR_IRFFT) ? 1 : 0;
    p.cout = (kind == FP_DFT || kind == FP_IDFT || kind == MR_RFFT) ? 1 : 0;
    p.n_in = kind == MR_IRFFT ? (int)(n / 2 + 1) : (int)n;
    p.n_out = kind == MR_RFFT ? (int)(n / 2 + 1) : (int)n;
    if (p.mid) {
        p.n_out = (int)n;   // the inverse of the pair writes n values (complex for IDFT)
        p.cout = mid_ikind == FP_IDFT ? 1 : 0;
    }
    p.nf = (int)T.fac.size();
    for (int q = 0; q < p.nf; ++q) p.fac[q] = T.fac[(size_t)q];
    p.root = T.mr_root;
    p.wq = T.mr_wq;
    p.half = T.mr_half ? 1 : 0;
    p.wt = T.mr_wt;
    p.perm = (const int*)T.mr_perm;
    p.out_mult = 1.0;
    const long long nl = na * nb;
    p.lines = 1;
    p.log_lines = 0;
    p.g.na = (int)na;
    p.g.nb = (int)nb;
    // lines per CTA: contiguous lines fill a 48 KB tile (several CTAs per SM);
    // strided lines are adjacent columns, so the tile is widened towards
    // FP_MR_STRIDED_BYTES row segments while 3 tiles still fit an SM (measured:
    // 1000^3 156 ms at 16-B rows vs 187 ms at 64-B rows with one tile per SM)
    static const int contig_kb = env_int("FP_MR_CONTIG_KB", 48);
    static const int strided_bytes = env_int("FP_MR_STRIDED_BYTES", 128);
    static const int strided_kb = env_int("FP_MR_STRIDED_KB", 72);
    const int eb = (p.cin ? 2 : 1) * (f32 ? 4 : 8);
    while (p.lines < 32 && p.lines < nl) {
        MrPass q = p;
        q.lines *= 2;
        const size_t sm = mr_smem_bytes(q, f32);
        const bool want = sm <= (size_t)contig_kb * 1024 ||
                          (strided && p.lines * eb < strided_bytes && sm <= (size_t)strided_kb * 1024);
        if (!want) break;
        p = q;
        p.log_lines += 1;
    }
    p.tiles = (int)((nl + p.lines - 1) / p.lines);
    return p;
}

// forward/backward transform ids of a (bc, kind) row (transforms.py:99-125)
void pair_for(int bc, int kind, int* fwd, int* bwd) {
    if (bc == FP_BC_PERIODIC) { *fwd = FP_DFT; *bwd = FP_IDFT; }
    else if (bc == FP_BC_DIRICHLET) {
        if (kind == FP_GRID_REGULAR) { *fwd = FP_DST1; *bwd = FP_DST1; }
        else { *fwd = FP_DST2; *bwd = FP_DST3; }
    } else {
        if (kind == FP_GRID_REGULAR) { *fwd = FP_DCT1; *bwd = FP_DCT1; }
        else { *fwd = FP_DCT2; *bwd = FP_DCT3; }
    }
}

double backward_scale(int fwd, long long n) {  // transforms.py:88-96
    if (fwd == FP_DFT) return 1.0;
    if (fwd == FP_DST1) return 1.0 / (2.0 * (double)(n + 1));
    if (fwd == FP_DCT1) return 1.0 / (2.0 * (double)(n - 1));
    return 1.0 / (2.0 * (double)n);
}

double ones_null_coeff(int fwd, long long n) {  // solver.py:58-62
    if (fwd == FP_DFT) return 1.0;
    if (fwd == FP_DCT1) return 2.0 * (double)(n - 1);
    return 2.0 * (double)n;
}

fp_status validate(const fp_config* c) {
    if (!c) return fail(FP_ERR_CONFIG, "config is NULL");
    if (c->ndim < 1 || c->ndim > 3)
        return fail(FP_ERR_CONFIG, "1 to 3 dimensions supported, got " + std::to_string(c->ndim));
    if (c->precision != FP_F64 && c->precision != FP_F32)
        return fail(FP_ERR_CONFIG, "precision must be one of ['double', 'single']");
    if (c->approx != FP_APPROX_SPECTRAL && c->approx != FP_APPROX_FD2)
        return fail(FP_ERR_CONFIG, "unknown approximation");
    int nrow_bc = -1, nrow_kind = -1;
    for (int a = 0; a < c->ndim; ++a) {
        const long long n = c->n[a];
        if (n < 1) return fail(FP_ERR_CONFIG, "point count must be positive, got n=" + std::to_string(n));
        if (!(c->length[a] > 0.0)) return fail(FP_ERR_CONFIG, "axis length must be positive");
        if (c->bc[a] < 0 || c->bc[a] > 2 || c->kind[a] < 0 || c->kind[a] > 1)
            return fail(FP_ERR_CONFIG, "unknown boundary condition or grid kind");
        if (c->bc[a] == FP_BC_PERIODIC && c->kind[a] == FP_GRID_STAGGERED)
            return fail(FP_ERR_CONFIG, "periodic boundary conditions admit only the regular grid");
        if (c->bc[a] == FP_BC_NEUMANN && c->kind[a] == FP_GRID_REGULAR && n < 2)
            return fail(FP_ERR_CONFIG, "Neumann on a regular grid needs n >= 2 (boundary nodes included)");
        if (c->bc[a] != FP_BC_PERIODIC) {
            if (nrow_bc < 0) { nrow_bc = c->bc[a]; nrow_kind = c->kind[a]; }
            else if (nrow_bc != c->bc[a] || nrow_kind != c->kind[a])
                return fail(FP_ERR_CONFIG,
                            "unsupported boundary pattern: non-periodic axes must all carry the same "
                            "condition and grid kind");
        }
        if (n > (1LL << 30)) return fail(FP_ERR_UNSUPPORTED, "axis too long");
    }
    return FP_OK;
}

// Which engine runs the transform along an axis, and its FFT length.
// rfft: axis is the real-FFT periodic axis.  Returns M (0 = dense).
// longest complex FFT line held in one tile (2^13: 139 KB of fp64 shared memory)
const long long kFftMax = 8192;

// complex FFT length of an axis on the FFT engine, 0 = dense engine
int fft_length(int bc, int kind, long long n, bool rfft, bool regular_fft = true) {
    if (bc == FP_BC_PERIODIC) {
        const long long M = rfft ? ((n % 2 == 0) ? n / 2 : 0) : n;
        if (M >= 16 && M <= kFftMax && is_pow2(M)) return (int)M;
        return 0;
    }
    if (kind != FP_GRID_STAGGERED) {
        // DCT-I (n = M + 1) / DST-I (n = M - 1) as the real FFT of the 2M-point extension
        if (!regular_fft) return 0;
        const long long M = bc == FP_BC_NEUMANN ? n - 1 : n + 1;
        if (M >= 16 && M <= kFftMax && is_pow2(M)) return (int)M;
        return 0;
    }
    if (n % 2) return 0;
    const long long M = n / 2;
    if (M >= 16 && M <= kFftMax && is_pow2(M)) return (int)M;
    return 0;
}

// longest dense-engine line: the register-tiled kernel stages one line next to
// its matrix tile (complex fp64 fits up to 8695 points); the matrix is n^2 entries
const long long kDenseMax = 8192;


// choose the tile shape of an FFT pass
void fft_tile_shape(FftPass& p, bool f32, bool in_cpx, long long na, long long nb) {
    const int logTL = p.logM - 4;
    const int real_bytes = f32 ? 4 : 8;
    int lines;
    // FP_TILE_THREADS_CONTIG / FP_TILE_BYTES_STRIDED: tuning overrides (benchmarks only)
    static const int contig_threads = env_int("FP_TILE_THREADS_CONTIG", 32);
    static const int strided_bytes_io = env_int("FP_TILE_BYTES_STRIDED", 128);
    static const int strided_bytes_mid = env_int("FP_TILE_BYTES_MID", 128);
    const int strided_bytes = p.op == OP_MID ? strided_bytes_mid : strided_bytes_io;
    if (p.family == FAM_CONTIG) {
        lines = std::max(1, contig_threads >> logTL);
        // long fp32 lines (64+ threads each): two per tile (c5 inverse rFFT 18.3 -> 17.1 ms)
        static const int contig_long_f32 = env_int("FP_CONTIG_LONG_F32_LINES", 2);
        if (f32 && logTL >= 6) lines = std::max(lines, contig_long_f32);
        const long long nl = na * nb;
        while (lines > 1 && lines / 2 >= nl) lines /= 2;
        p.lines = lines;
        p.logLines = ilog2(lines);
        while (p.lines > 1 && fft_pass_smem_bytes(p, real_bytes) > 100 * 1024) {
            p.lines /= 2;
            p.logLines -= 1;
        }
        p.tiles = (int)((nl + p.lines - 1) / p.lines);
        p.nbt = 0;
    } else {
        const int eb = (in_cpx ? 2 : 1) * real_bytes;
        lines = std::max(1, strided_bytes / eb);
        while (lines > 1 && lines / 2 >= nb) lines /= 2;
        p.lines = lines;
        p.logLines = ilog2(lines);
        p.ls = strided_line_stride(p, f32);
        while (p.lines > 1 && ((p.lines << logTL) > 512 || fft_pass_smem_bytes(p, real_bytes) > 200 * 1024)) {
            p.lines /= 2;
            p.logLines -= 1;
            p.ls = strided_line_stride(p, f32);
        }
        // 256 threads while the rows stay >= 64 B (two resident tiles per SM beat
        // 128-B rows at one: c4 y-rFFT 2.53 -> 2.16 ms, c4 MID 4.18 -> 3.74 ms;
        // c3's real-line MID keeps 128-B rows at 256 threads: 0.729 -> 0.713 ms)
        static const int io_threads = env_int("FP_TILE_THREADS_STRIDED", 256);
        while (p.lines > 1 && (p.lines << logTL) > io_threads && p.lines * eb > 64) {
            p.lines /= 2;
            p.logLines -= 1;
            p.ls = strided_line_stride(p, f32);
        }
        // complex fp32 MID on 2048 / 4096-point lines: the 512-thread cap leaves
        // 32-B (16-B) rows; a tile of twice the width runs as two compute halves
        static const int mid_wide = env_int("FP_MID_WIDE", 1);
        static const int io_wide = env_int("FP_IO_WIDE", 1);
        const bool cfft = (p.op == OP_INV) ? p.ikind == IK_ICFFT : p.fkind == FK_CFFT;
        const bool want_wide = (p.op == OP_MID) ? mid_wide == 1 : io_wide == 1;
        p.sub = 1;
        if (want_wide && f32 && in_cpx && cfft && (p.logM == 11 || p.logM == 12) &&
            (p.lines << logTL) == 512 && p.lines * 2 <= nb && p.lines * 2 * eb <= strided_bytes) {
            FftPass q = p;
            q.lines *= 2;
            q.logLines += 1;
            q.ls = strided_line_stride(q, f32);
            if (fft_pass_smem_bytes(q, real_bytes) <= 200 * 1024) { p = q; p.sub = 2; }
        }
        p.nbt = (int)((nb + p.lines - 1) / p.lines);
        p.tiles = (int)(na * p.nbt);
    }
}

// ---------------------------------------------------------------------------
// Bluestein engine (fp_blue.cu): plan-time tables and the per-pass launch sequence.
//
// FFT_L of `cl` contiguous scratch rows (complex, plan precision) on the FFT
// engine: one contiguous pass for L <= 8192, else the four-step L1 x L2
// (strided FFT over j1, twiddle, contiguous FFT over j2; the output sits at
// k1 L2 + k2 for frequency k1 + L1 k2 -- the filter spectrum uses the same order,
// and the inverse runs the steps backwards, so no transpose is ever needed).
cudaError_t blue_cfft(const DevTables& T, void* S, long long cl, bool inv, bool f32, cudaStream_t st) {
    const int et = f32 ? ET_C64 : ET_C128;
    auto pass = [&](int M, const void* w, bool strided, long long na, long long nb, long long s_t, long long sa,
                    long long sb) {
        FftPass p{};
        p.op = inv ? OP_INV : OP_FWD;
        p.fkind = FK_CFFT;
        p.ikind = IK_ICFFT;
        p.family = strided ? FAM_STRIDED : FAM_CONTIG;
        p.n = M;
        p.M = M;
        p.logM = ilog2(M);
        p.ls = p.M + p.M / 16 + 1;
        if ((p.ls & 1) == 0) p.ls += 1;
        p.g.na = (int)na;
        p.g.nb = (int)nb;
        p.g.in = S;
        p.g.out = S;
        p.g.in_type = p.g.out_type = et;
        p.g.in_st = p.g.out_st = s_t;
        p.g.in_sa = p.g.out_sa = sa;
        p.g.in_sb = p.g.out_sb = sb;
        fft_tile_shape(p, f32, true, na, nb);
        p.wfft = w;
        p.out_mult = 1.0;
        return launch_fft_pass(p, f32, st);
    };
    const long long L = T.bL, L1 = T.bL1, L2 = T.bL2;
    if (L1 == 1) return pass((int)L, T.b_w2, false, cl, 1, 1, L, 0);
    cudaError_t e;
    if (!inv) {
        if ((e = pass((int)L1, T.b_w1, true, cl, L2, L2, L, 1)) != cudaSuccess) return e;
        if ((e = launch_blue_twiddle(S, cl, (int)L1, (int)L2, 0, f32, st)) != cudaSuccess) return e;
        return pass((int)L2, T.b_w2, false, cl, L1, 1, L, L2);
    }
    if ((e = pass((int)L2, T.b_w2, false, cl, L1, 1, L, L2)) != cudaSuccess) return e;
    if ((e = launch_blue_twiddle(S, cl, (int)L1, (int)L2, 1, f32, st)) != cudaSuccess) return e;
    return pass((int)L1, T.b_w1, true, cl, L2, L2, L, 1);
}

// DFT length of a kind's Bluestein recipe
long long blue_length(int kind, long long n) {
    if (kind == FP_DCT1) return 2 * (n - 1);
    if (kind == FP_DST1) return 2 * (n + 1);
    return n;
}

// shortest line that takes the Bluestein engine instead of the dense one
// (FP_BLUE_MIN overrides; FP_BLUE=0 disables it below the dense engine's cap)
long long blue_min_length() {
    static const long long v = [] {
        const char* e = std::getenv("FP_BLUE");
        if (e && *e == '0') return (long long)kDenseMax + 1;
        return (long long)env_int("FP_BLUE_MIN", 128);
    }();
    return v;
}

// tables of a Bluestein axis (pair of kinds with one DFT length); the filter
// spectra are computed on the device with the same FFT_L the solve uses
template <typename AllocT>
fp_status blue_setup(AllocT& allocs, DevTables& T, int fwd_kind, long long n, bool f32) {
    const long long N = blue_length(fwd_kind, n);
    long long L = 16;
    while (L < 2 * N - 1) L *= 2;
    const long long max_fft = 8192;
    if (L > max_fft * max_fft) return fail(FP_ERR_UNSUPPORTED, "line too long for the Bluestein engine");
    T.bN = (int)N;
    T.bL = (int)L;
    T.bL1 = 1;
    T.bL2 = (int)L;
    if (L > max_fft) {
        T.bL1 = (int)std::max<long long>(16, L / max_fft);
        T.bL2 = (int)(L / T.bL1);
    }
    fp_status st;
    std::vector<long double> c(2 * (size_t)N);
    for (long long m = 0; m < N; ++m) {   // c_m = e^{i pi m^2/N} = e^{2 pi i (m^2 mod 2N)/(2N)}
        const long long r = (long long)(((unsigned long long)m * (unsigned long long)m) % (unsigned long long)(2 * N));
        exact_cis(r, 2 * N, &c[2 * m], &c[2 * m + 1]);
    }
    if ((st = upload(allocs, c, f32, &T.b_chirp)) != FP_OK) return st;
    std::vector<long double> r;
    root_table(4 * n, n + 1, r);   // e^{-i pi k/(2n)}
    if ((st = upload(allocs, r, f32, &T.b_wq)) != FP_OK) return st;
    std::vector<long double> wf, wt, ww;
    fft_tables(T.bL2, T.bL2, false, wf, wt, ww);
    if ((st = upload(allocs, wf, f32, &T.b_w2)) != FP_OK) return st;
    if (T.bL1 > 1) {
        fft_tables(T.bL1, T.bL1, false, wf, wt, ww);
        if ((st = upload(allocs, wf, f32, &T.b_w1)) != FP_OK) return st;
    }
    const size_t cb = (size_t)L * (f32 ? 8 : 16);
    for (int conj = 0; conj < 2; ++conj) {
        void* bh = nullptr;
        CUDA_TRY(cudaMalloc(&bh, cb));
        allocs.push_back(bh);
        (conj ? T.b_bhat_p : T.b_bhat_m) = bh;
    }
    void* S = nullptr;
    CUDA_TRY(cudaMalloc(&S, cb));
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) { cudaFree(S); return fail(FP_ERR_CUDA, "stream"); }
    cudaError_t e = cudaSuccess;
    for (int conj = 0; conj < 2 && e == cudaSuccess; ++conj) {
        e = launch_blue_filter(S, T.b_chirp, (int)N, (int)L, conj, f32, s);
        if (e == cudaSuccess) e = blue_cfft(T, S, 1, false, f32, s);
        if (e == cudaSuccess) e = launch_blue_scale(conj ? T.b_bhat_p : T.b_bhat_m, S, (int)L, 1.0 / (double)L, f32, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    cudaFree(S);
    if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("Bluestein filter spectrum: ") + cudaGetErrorString(e));
    T.blue = true;
    return FP_OK;
}

// the pass descriptor of one Bluestein transform (geometry filled at solve time)
BluePass blue_pass(const DevTables& T, int kind, long long n, long long na, long long nb) {
    BluePass p{};
    p.kind = kind;
    p.n = (int)n;
    p.n_out = kind == MR_RFFT ? (int)(n / 2 + 1) : (int)n;
    p.N = T.bN;
    p.L = T.bL;
    p.inv = (kind == FP_IDFT || kind == MR_IRFFT || kind == FP_DCT3 || kind == FP_DST3) ? 1 : 0;
    p.g.na = (int)na;
    p.g.nb = (int)nb;
    p.chirp = T.b_chirp;
    p.wq = T.b_wq;
    p.out_mult = 1.0;
    return p;
}

// scratch bytes of one Bluestein pass: whole chunks of rows, at most ~256 MB
size_t blue_scratch_bytes(const DevTables& T, long long lines, bool f32) {
    const size_t row = (size_t)T.bL * (f32 ? 8 : 16);
    const size_t cap = (size_t)env_int("FP_BLUE_SCRATCH_MB", 256) << 20;
    long long cl = (long long)std::max<size_t>(1, cap / row);
    if (cl > lines) cl = lines;
    return row * (size_t)std::max<long long>(cl, 1);
}

// one Bluestein pass over every line, in chunks that fit `scratch`
cudaError_t run_blue(const DevTables& T, const BluePass& p, void* scratch, size_t scratch_bytes, bool f32,
                     cudaStream_t st) {
    const long long nl = (long long)p.g.na * p.g.nb;
    const size_t row = (size_t)p.L * (f32 ? 8 : 16);
    const long long cmax = (long long)(scratch_bytes / row);
    if (cmax < 1) return cudaErrorInvalidValue;
    const void* bhat = p.inv ? T.b_bhat_p : T.b_bhat_m;
    cudaError_t e = cudaSuccess;
    for (long long l0 = 0; l0 < nl && e == cudaSuccess; l0 += cmax) {
        const long long cl = std::min(cmax, nl - l0);
        if ((e = launch_blue_gather(p, scratch, l0, cl, f32, st)) != cudaSuccess) break;
        if ((e = blue_cfft(T, scratch, cl, false, f32, st)) != cudaSuccess) break;
        if ((e = launch_blue_mul(scratch, bhat, cl, p.L, f32, st)) != cudaSuccess) break;
        if ((e = blue_cfft(T, scratch, cl, true, f32, st)) != cudaSuccess) break;
        e = launch_blue_emit(p, scratch, l0, cl, f32, st);
    }
    return e;
}

}  // namespace

// ----------------------------------------------------------------------------
// Slab decomposition layout (device-free; shared by the planner and fp_dist_layout).
struct DistLayout {
    long long a0, off0, A;           // this rank's planes of axis 0, its first plane, the exchange pitch
    long long q, r;                  // balanced split: ranks < r own q + 1 planes, the others q
    long long e1, e2, E1, B;
    int r_axis;
    bool cpx;
    bool wall0_cpx;                  // wall axis 0 on a complex state: the MID runs on its real view
};

// first global plane of rank `k` under the balanced split
static long long dist_off(const DistLayout& L, long long k) { return k * L.q + std::min(k, L.r); }

static fp_status dist_layout(const fp_config* cfg, int nranks, int rank, DistLayout* L) {
    const int d = cfg->ndim;
    if (nranks < 1) return fail(FP_ERR_VALUE, "nranks must be >= 1");
    if (nranks == 1) {
        *L = DistLayout{cfg->n[0], 0, cfg->n[0], cfg->n[0], 0, d > 1 ? cfg->n[1] : 1, d > 2 ? cfg->n[2] : 1, 0, 0, -1, false, false};
        return FP_OK;
    }
    if (d < 2) return fail(FP_ERR_UNSUPPORTED, "a 1D problem does not decompose over ranks");
    if (cfg->n[0] < nranks) return fail(FP_ERR_UNSUPPORTED, "axis 0 has fewer planes than ranks");
    bool other_periodic = false;
    for (int a = 1; a < d; ++a) other_periodic |= cfg->bc[a] == FP_BC_PERIODIC;
    if (fft_length(cfg->bc[0], cfg->kind[0], cfg->n[0], cfg->bc[0] == FP_BC_PERIODIC && !other_periodic, true) == 0)
        return fail(FP_ERR_UNSUPPORTED, "distributed solve: axis 0 must be on the FFT engine (power-of-two FFT length: "
                                        "n = 2^k, or 2^k +- 1 for DCT-I / DST-I)");
    // (DCT-I plans: the exact mean removal is global -- fp_dist_mean_partial + all-reduce +
    //  fp_dist_mean_subtract, driven by the caller after phase 2)
    // forward order without axis 0: real axes descending, then periodic descending
    int r_axis = -1;
    for (int a = d - 1; a >= 1; --a) if (cfg->bc[a] == FP_BC_PERIODIC && r_axis < 0) r_axis = a;
    if (r_axis < 0 && cfg->bc[0] == FP_BC_PERIODIC) r_axis = 0;
    DistLayout l{};
    l.q = cfg->n[0] / nranks;
    l.r = cfg->n[0] % nranks;
    l.A = l.q + (l.r ? 1 : 0);
    l.a0 = l.q + (rank < l.r ? 1 : 0);
    l.off0 = dist_off(l, rank);
    l.r_axis = r_axis;
    l.cpx = r_axis > 0;
    l.wall0_cpx = l.cpx && cfg->bc[0] != FP_BC_PERIODIC;
    l.e1 = cfg->n[1];
    l.e2 = d > 2 ? cfg->n[2] : 1;
    if (r_axis == 1) l.e1 = cfg->n[1] / 2 + 1;
    if (r_axis == 2) l.e2 = cfg->n[2] / 2 + 1;
    l.E1 = (l.e1 + nranks - 1) / nranks * nranks;
    l.B = l.E1 / nranks;
    *L = l;
    return FP_OK;
}

// ============================================================================
extern "C" {

FP_API int fp_abi_version(void) { return FP_ABI_VERSION; }
FP_API const char* fp_last_error(void) { return g_err.c_str(); }

static fp_status build_plan(const fp_config* cfg, int device, int nranks, int rank, fp_plan** out) {
    if (!out) return fail(FP_ERR_VALUE, "plan out-pointer is NULL");
    *out = nullptr;
    fp_status st = validate(cfg);
    if (st != FP_OK) return st;
    if (rank < 0 || rank >= nranks) return fail(FP_ERR_VALUE, "rank out of range");
    DistLayout DL{};
    if ((st = dist_layout(cfg, nranks, rank, &DL)) != FP_OK) return st;
    const bool dist = nranks > 1;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(FP_ERR_CUDA, "no CUDA device available (the solve path has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(FP_ERR_VALUE, "invalid device ordinal");
    DeviceGuard dg(device);

    fp_plan* P = new fp_plan();
    P->device = device;
    P->cfg = *cfg;
    P->nranks = nranks;
    P->rank = rank;
    const int d = cfg->ndim;
    P->ndim = d;
    P->f32 = cfg->precision == FP_F32;
    int fwd[3] = {0, 0, 0}, bwd[3] = {0, 0, 0};
    P->singular = true;
    for (int a = 0; a < d; ++a) {
        P->n[a] = cfg->n[a];
        pair_for(cfg->bc[a], cfg->kind[a], &fwd[a], &bwd[a]);
        if (cfg->bc[a] == FP_BC_PERIODIC) P->periodic_mask |= 1 << a;
        if (cfg->bc[a] == FP_BC_DIRICHLET) P->singular = false;
        P->bscale *= backward_scale(fwd[a], cfg->n[a]);
        if (cfg->bc[a] == FP_BC_PERIODIC) P->np_prod *= (double)cfg->n[a];
    }
    {   // SolverConfig.mode (solver.py:111-114): uniform iff one (bc, kind) row
        bool uniform = true;
        for (int a = 1; a < d; ++a) if (cfg->bc[a] != cfg->bc[0] || cfg->kind[a] != cfg->kind[0]) uniform = false;
        P->mixed = !uniform;
    }
    if (P->singular) {
        // solver.py:224-225: the reference subtracts the arithmetic mean after the
        // backward pass.  With DFT / DCT-II the zeroed null coefficient already IS
        // the mean (no-op to roundoff); with DCT-I it is a trapezoid-weighted mean,
        // so those plans get the explicit reduction + subtraction.
        for (int a = 0; a < d; ++a)
            if (cfg->bc[a] == FP_BC_NEUMANN && cfg->kind[a] == FP_GRID_REGULAR) P->mean_fix = true;
        double ns = 1.0;
        for (int a = 0; a < d; ++a) ns *= ones_null_coeff(fwd[a], cfg->n[a]);
        P->null_scale = ns;
    }

    // forward order: real axes descending, then periodic axes descending
    // (distributed: axis 0 -- the decomposed one -- always last, i.e. the MID axis)
    std::vector<int> order;
    const int amin = dist ? 1 : 0;
    for (int a = d - 1; a >= amin; --a) if (cfg->bc[a] != FP_BC_PERIODIC) order.push_back(a);
    for (int a = d - 1; a >= amin; --a) if (cfg->bc[a] == FP_BC_PERIODIC) { if (P->r_axis < 0) P->r_axis = a; order.push_back(a); }
    if (dist) {
        if (P->r_axis < 0 && cfg->bc[0] == FP_BC_PERIODIC) P->r_axis = 0;
        order.push_back(0);
        P->a0 = DL.a0;
        P->A = DL.A;
        P->n[0] = DL.a0;             // local extents from here on; cfg->n keeps the global ones
        P->e1 = DL.e1; P->e2 = DL.e2; P->E1 = DL.E1; P->B = DL.B; P->x_cpx = DL.cpx;
        P->wall0_cpx = DL.wall0_cpx;
        // send layout: axis 1 outermost -> peer q's block (axis-1 rows [qB,(q+1)B)) is contiguous;
        // every rank's block holds A (= max local planes) planes, so all blocks have one size
        if (d == 3) { P->xs[0] = DL.e2; P->xs[1] = DL.A * DL.e2; P->xs[2] = 1; }
        else { P->xs[0] = 1; P->xs[1] = DL.A; }
        if (DL.r != 0 || !is_pow2(DL.A)) {
            // receive layout row of global plane j: src(j) * (B * xs1) + (j - off(src)) * xs0,
            // in the units the MID addresses (reals for the real view)
            const long long u = DL.wall0_cpx ? 2 : 1;
            std::vector<long long> tab((size_t)cfg->n[0]);
            long long src = 0;
            for (long long j = 0; j < cfg->n[0]; ++j) {
                while (src + 1 < nranks && j >= dist_off(DL, src + 1)) ++src;
                tab[(size_t)j] = u * (src * DL.B * P->xs[1] + (j - dist_off(DL, src)) * P->xs[0]);
            }
            void* dt = nullptr;
            if (cudaMalloc(&dt, tab.size() * sizeof(long long)) != cudaSuccess) { delete P; return fail(FP_ERR_ALLOC, "cudaMalloc row table"); }
            P->allocs.push_back(dt);
            if (cudaMemcpy(dt, tab.data(), tab.size() * sizeof(long long), cudaMemcpyHostToDevice) != cudaSuccess) { delete P; return fail(FP_ERR_CUDA, "upload row table"); }
            P->row_tab = (const long long*)dt;
        }
    }
    P->middle = order.back();
    for (int a = 0; a < 3; ++a) P->cext[a] = P->n[a];
    if (P->r_axis >= 0) P->cext[P->r_axis] = P->n[P->r_axis] / 2 + 1;
    P->cpitch_last = (P->cext[d - 1] + 7) / 8 * 8;
    if (P->r_axis < 0 || P->cext[d - 1] == P->n[d - 1]) P->cpitch_last = P->cext[d - 1];

    std::vector<double> lam_host[3];
    // eigenvalue tables (host mirror may pass numpy-built ones)
    for (int a = 0; a < d; ++a) {
        std::vector<double> lam;
        if (cfg->eig[a]) lam.assign(cfg->eig[a], cfg->eig[a] + cfg->n[a]);
        else lam = eigenvalue_table(AxisSpec{cfg->n[a], cfg->length[a], cfg->bc[a], cfg->kind[a]}, cfg->approx);
        // one leading pad entry: a DST-I axis on the FFT engine reads its table from
        // the pad (spectral index k = 1..M-1 <-> eigenvalue k - 1)
        lam_host[a] = lam;
        lam.insert(lam.begin(), 0.0);
        void* dl = nullptr;
        if (cudaMalloc(&dl, lam.size() * sizeof(double)) != cudaSuccess) { delete P; return fail(FP_ERR_ALLOC, "cudaMalloc eigenvalue table"); }
        P->allocs.push_back(dl);
        if (cudaMemcpy(dl, lam.data(), lam.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) { delete P; return fail(FP_ERR_CUDA, "upload eigenvalue table"); }
        P->d_lam_pad[a] = (double*)dl;
        P->d_lam[a] = (double*)dl + 1;
    }

    // per-axis engines + tables
    int Mx[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) {
        const bool rf = (a == P->r_axis);
        // (slab phases: the local DCT-I / DST-I axes on the mixed-radix / dense engines;
        //  axis 0's MID on the FFT engine over the receive layout)
        Mx[a] = fft_length(cfg->bc[a], cfg->kind[a], cfg->n[a], rf, !dist || a == 0);
        DevTables& T = P->tab[a];
        if (Mx[a] > 0) {
            P->fft_mask |= 1 << a;
            std::vector<long double> wf, wt, ww;
            const bool real_kind = cfg->bc[a] != FP_BC_PERIODIC || rf;
            const bool regular = cfg->bc[a] != FP_BC_PERIODIC && cfg->kind[a] != FP_GRID_STAGGERED;
            fft_tables(regular ? 2 * Mx[a] : (int)cfg->n[a], Mx[a], real_kind, wf, wt, ww);
            if ((st = upload(P->allocs, wf, P->f32, &T.wfft)) != FP_OK) { delete P; return st; }
            if ((st = upload(P->allocs, wt, P->f32, &T.wt)) != FP_OK) { delete P; return st; }
            if ((st = upload(P->allocs, ww, P->f32, &T.ww)) != FP_OK) { delete P; return st; }
            if (cfg->bc[a] != FP_BC_PERIODIC && !regular) {
                std::vector<long double> wb;
                mid_table((int)cfg->n[a], Mx[a], wb);
                if ((st = upload(P->allocs, wb, P->f32, &T.wb)) != FP_OK) { delete P; return st; }
                // eigenvalue pairs at the physical indices of the quads (DST: k -> n-1-k)
                const long long nn = cfg->n[a], MM = Mx[a];
                const bool dst_ax = cfg->bc[a] == FP_BC_DIRICHLET;
                auto kp = [&](long long k) { return dst_ax ? nn - 1 - k : k; };
                std::vector<double> l2(2 * (size_t)(MM + 1), 0.0);
                for (long long q = 0; q <= MM; ++q) {
                    l2[2 * q] = lam_host[a][(size_t)kp(q)];
                    l2[2 * q + 1] = q > 0 ? lam_host[a][(size_t)kp(nn - q)] : 0.0;
                }
                void* d2 = nullptr;
                if (cudaMalloc(&d2, l2.size() * sizeof(double)) != cudaSuccess) { delete P; return fail(FP_ERR_ALLOC, "cudaMalloc eigenvalue pairs"); }
                P->allocs.push_back(d2);
                if (cudaMemcpy(d2, l2.data(), l2.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) { delete P; return fail(FP_ERR_CUDA, "upload eigenvalue pairs"); }
                T.lam2 = d2;
            }
        } else {
            const int fk = cfg->bc[a] == FP_BC_PERIODIC ? (rf ? 100 : FP_DFT) : fwd[a];
            const int bk = cfg->bc[a] == FP_BC_PERIODIC ? (rf ? 101 : FP_IDFT) : bwd[a];
            T.fwd_kind = fk;
            T.bwd_kind = bk;
            if ((st = mr_setup(P->allocs, T, fk, cfg->n[a], P->f32)) != FP_OK) { delete P; return st; }
            if (T.mr) continue;
            if (cfg->n[a] > kDenseMax || cfg->n[a] >= blue_min_length()) {
                // a prime factor above 61 (or a line too long for one CTA): Bluestein
                T.fwd_kind = fk;
                T.bwd_kind = bk;
                if ((st = blue_setup(P->allocs, T, fk, cfg->n[a], P->f32)) != FP_OK) { delete P; return st; }
                continue;
            }
            std::vector<double> m;
            int no, ni;
            bool cpx;
            dense_matrix(fk, (int)cfg->n[a], m, &no, &ni, &cpx);
            T.fwd_nout = no; T.fwd_nin = ni; T.fwd_cpx = cpx;
            if ((st = upload(P->allocs, m, P->f32, &T.mat_f)) != FP_OK) { delete P; return st; }
            dense_matrix(bk, (int)cfg->n[a], m, &no, &ni, &cpx);
            T.bwd_nout = no; T.bwd_nin = ni; T.bwd_cpx = cpx;
            if ((st = upload(P->allocs, m, P->f32, &T.mat_b)) != FP_OK) { delete P; return st; }
        }
    }

    // ---- pass schedule
    // extents of the state: before the r-axis forward pass (and after its
    // inverse) everything is real with extents n; in between, complex with cext.
    auto other_axes = [&](int t, int* a_, int* b_) {
        int o[2] = {-1, -1}, k = 0;
        for (int a = 0; a < d; ++a) if (a != t) o[k++] = a;
        if (k == 2) { *a_ = o[0]; *b_ = o[1]; }
        else if (k == 1) { *a_ = -1; *b_ = o[0]; }
        else { *a_ = -1; *b_ = -1; }
    };
    const double inv_np = 1.0 / P->np_prod;
    bool complex_state = false;
    int cur = B_RHS;
    bool rs_dummy = false;
    const int realbuf = B_RS;  // resolved at solve time to OUT when out is dense

    auto make_fft = [&](int t, int op, bool in_cpx, bool out_cpx, int in_buf, int out_buf, int phase) {
        PassT ps{};
        ps.engine = EN_FFT;
        ps.phase = phase;
        ps.t = t;
        ps.in_buf = in_buf;
        ps.out_buf = out_buf;
        ps.in_layout = in_cpx ? LY_CPLX : LY_REAL;
        ps.out_layout = out_cpx ? LY_CPLX : LY_REAL;
        other_axes(t, &ps.a, &ps.b);
        FftPass& p = ps.fp;
        const bool periodic = cfg->bc[t] == FP_BC_PERIODIC;
        const bool rf = t == P->r_axis;
        p.op = op;
        const bool regular = !periodic && cfg->kind[t] != FP_GRID_STAGGERED;
        const bool dir = cfg->bc[t] == FP_BC_DIRICHLET;
        p.fkind = periodic ? (rf ? FK_RFFT : FK_CFFT) : (regular ? (dir ? FK_DST1 : FK_DCT1) : (dir ? FK_DST2 : FK_DCT2));
        p.ikind = periodic ? (rf ? IK_IRFFT : IK_ICFFT) : (regular ? (dir ? IK_DST1 : IK_DCT1) : (dir ? IK_DST3 : IK_DCT3));
        p.family = (t == d - 1) ? FAM_CONTIG : FAM_STRIDED;
        p.n = (int)cfg->n[t];
        p.M = Mx[t];
        p.logM = ilog2(p.M);
        p.ls = p.M + p.M / 16 + 1;
        if ((p.ls & 1) == 0) p.ls += 1;
        const long long* ext = complex_state ? P->cext : P->n;
        const long long na = ps.a >= 0 ? ext[ps.a] : 1;
        const long long nb = ps.b >= 0 ? ext[ps.b] : 1;
        p.g.na = (int)na;
        p.g.nb = (int)nb;
        fft_tile_shape(p, P->f32, in_cpx, na, nb);
        p.wfft = P->tab[t].wfft;
        p.wt = P->tab[t].wt;
        p.ww = P->tab[t].ww;
        p.wb = P->tab[t].wb;
        p.out_mult = 1.0;
        Scaling& s = p.s;
        // DST-I spectra sit at k = 1..M-1 of the extended line: eigenvalue k - 1
        s.lam_t = (regular && dir) ? P->d_lam_pad[t] : P->d_lam[t];
        s.lam_pair = (const double*)P->tab[t].lam2;
        s.lam_a = ps.a >= 0 ? P->d_lam[ps.a] : nullptr;
        s.lam_b = ps.b >= 0 ? P->d_lam[ps.b] : nullptr;
        s.pos_t = t; s.pos_a = ps.a; s.pos_b = ps.b;
        s.bscale = P->bscale;
        s.inv_np = inv_np;
        s.singular = P->singular;
        return ps;
    };
    auto make_dense = [&](int t, bool forward, bool in_cpx, bool out_cpx, int in_buf, int out_buf, int phase) {
        PassT ps{};
        ps.engine = EN_DENSE;
        ps.phase = phase;
        ps.t = t;
        ps.in_buf = in_buf;
        ps.out_buf = out_buf;
        ps.in_layout = in_cpx ? LY_CPLX : LY_REAL;
        ps.out_layout = out_cpx ? LY_CPLX : LY_REAL;
        other_axes(t, &ps.a, &ps.b);
        const DevTables& T = P->tab[t];
        if (T.blue) {
            ps.engine = EN_BLUE;
            const long long* ext = complex_state ? P->cext : P->n;
            const long long na = ps.a >= 0 ? ext[ps.a] : 1;
            const long long nb = ps.b >= 0 ? ext[ps.b] : 1;
            ps.bp = blue_pass(T, forward ? T.fwd_kind : T.bwd_kind, cfg->n[t], na, nb);
            P->blue_bytes = std::max(P->blue_bytes, blue_scratch_bytes(T, na * nb, P->f32));
            return ps;
        }
        if (T.mr) {
            ps.engine = EN_MR;
            const long long* ext = complex_state ? P->cext : P->n;
            const long long na = ps.a >= 0 ? ext[ps.a] : 1;
            const long long nb = ps.b >= 0 ? ext[ps.b] : 1;
            ps.mp = mr_pass(T, forward ? T.fwd_kind : T.bwd_kind, cfg->n[t], na, nb, P->f32, t != d - 1);
            return ps;
        }
        DensePass& p = ps.dp;
        p.n_in = forward ? T.fwd_nin : T.bwd_nin;
        p.n_out = forward ? T.fwd_nout : T.bwd_nout;
        p.mat = forward ? T.mat_f : T.mat_b;
        p.cls = !in_cpx && !out_cpx ? DC_R2R : (!in_cpx ? DC_R2C : (out_cpx ? DC_C2C : DC_C2R));
        const long long* ext = complex_state ? P->cext : P->n;
        const long long na = ps.a >= 0 ? ext[ps.a] : 1;
        const long long nb = ps.b >= 0 ? ext[ps.b] : 1;
        p.g.na = (int)na;
        p.g.nb = (int)nb;
        p.in_ls = in_cpx ? 2 * p.n_in : p.n_in;
        const int rb = P->f32 ? 4 : 8;
        int lines = std::max(1, (48 * 1024) / (p.in_ls * rb));
        lines = std::min(lines, 64);
        const long long nl = na * nb;
        if (lines > nl) lines = (int)nl;
        p.lines = lines;
        p.tiles = (int)((nl + lines - 1) / lines);
        p.out_mult = 1.0;
        return ps;
    };
    auto make_scale = [&](int phase, int buf, bool cpx) {
        PassT ps{};
        ps.engine = EN_SCALE;
        ps.phase = phase;
        ps.t = -1;
        ps.in_buf = ps.out_buf = buf;
        ps.in_layout = ps.out_layout = cpx ? LY_CPLX : LY_REAL;
        ps.a = ps.b = -1;
        ScalePass& s = ps.sp;
        s.ndim = d;
        for (int a = 0; a < 3; ++a) s.lam[a] = a < d ? P->d_lam[a] : nullptr;
        s.bscale = P->bscale;
        s.inv_np = inv_np;
        s.singular = P->singular;
        return ps;
    };

    auto schedule = [&](bool split, std::vector<PassT>& L, bool& need_cw) {
    complex_state = false;
    cur = B_RHS;
    const bool only_middle = order.size() == 1;
    // forward passes
    for (size_t i = 0; i + 1 < order.size(); ++i) {
        const int t = order[i];
        const bool rf = t == P->r_axis;
        const bool in_cpx = complex_state;
        const bool out_cpx = complex_state || rf;
        int dst = out_cpx ? B_CW : realbuf;
        if (dist && i + 2 == order.size()) dst = B_X;   // pack for the all-to-all
        else if (out_cpx) need_cw = true; else rs_dummy = true;
        if (Mx[t] > 0) L.push_back(make_fft(t, OP_FWD, in_cpx, out_cpx, cur, dst, 0));
        else L.push_back(make_dense(t, true, in_cpx, out_cpx, cur, dst, 0));
        if (rf) complex_state = true;
        cur = dst;
    }
    // middle
    {
        const int t = P->middle;
        const bool rf = t == P->r_axis;
        const int dst = only_middle ? B_OUT : cur;
        if (split) {
            // _inv_lam override (SolverPlan._inv_lam written by the caller, verifysuite.py:83-88):
            // forward along the middle axis, the stand-alone scale reading the caller's dense
            // factor table, inverse -- the reference's `work *= _inv_lam` (solver.py:221)
            const bool in_c = complex_state, mid_c = complex_state || rf;
            int work = cur;
            if (only_middle || rf) work = mid_c ? B_CW : realbuf;
            if (mid_c && work == B_CW) need_cw = true;
            if (Mx[t] > 0) L.push_back(make_fft(t, OP_FWD, in_c, mid_c, cur, work, 1));
            else L.push_back(make_dense(t, true, in_c, mid_c, cur, work, 1));
            L.push_back(make_scale(1, work, mid_c));
            if (Mx[t] > 0) L.push_back(make_fft(t, OP_INV, mid_c, in_c, work, dst, 1));
            else L.push_back(make_dense(t, false, mid_c, in_c, work, dst, 1));
        } else if (dist) {
            // MID over the receive layout: global axis 0 in P blocks of a0 planes
            // (a wall axis 0 on a complex state: the real kind on the real view -- real and
            // imaginary parts are two real lines, the eigenvalue factors are real)
            const bool rv = DL.wall0_cpx;
            PassT mid = make_fft(t, OP_MID, complex_state && !rv, complex_state && !rv, B_X, B_X, 1);
            mid.dist_mid = true;
            const int pr = rv ? 2 : 1;
            if (d == 3) { mid.fp.g.na = (int)DL.B; mid.fp.g.nb = (int)(pr * DL.e2); }
            else { mid.fp.g.na = 1; mid.fp.g.nb = (int)(pr * DL.B); }
            fft_tile_shape(mid.fp, P->f32, complex_state && !rv, mid.fp.g.na, mid.fp.g.nb);
            L.push_back(mid);
        } else if (Mx[t] > 0) {
            L.push_back(make_fft(t, OP_MID, complex_state, complex_state, cur, dst, 1));
        } else if (P->tab[t].mr && mr_mid_fits(P->tab[t], cfg->n[t], P->f32)) {
            // mixed-radix MID: forward, eigenvalue scale, inverse on the tile
            PassT ps{};
            ps.engine = EN_MR;
            ps.phase = 1;
            ps.t = t;
            ps.in_buf = cur;
            ps.out_buf = dst;
            ps.in_layout = ps.out_layout = complex_state ? LY_CPLX : LY_REAL;
            other_axes(t, &ps.a, &ps.b);
            const long long* ext = complex_state ? P->cext : P->n;
            const long long na = ps.a >= 0 ? ext[ps.a] : 1;
            const long long nb = ps.b >= 0 ? ext[ps.b] : 1;
            const DevTables& T = P->tab[t];
            ps.mp = mr_pass(T, T.fwd_kind, cfg->n[t], na, nb, P->f32, t != d - 1, T.bwd_kind);
            Scaling& sc = ps.mp.s;
            sc.lam_t = P->d_lam[t];
            sc.lam_a = ps.a >= 0 ? P->d_lam[ps.a] : nullptr;
            sc.lam_b = ps.b >= 0 ? P->d_lam[ps.b] : nullptr;
            sc.pos_t = t; sc.pos_a = ps.a; sc.pos_b = ps.b;
            sc.bscale = P->bscale;
            sc.inv_np = inv_np;
            sc.singular = P->singular;
            L.push_back(ps);
        } else if (!rf) {
            // dense forward, scale, dense inverse on the same buffer
            int work = cur;
            if (only_middle) work = complex_state ? B_CW : realbuf;
            if (only_middle && !complex_state) rs_dummy = true;
            L.push_back(make_dense(t, true, complex_state, complex_state, cur, work, 1));
            L.push_back(make_scale(1, work, complex_state));
            L.push_back(make_dense(t, false, complex_state, complex_state, work, dst, 1));
        } else {
            // real-FFT middle axis on the dense engine: real -> half spectrum -> real
            need_cw = true;
            L.push_back(make_dense(t, true, false, true, cur, B_CW, 1));
            complex_state = true;
            L.push_back(make_scale(1, B_CW, true));
            // the inverse writes real data: extents of other axes unchanged
            PassT inv = make_dense(t, false, true, false, B_CW, dst, 1);
            L.push_back(inv);
            complex_state = false;
        }
    }
    // backward passes
    for (int i = (int)order.size() - 2; i >= 0; --i) {
        const int t = order[i];
        const bool rf = t == P->r_axis;
        const bool in_cpx = complex_state;
        const bool out_cpx = complex_state && !rf;
        const bool last = i == 0;
        int dst = last ? B_OUT : (out_cpx ? B_CW : (in_cpx ? realbuf : cur));
        if (!last && cur == B_X) dst = out_cpx ? B_CW : realbuf;   // unpack out of the exchange buffer
        if (!out_cpx && !last) rs_dummy = true;
        if (out_cpx && !last) need_cw = true;
        if (Mx[t] > 0) L.push_back(make_fft(t, OP_INV, in_cpx, out_cpx, cur, dst, 2));
        else L.push_back(make_dense(t, false, in_cpx, out_cpx, cur, dst, 2));
        if (rf) complex_state = false;
        cur = dst;
    }
    };
    schedule(false, P->passes, P->need_cw);
    if (!dist) schedule(true, P->passes_ovr, P->need_cw_ovr);
    // the first pass checks finiteness of the rhs (solver.py:201-202)
    *out = P;
    return FP_OK;
}

FP_API fp_status fp_plan_create(const fp_config* cfg, int device, fp_plan** plan) {
    return build_plan(cfg, device, 1, 0, plan);
}

FP_API fp_status fp_plan_destroy(fp_plan* plan) {
    delete plan;
    return FP_OK;
}

FP_API fp_status fp_plan_info_get(const fp_plan* P, fp_plan_info* info) {
    if (!P || !info) return fail(FP_ERR_VALUE, "NULL argument");
    info->ndim = P->ndim;
    info->mode_mixed = P->mixed;
    info->singular = P->singular;
    info->periodic_mask = P->periodic_mask;
    info->null_scale = P->null_scale * P->np_prod;
    info->num_passes = (int)P->passes.size();  // + 3 small launches when mean_fix
    info->middle_axis = P->middle;
    info->fft_axes_mask = P->fft_mask;
    info->exact_mean = P->mean_fix ? 1 : 0;
    return FP_OK;
}

static size_t align_up(size_t x) { return (x + 255) / 256 * 256; }

static size_t cw_bytes(const fp_plan* P, bool ovr = false) {
    if (!(ovr ? P->need_cw_ovr : P->need_cw)) return 0;
    size_t cnt = 1;
    for (int a = 0; a < P->ndim - 1; ++a) cnt *= (size_t)P->cext[a];
    cnt *= (size_t)P->cpitch_last;
    return align_up(cnt * 2 * (P->f32 ? 4 : 8));
}
static size_t rs_bytes(const fp_plan* P) {
    size_t cnt = 1;
    for (int a = 0; a < P->ndim; ++a) cnt *= (size_t)P->n[a];
    return align_up(cnt * (P->f32 ? 4 : 8));
}

static size_t mean_bytes(const fp_plan* P) {
    return P->mean_fix ? align_up((size_t)(kMeanParts + 1) * sizeof(double)) : 0;
}

FP_API fp_status fp_plan_workspace_bytes(const fp_plan* P, int out_dense, size_t* bytes) {
    return fp_plan_workspace_bytes_ex(P, out_dense, 0, bytes);
}

FP_API fp_status fp_plan_workspace_bytes_ex(const fp_plan* P, int out_dense, int inv_lam_override, size_t* bytes) {
    if (!P || !bytes) return fail(FP_ERR_VALUE, "NULL argument");
    size_t b = cw_bytes(P, inv_lam_override != 0);
    // with a strided `out` the real scratch (also the dtype-cast target) lives here
    if (!out_dense) b += rs_bytes(P);
    b += align_up(P->blue_bytes);
    b += mean_bytes(P);
    *bytes = b;
    return FP_OK;
}

static void dense_strides(const fp_plan* P, bool cpx, long long s[3]) {
    const int d = P->ndim;
    long long acc = 1;
    for (int a = d - 1; a >= 0; --a) {
        s[a] = acc;
        if (cpx) acc *= (a == d - 1) ? P->cpitch_last : P->cext[a];
        else acc *= P->n[a];
    }
    for (int a = d; a < 3; ++a) s[a] = 0;
}

FP_API fp_status fp_solve(const fp_plan* P, const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                          void* out, const int64_t* out_strides, void* workspace, size_t workspace_bytes,
                          void* stream, fp_solve_info* dev_info, void* const* phase_events) {
    return fp_solve_ex(P, rhs, rhs_dtype, rhs_strides, out, out_strides, workspace, workspace_bytes, stream,
                       dev_info, phase_events, nullptr);
}

static fp_status solve_impl(const fp_plan* P, const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                            void* out, const int64_t* out_strides, void* workspace, size_t workspace_bytes,
                            void* stream, fp_solve_info* dev_info, void* const* phase_events,
                            void* const* pass_events, void* xbuf, int ph_lo, int ph_hi,
                            const Producer* prod = nullptr, const void* ovr = nullptr, long long mid_row0 = 0,
                            long long mid_rows = -1) {
    if (!P) return fail(FP_ERR_VALUE, "plan is NULL");
    static const char* const kRange[3][3] = {{"fp_solve_phase 0", "fp_solve_phases 0-1", "fp_solve"},
                                             {"", "fp_solve_phase 1", "fp_solve_phases 1-2"},
                                             {"", "", "fp_solve_phase 2"}};
    NvtxRange solve_range(ph_lo >= 0 && ph_hi <= 2 && ph_lo <= ph_hi ? kRange[ph_lo][ph_hi] : "fp_solve");
    if (ovr && P->passes_ovr.empty()) return fail(FP_ERR_UNSUPPORTED, "_inv_lam override: single-GPU plans only");
    const std::vector<PassT>& PL = ovr ? P->passes_ovr : P->passes;
    const bool need_rhs = ph_lo == 0, need_out = ph_hi == 2;
    if ((need_rhs && !rhs) || (need_out && !out)) return fail(FP_ERR_VALUE, "rhs/out is NULL");
    if (P->nranks > 1 && !xbuf) return fail(FP_ERR_VALUE, "distributed plan: exchange buffer is NULL");
    if (!rhs) { rhs = out ? out : xbuf; rhs_dtype = P->f32 ? FP_F32 : FP_F64; }
    if (!out) out = const_cast<void*>(rhs);
    if (rhs_dtype != FP_F64 && rhs_dtype != FP_F32) return fail(FP_ERR_VALUE, "rhs dtype must be f64 or f32");
    const int d = P->ndim;
    long long dense_r[3];
    dense_strides(P, false, dense_r);
    long long rs_s[3], os_s[3], cw_s[3];
    for (int a = 0; a < 3; ++a) {
        rs_s[a] = (a < d) ? (rhs_strides ? rhs_strides[a] : dense_r[a]) : 0;
        os_s[a] = (a < d) ? (out_strides ? out_strides[a] : dense_r[a]) : 0;
        if (a < d && (rs_s[a] < 0 || os_s[a] < 0)) return fail(FP_ERR_VALUE, "negative strides are not supported");
    }
    dense_strides(P, true, cw_s);
    bool out_dense = true;
    for (int a = 0; a < d; ++a) if (P->n[a] > 1 && os_s[a] != dense_r[a]) out_dense = false;
    size_t need = 0;
    fp_plan_workspace_bytes_ex(P, out_dense, ovr != nullptr, &need);
    if (need > 0 && (!workspace || workspace_bytes < need))
        return fail(FP_ERR_VALUE, "workspace too small: need " + std::to_string(need) + " bytes");
    DeviceGuard dg(P->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (dev_info && ph_lo == 0) CUDA_TRY(cudaMemsetAsync(dev_info, 0, sizeof(fp_solve_info), st));

    void* cw = workspace;
    void* rsb = out_dense ? out : (void*)((char*)workspace + cw_bytes(P, ovr != nullptr));
    // rhs in another precision: cast once into the real scratch (dense, plan-typed)
    const int plan_fp = P->f32 ? FP_F32 : FP_F64;
    if (rhs_dtype != plan_fp && ph_lo == 0) {
        CastPass cp{};
        for (int k = 0; k < 3; ++k) { cp.ext[k] = 1; cp.st[k] = 0; }
        for (int a = 0; a < d; ++a) { cp.ext[3 - d + a] = (int)P->n[a]; cp.st[3 - d + a] = rs_s[a]; }
        cudaError_t e = launch_cast(rhs, rhs_dtype == FP_F32 ? ET_F32 : ET_F64, cp, rsb, P->f32 ? ET_F32 : ET_F64,
                                    (cudaStream_t)stream);
        if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("cast launch failed: ") + cudaGetErrorString(e));
        rhs = rsb;
        rhs_dtype = plan_fp;
        for (int a = 0; a < 3; ++a) rs_s[a] = (a < d) ? (out_dense ? os_s[a] : dense_r[a]) : 0;
    }
    // projection step: the first pass produces its lines from the face velocities
    // (contiguous real-kind FFT pass on the last axis); otherwise a stand-alone
    // divergence kernel fills the (dense) real scratch and the solve reads that
    bool prod_in_pass = false;
    if (prod && ph_lo == 0) {
        const PassT& F = PL[0];
        prod_in_pass = F.engine == EN_FFT && F.fp.op == OP_FWD && F.fp.family == FAM_CONTIG && F.t == d - 1 &&
                       (F.fp.fkind == FK_DCT2 || F.fp.fkind == FK_RFFT);
        if (!prod_in_pass) {
            cudaError_t e = launch_divergence(*prod, rsb, P->f32, (cudaStream_t)stream);
            if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("divergence launch failed: ") + cudaGetErrorString(e));
            rhs = rsb;
            rhs_dtype = plan_fp;
            for (int a = 0; a < 3; ++a) rs_s[a] = (a < d) ? (out_dense ? os_s[a] : dense_r[a]) : 0;
        }
    }
    double* mean_ws = P->mean_fix ? (double*)((char*)workspace + need - mean_bytes(P)) : nullptr;
    const size_t blue_b = align_up(P->blue_bytes);
    void* blue_ws = blue_b ? (void*)((char*)workspace + need - mean_bytes(P) - blue_b) : nullptr;
    const int plan_type = P->f32 ? ET_F32 : ET_F64;
    const int plan_ctype = P->f32 ? ET_C64 : ET_C128;

    auto buf_ptr = [&](int b) -> void* {
        switch (b) {
            case B_RHS: return const_cast<void*>(rhs);
            case B_OUT: return out;
            case B_RS: return rsb;
            case B_X: return xbuf;
            default: return cw;
        }
    };
    auto buf_strides = [&](int b, int layout, long long s[3]) {
        if (b == B_RHS) { for (int a = 0; a < 3; ++a) s[a] = rs_s[a]; return; }
        if (b == B_OUT) { for (int a = 0; a < 3; ++a) s[a] = os_s[a]; return; }
        if (b == B_RS) { for (int a = 0; a < 3; ++a) s[a] = out_dense ? os_s[a] : dense_r[a]; return; }
        if (b == B_X) { for (int a = 0; a < 3; ++a) s[a] = P->xs[a]; return; }
        (void)layout;
        for (int a = 0; a < 3; ++a) s[a] = cw_s[a];
    };
    auto buf_type = [&](int b, int layout) -> int {
        if (layout == LY_CPLX) return plan_ctype;
        if (b == B_RHS) return rhs_dtype == FP_F32 ? ET_F32 : ET_F64;
        return plan_type;
    };

    cudaEvent_t* ev = (cudaEvent_t*)phase_events;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    int phase = 0;
    bool first = true;
    for (size_t i = 0; i < PL.size(); ++i) {
        const PassT& T = PL[i];
        if (T.phase < ph_lo || T.phase > ph_hi) continue;
        while (ev && phase < T.phase) { ++phase; CUDA_TRY(cudaEventRecord(ev[phase], st)); }
        if (pass_events) CUDA_TRY(cudaEventRecord((cudaEvent_t)pass_events[i], st));
        long long si[3], so[3];
        buf_strides(T.in_buf, T.in_layout, si);
        buf_strides(T.out_buf, T.out_layout, so);
        Geometry g{};
        if (T.engine != EN_SCALE) {
            g.in = buf_ptr(T.in_buf);
            g.out = buf_ptr(T.out_buf);
            g.in_type = buf_type(T.in_buf, T.in_layout);
            g.out_type = buf_type(T.out_buf, T.out_layout);
            g.in_st = si[T.t];
            g.out_st = so[T.t];
            g.in_sa = T.a >= 0 ? si[T.a] : 0;
            g.out_sa = T.a >= 0 ? so[T.a] : 0;
            g.in_sb = T.b >= 0 ? si[T.b] : 0;
            g.out_sb = T.b >= 0 ? so[T.b] : 0;
        }
        cudaError_t e = cudaSuccess;
        char range_name[64];
        {
            static const char* const kEngine[5] = {"fft", "dense", "scale", "mixed-radix", "bluestein"};
            static const char* const kPhase[3] = {"forward", "middle", "backward"};
            const bool mid = T.engine == EN_FFT && T.fp.op == OP_MID;
            std::snprintf(range_name, sizeof range_name, "pass %zu: %s axis %d (%s)", i,
                          mid ? "MID" : kPhase[T.phase % 3], T.t, kEngine[T.engine % 5]);
        }
        NvtxRange pass_range(range_name);
        if (T.engine == EN_FFT) {
            FftPass p = T.fp;
            g.na = p.g.na; g.nb = p.g.nb;
            if (T.dist_mid) {
                // receive layout [source rank][axis-1 block][A planes][axis 2]: global plane
                // j = off(src) + i  ->  src * (B * A * e2) + i * e2 (shift / mask when every
                // rank holds A = 2^lg planes, else the plan's row table)
                const long long u = P->wall0_cpx ? 2 : 1;   // real view: strides in reals
                g.in_st_hi = g.out_st_hi = u * P->B * P->xs[1];
                if (P->row_tab) {
                    g.row_tab = P->row_tab;
                } else {
                    int lg = 0;
                    while ((1LL << lg) < P->A) ++lg;
                    g.blk_lg = lg;
                    if (lg == 0) { g.in_st = g.out_st = g.in_st_hi / u; }
                }
                if (u == 2) {
                    g.in_type = g.out_type = plan_type;
                    g.in_st *= 2; g.out_st *= 2;
                    g.in_sa *= 2; g.out_sa *= 2;
                    g.in_sb *= 2; g.out_sb *= 2;
                    g.pair_b = 1;
                }
                if (d == 3) { g.a_off = (int)(P->rank * P->B); g.a_lim = (int)P->e1; }
                else { g.b_off = (int)(P->rank * P->B); g.b_lim = (int)P->e1; }
                if (mid_rows >= 0) {
                    // a chunk of this rank's axis-1 rows (pipelined exchange): the a axis in 3D,
                    // the b axis in 2D; global indices keep the eigenvalues and the null line
                    const size_t eb = (size_t)(g.in_type == ET_C128 || g.in_type == ET_C64 ? 2 : 1) * (P->f32 ? 4 : 8);
                    if (d == 3) {
                        g.in = (const char*)g.in + mid_row0 * g.in_sa * eb;
                        g.out = (char*)g.out + mid_row0 * g.out_sa * eb;
                        g.a_off += (int)mid_row0;
                        p.g.na = (int)mid_rows;
                    } else {
                        const long long u = g.pair_b ? 2 : 1;   // real view: b counts real lines
                        g.in = (const char*)g.in + mid_row0 * g.in_sb * eb;
                        g.out = (char*)g.out + mid_row0 * g.out_sb * eb;
                        g.b_off += (int)mid_row0;
                        p.g.nb = (int)(u * mid_rows);
                    }
                    g.na = p.g.na; g.nb = p.g.nb;
                    p.nbt = (p.g.nb + p.lines - 1) / p.lines;
                    p.tiles = p.g.na * p.nbt;
                    if (mid_row0 > 0) p.s.dc_out = nullptr;
                }
            }
            p.g = g;
            p.nonfinite = first && dev_info ? &dev_info->nonfinite : nullptr;
            p.s.dc_out = dev_info ? &dev_info->dc : nullptr;
            p.prod.active = 0;
            if (first && prod_in_pass) { p.prod = *prod; p.prod.active = 1; }
            const size_t rb = P->f32 ? 4 : 8;
            auto even_ok = [&](long long s, int ext) { return ext <= 1 || (s % 2) == 0; };
            p.vec_in = (p.family == FAM_CONTIG) && g.in_st == 1 && (g.in_type == plan_type) &&
                       even_ok(g.in_sa, g.na) && even_ok(g.in_sb, g.nb) &&
                       ((uintptr_t)g.in % (2 * rb) == 0);
            p.vec_out = (p.family == FAM_CONTIG) && g.out_st == 1 && (g.out_type == plan_type) &&
                        even_ok(g.out_sa, g.na) && even_ok(g.out_sb, g.nb) &&
                        ((uintptr_t)g.out % (2 * rb) == 0);
            tma_prepare(p, P->f32);   // TMA-staged kernel where eligible (fp_tma.cu)
            e = launch_fft_pass(p, P->f32, st);
        } else if (T.engine == EN_MR) {
            MrPass p = T.mp;
            g.na = p.g.na; g.nb = p.g.nb;
            p.g = g;
            p.nonfinite = first && dev_info ? &dev_info->nonfinite : nullptr;
            p.s.dc_out = dev_info ? &dev_info->dc : nullptr;
            e = launch_mr_pass(p, P->f32, st);
        } else if (T.engine == EN_DENSE) {
            DensePass p = T.dp;
            g.na = p.g.na; g.nb = p.g.nb;
            p.g = g;
            p.nonfinite = first && dev_info ? &dev_info->nonfinite : nullptr;
            e = launch_dense_pass(p, P->f32, st);
        } else if (T.engine == EN_BLUE) {
            BluePass p = T.bp;
            g.na = p.g.na; g.nb = p.g.nb;
            p.g = g;
            p.nonfinite = first && dev_info ? &dev_info->nonfinite : nullptr;
            e = run_blue(P->tab[T.t], p, blue_ws, blue_b, P->f32, st);
        } else {
            ScalePass p = T.sp;
            const bool cpx = T.in_layout == LY_CPLX;
            p.data = buf_ptr(T.in_buf);
            p.type = cpx ? plan_ctype : plan_type;
            // pad to 3 axes at the front
            for (int k = 0; k < 3; ++k) { p.ext[k] = 1; p.st[k] = 0; }
            for (int a = 0; a < d; ++a) {
                p.ext[3 - d + a] = (int)(cpx ? P->cext[a] : P->n[a]);
                p.st[3 - d + a] = si[a];
            }
            p.dc_out = dev_info ? &dev_info->dc : nullptr;
            p.ovr = ovr;
            e = launch_scale_pass(p, P->f32, st);
        }
        if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
        first = false;
    }
    if (P->mean_fix && ph_hi == 2 && P->nranks == 1) {   // (distributed: fp_dist_mean_*)
        MeanPass m{};
        for (int k = 0; k < 3; ++k) { m.ext[k] = 1; m.st[k] = 0; }
        for (int a = 0; a < d; ++a) { m.ext[3 - d + a] = (int)P->n[a]; m.st[3 - d + a] = os_s[a]; }
        m.data = out;
        m.partials = mean_ws;
        cudaError_t e = launch_mean_pass(m, P->f32, st);
        if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("mean removal launch failed: ") + cudaGetErrorString(e));
    }
    if (pass_events) CUDA_TRY(cudaEventRecord((cudaEvent_t)pass_events[PL.size()], st));
    while (ev && phase < 3) { ++phase; CUDA_TRY(cudaEventRecord(ev[phase], st)); }
    return FP_OK;
}

FP_API fp_status fp_solve_ex(const fp_plan* P, const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                             void* out, const int64_t* out_strides, void* workspace, size_t workspace_bytes,
                             void* stream, fp_solve_info* dev_info, void* const* phase_events,
                             void* const* pass_events) {
    if (P && P->nranks > 1) return fail(FP_ERR_VALUE, "distributed plan: use fp_solve_phase");
    return solve_impl(P, rhs, rhs_dtype, rhs_strides, out, out_strides, workspace, workspace_bytes, stream,
                      dev_info, phase_events, pass_events, nullptr, 0, 2);
}

FP_API fp_status fp_solve_override(const fp_plan* P, const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                                   void* out, const int64_t* out_strides, void* workspace, size_t workspace_bytes,
                                   void* stream, fp_solve_info* dev_info, void* const* phase_events,
                                   const void* inv_lam) {
    if (P && P->nranks > 1) return fail(FP_ERR_UNSUPPORTED, "_inv_lam override: single-GPU plans only");
    if (!inv_lam) return fail(FP_ERR_VALUE, "inv_lam is NULL");
    return solve_impl(P, rhs, rhs_dtype, rhs_strides, out, out_strides, workspace, workspace_bytes, stream,
                      dev_info, phase_events, nullptr, nullptr, 0, 2, nullptr, inv_lam);
}

FP_API fp_status fp_plan_spectrum(const fp_plan* P, int64_t ext[3], int* r_axis) {
    if (!P || !ext || !r_axis) return fail(FP_ERR_VALUE, "NULL argument");
    for (int a = 0; a < 3; ++a) ext[a] = a < P->ndim ? P->cext[a] : 1;
    *r_axis = P->r_axis;
    return FP_OK;
}

FP_API fp_status fp_solve_mid_rows(const fp_plan* P, int64_t row0, int64_t nrows, void* xbuf, void* workspace,
                                   size_t workspace_bytes, void* stream, fp_solve_info* dev_info) {
    if (!P || P->nranks < 2) return fail(FP_ERR_VALUE, "fp_solve_mid_rows: distributed plans only");
    if (row0 < 0 || nrows < 1 || row0 + nrows > P->B) return fail(FP_ERR_VALUE, "row range outside this rank's block");
    return solve_impl(P, nullptr, 0, nullptr, nullptr, nullptr, workspace, workspace_bytes, stream, dev_info, nullptr,
                      nullptr, xbuf, 1, 1, nullptr, nullptr, row0, nrows);
}

FP_API fp_status fp_solve_phase(const fp_plan* P, int phase, const void* rhs, int rhs_dtype,
                                const int64_t* rhs_strides, void* out, const int64_t* out_strides,
                                void* xbuf, void* workspace, size_t workspace_bytes, void* stream,
                                fp_solve_info* dev_info) {
    if (phase < 0 || phase > 2) return fail(FP_ERR_VALUE, "phase must be 0 (forward), 1 (middle) or 2 (backward)");
    return solve_impl(P, rhs, rhs_dtype, rhs_strides, out, out_strides, workspace, workspace_bytes, stream,
                      dev_info, nullptr, nullptr, xbuf, phase, phase);
}

// ---- projection step of the 2D staggered-grid flow (flow.py:284-295) ----------
static fp_status projection_geometry(const fp_plan* P, double* dx, double* dz, int* w_periodic) {
    if (!P) return fail(FP_ERR_VALUE, "plan is NULL");
    if (P->nranks > 1) return fail(FP_ERR_UNSUPPORTED, "projection step: single-GPU plans only");
    const fp_config& c = P->cfg;
    const bool zp = c.bc[1] == FP_BC_PERIODIC, zw = c.bc[1] == FP_BC_NEUMANN && c.kind[1] == FP_GRID_STAGGERED;
    if (c.ndim != 2 || c.bc[0] != FP_BC_PERIODIC || !(zp || zw))
        return fail(FP_ERR_UNSUPPORTED, "projection step: needs the flow plan (x periodic; z periodic or staggered "
                                        "Neumann walls), flow.py:241-250");
    *dx = c.length[0] / (double)c.n[0];
    *dz = c.length[1] / (double)c.n[1];
    *w_periodic = zp ? 1 : 0;
    return FP_OK;
}

FP_API fp_status fp_solve_divergence(const fp_plan* P, const void* u, const int64_t* u_strides, const void* w,
                                     const int64_t* w_strides, double scale, void* phi, const int64_t* phi_strides,
                                     void* workspace, size_t workspace_bytes, void* stream, fp_solve_info* dev_info) {
    double dx, dz;
    int wp;
    fp_status st = projection_geometry(P, &dx, &dz, &wp);
    if (st != FP_OK) return st;
    if (!u || !w || !phi) return fail(FP_ERR_VALUE, "u/w/phi is NULL");
    if (!(scale != 0.0) || !std::isfinite(scale)) return fail(FP_ERR_VALUE, "scale must be finite and non-zero");
    Producer q{};
    q.u = u;
    q.w = w;
    q.nx = (int)P->n[0];
    q.nz = (int)P->n[1];
    q.w_periodic = wp;
    q.us0 = u_strides ? u_strides[0] : q.nz;
    q.us1 = u_strides ? u_strides[1] : 1;
    q.ws0 = w_strides ? w_strides[0] : (wp ? q.nz : q.nz + 1);
    q.ws1 = w_strides ? w_strides[1] : 1;
    if (q.us0 < 0 || q.us1 < 0 || q.ws0 < 0 || q.ws1 < 0) return fail(FP_ERR_VALUE, "negative strides are not supported");
    q.sx = 1.0 / (dx * scale);
    q.sz = 1.0 / (dz * scale);
    q.active = 0;
    return solve_impl(P, u, P->f32 ? FP_F32 : FP_F64, nullptr, phi, phi_strides, workspace, workspace_bytes, stream,
                      dev_info, nullptr, nullptr, nullptr, 0, 2, &q);
}

FP_API fp_status fp_project_correct(const fp_plan* P, const void* phi, const void* u_star, const void* w_star,
                                    void* u_out, void* w_out, void* p_inout, double scale, void* stream) {
    double dx, dz;
    int wp;
    fp_status st = projection_geometry(P, &dx, &dz, &wp);
    if (st != FP_OK) return st;
    if (!phi || !u_star || !w_star || !u_out || !w_out) return fail(FP_ERR_VALUE, "NULL array");
    DeviceGuard dg(P->device);
    CorrectPass c{};
    c.phi = phi; c.u_in = u_star; c.w_in = w_star; c.u_out = u_out; c.w_out = w_out; c.p = p_inout;
    c.cx = scale / dx;
    c.cz = scale / dz;
    c.nx = (int)P->n[0];
    c.nz = (int)P->n[1];
    c.w_periodic = wp;
    cudaError_t e = launch_correct(c, P->f32, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("corrector launch failed: ") + cudaGetErrorString(e));
    return FP_OK;
}

FP_API fp_status fp_dist_layout(const fp_config* cfg, int nranks, int rank, fp_dist_info* info) {
    if (!info) return fail(FP_ERR_VALUE, "NULL argument");
    fp_status st = validate(cfg);
    if (st != FP_OK) return st;
    if (rank < 0 || rank >= nranks) return fail(FP_ERR_VALUE, "rank out of range");
    DistLayout L{};
    if ((st = dist_layout(cfg, nranks, rank, &L)) != FP_OK) return st;
    std::memset(info, 0, sizeof(*info));
    info->nranks = nranks;
    info->rank = rank;
    info->local_n0 = nranks > 1 ? L.a0 : cfg->n[0];
    info->offset0 = nranks > 1 ? L.off0 : 0;
    info->pitch_n0 = nranks > 1 ? L.A : cfg->n[0];
    info->exch_n1 = nranks > 1 ? L.E1 : 0;
    info->true_n1 = nranks > 1 ? L.e1 : 0;
    info->exch_n2 = nranks > 1 ? L.e2 : 0;
    info->block_n1 = nranks > 1 ? L.B : 0;
    info->exch_complex = L.cpx;
    info->r_axis = L.r_axis;
    const int rb = cfg->precision == FP_F32 ? 4 : 8;
    info->elem_bytes = (L.cpx ? 2 : 1) * rb;
    info->exchange_bytes = nranks > 1 ? (size_t)L.A * L.E1 * L.e2 * info->elem_bytes : 0;
    return FP_OK;
}

FP_API fp_status fp_plan_create_dist(const fp_config* cfg, int device, int nranks, int rank, fp_plan** plan) {
    return build_plan(cfg, device, nranks, rank, plan);
}

// exact mean removal of a distributed DCT-I plan (solver.py:224-225 over the global grid)
static fp_status dist_mean_pass(const fp_plan* P, void* out_local, const int64_t* out_strides, MeanPass& m) {
    if (!P || !out_local) return fail(FP_ERR_VALUE, "NULL argument");
    const int d = P->ndim;
    long long dense[3];
    dense_strides(P, false, dense);
    for (int k = 0; k < 3; ++k) { m.ext[k] = 1; m.st[k] = 0; }
    for (int a = 0; a < d; ++a) {
        m.ext[3 - d + a] = (int)P->n[a];
        m.st[3 - d + a] = out_strides ? out_strides[a] : dense[a];
    }
    m.data = out_local;
    return FP_OK;
}

FP_API fp_status fp_dist_mean_partial(const fp_plan* P, void* out_local, const int64_t* out_strides, void* workspace,
                                      size_t workspace_bytes, void* stream, double* dev_sum) {
    MeanPass m{};
    fp_status st = dist_mean_pass(P, out_local, out_strides, m);
    if (st != FP_OK) return st;
    if (!dev_sum) return fail(FP_ERR_VALUE, "dev_sum is NULL");
    if (!workspace || workspace_bytes < mean_bytes(P) || !P->mean_fix)
        return fail(FP_ERR_VALUE, "fp_dist_mean_partial: plan without exact mean removal, or workspace too small");
    DeviceGuard dg(P->device);
    m.partials = (double*)workspace;
    m.sum_out = dev_sum;
    cudaError_t e = launch_mean_pass(m, P->f32, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("mean partial launch failed: ") + cudaGetErrorString(e));
    return FP_OK;
}

FP_API fp_status fp_dist_mean_subtract(const fp_plan* P, void* out_local, const int64_t* out_strides,
                                       const double* dev_total, void* stream) {
    MeanPass m{};
    fp_status st = dist_mean_pass(P, out_local, out_strides, m);
    if (st != FP_OK) return st;
    if (!dev_total) return fail(FP_ERR_VALUE, "dev_total is NULL");
    DeviceGuard dg(P->device);
    double N = 1.0;
    for (int a = 0; a < P->ndim; ++a) N *= (double)P->cfg.n[a];   // global point count
    m.mean_in = dev_total;
    m.inv_total = 1.0 / N;
    cudaError_t e = launch_mean_pass(m, P->f32, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("mean subtract launch failed: ") + cudaGetErrorString(e));
    return FP_OK;
}

FP_API fp_status fp_removed_mean(const fp_plan* P, const fp_solve_info* h, double* rm) {
    if (!P || !h || !rm) return fail(FP_ERR_VALUE, "NULL argument");
    if (!P->singular) { *rm = 0.0; return FP_OK; }
    // reference: Re(fftn(work)/prod n_p)[null] / _null_scale
    *rm = (h->dc / P->np_prod) / P->null_scale;
    return FP_OK;
}

FP_API fp_status fp_solve_host(const fp_plan* P, const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                               void* out, const int64_t* out_strides, fp_solve_result* result) {
    if (!P || !rhs || !out) return fail(FP_ERR_VALUE, "NULL argument");
    if (rhs_dtype != FP_F64 && rhs_dtype != FP_F32) return fail(FP_ERR_VALUE, "rhs dtype must be f64 or f32");
    DeviceGuard dg(P->device);
    const int d = P->ndim;
    size_t cnt = 1;
    for (int a = 0; a < d; ++a) cnt *= (size_t)P->n[a];
    const size_t in_es = rhs_dtype == FP_F32 ? 4 : 8;
    const size_t out_es = P->f32 ? 4 : 8;
    long long dense_r[3];
    dense_strides(P, false, dense_r);
    // pack host arrays to dense C order (host-side gather for strided views)
    auto is_dense = [&](const int64_t* s) {
        if (!s) return true;
        for (int a = 0; a < d; ++a) if (P->n[a] > 1 && s[a] != dense_r[a]) return false;
        return true;
    };
    std::vector<unsigned char> in_pack, out_pack;
    const unsigned char* hin = (const unsigned char*)rhs;
    if (!is_dense(rhs_strides)) {
        in_pack.resize(cnt * in_es);
        size_t idx = 0;
        for (long long i0 = 0; i0 < (d > 0 ? P->n[0] : 1); ++i0)
            for (long long i1 = 0; i1 < (d > 1 ? P->n[1] : 1); ++i1)
                for (long long i2 = 0; i2 < (d > 2 ? P->n[2] : 1); ++i2, ++idx) {
                    long long off = i0 * rhs_strides[0] + (d > 1 ? i1 * rhs_strides[1] : 0) + (d > 2 ? i2 * rhs_strides[2] : 0);
                    std::memcpy(&in_pack[idx * in_es], hin + off * in_es, in_es);
                }
        hin = in_pack.data();
    }
    cudaStream_t st;
    CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t ev[6];
    for (int i = 0; i < 6; ++i) CUDA_TRY(cudaEventCreate(&ev[i]));
    size_t ws = 0;
    fp_plan_workspace_bytes(P, 1, &ws);
    void *din = nullptr, *dout = nullptr, *dws = nullptr, *dinfo = nullptr;
    fp_status rc = FP_OK;
    fp_solve_info hinfo{};
    CUDA_TRY(cudaEventRecord(ev[4], st));
    if (cudaMallocAsync(&din, cnt * in_es, st) != cudaSuccess || cudaMallocAsync(&dout, cnt * out_es, st) != cudaSuccess ||
        cudaMallocAsync(&dinfo, sizeof(fp_solve_info), st) != cudaSuccess ||
        (ws && cudaMallocAsync(&dws, ws, st) != cudaSuccess)) {
        rc = fail(FP_ERR_ALLOC, "device allocation failed");
    }
    if (rc == FP_OK && cudaMemcpyAsync(din, hin, cnt * in_es, cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = fail(FP_ERR_CUDA, "H2D copy failed");
    if (rc == FP_OK)
        rc = fp_solve(P, din, rhs_dtype, nullptr, dout, nullptr, dws, ws, st, (fp_solve_info*)dinfo, (void* const*)ev);
    if (rc == FP_OK && cudaMemcpyAsync(&hinfo, dinfo, sizeof(hinfo), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(FP_ERR_CUDA, "D2H info copy failed");
    if (rc == FP_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(FP_ERR_CUDA, "solve failed");
    if (rc == FP_OK && hinfo.nonfinite) rc = fail(FP_ERR_NONFINITE, "rhs contains non-finite values");
    if (rc == FP_OK) {
        if (is_dense(out_strides)) {
            if (cudaMemcpyAsync(out, dout, cnt * out_es, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = fail(FP_ERR_CUDA, "D2H copy failed");
        } else {
            out_pack.resize(cnt * out_es);
            if (cudaMemcpyAsync(out_pack.data(), dout, cnt * out_es, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = fail(FP_ERR_CUDA, "D2H copy failed");
        }
    }
    CUDA_TRY(cudaEventRecord(ev[5], st));
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == FP_OK) rc = fail(FP_ERR_CUDA, "D2H failed");
    if (rc == FP_OK && !out_pack.empty()) {
        unsigned char* hout = (unsigned char*)out;
        size_t idx = 0;
        for (long long i0 = 0; i0 < (d > 0 ? P->n[0] : 1); ++i0)
            for (long long i1 = 0; i1 < (d > 1 ? P->n[1] : 1); ++i1)
                for (long long i2 = 0; i2 < (d > 2 ? P->n[2] : 1); ++i2, ++idx) {
                    long long off = i0 * out_strides[0] + (d > 1 ? i1 * out_strides[1] : 0) + (d > 2 ? i2 * out_strides[2] : 0);
                    std::memcpy(hout + off * out_es, &out_pack[idx * out_es], out_es);
                }
    }
    if (rc == FP_OK && result) {
        float ms[4] = {0, 0, 0, 0};
        cudaEventElapsedTime(&ms[0], ev[0], ev[1]);
        cudaEventElapsedTime(&ms[1], ev[1], ev[2]);
        cudaEventElapsedTime(&ms[2], ev[2], ev[3]);
        cudaEventElapsedTime(&ms[3], ev[4], ev[5]);
        for (int i = 0; i < 3; ++i) result->timing[i] = ms[i] * 1e-3;
        result->total_seconds = ms[3] * 1e-3;
        fp_removed_mean(P, &hinfo, &result->removed_mean);
    }
    if (din) cudaFreeAsync(din, st);
    if (dout) cudaFreeAsync(dout, st);
    if (dws) cudaFreeAsync(dws, st);
    if (dinfo) cudaFreeAsync(dinfo, st);
    cudaStreamSynchronize(st);
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
    cudaStreamDestroy(st);
    return rc;
}

// ---------------------------------------------------------------------------
// TransformPlan (transforms.py:128-177) on the device
FP_API fp_status fp_transform_create(int kind, int64_t n, int precision, int device, fp_transform** out) {
    if (!out) return fail(FP_ERR_VALUE, "NULL argument");
    *out = nullptr;
    if (kind < FP_DFT || kind > FP_DCT3) return fail(FP_ERR_VALUE, "unknown transform kind");
    const long long min_len = kind == FP_DCT1 ? 2 : 1;
    if (n < min_len) return fail(FP_ERR_CONFIG, "transform length too small");
    if (precision != FP_F64 && precision != FP_F32) return fail(FP_ERR_VALUE, "precision must be f64 or f32");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(FP_ERR_CUDA, "no CUDA device available");
    DeviceGuard dg(device);
    fp_transform* T = new fp_transform();
    T->device = device;
    T->kind = kind;
    T->n = n;
    T->f32 = precision == FP_F32;
    long long M = 0;
    if (kind == FP_DFT || kind == FP_IDFT) M = n;
    else if (kind == FP_DST2 || kind == FP_DST3 || kind == FP_DCT2 || kind == FP_DCT3) M = (n % 2 == 0) ? n / 2 : 0;
    else if (kind == FP_DCT1) M = n - 1;   // real FFT of the 2M-point even extension
    else if (kind == FP_DST1) M = n + 1;   // ... of the odd extension
    T->fft = M >= 16 && M <= kFftMax && is_pow2(M);
    fp_status st;
    if (T->fft) {
        T->M = (int)M;
        std::vector<long double> wf, wt, ww;
        fft_tables((kind == FP_DCT1 || kind == FP_DST1) ? 2 * (int)M : (int)n, (int)M, !(kind == FP_DFT || kind == FP_IDFT),
                   wf, wt, ww);
        if ((st = upload(T->allocs, wf, T->f32, &T->tab.wfft)) != FP_OK) { delete T; return st; }
        if ((st = upload(T->allocs, wt, T->f32, &T->tab.wt)) != FP_OK) { delete T; return st; }
        if ((st = upload(T->allocs, ww, T->f32, &T->tab.ww)) != FP_OK) { delete T; return st; }
    } else {
        if ((st = mr_setup(T->allocs, T->tab, kind, n, T->f32)) != FP_OK) { delete T; return st; }
        if (T->tab.mr) { *out = T; return FP_OK; }
        if (n > kDenseMax || n >= blue_min_length()) {   // Bluestein
            T->tab.fwd_kind = kind;
            if ((st = blue_setup(T->allocs, T->tab, kind, n, T->f32)) != FP_OK) { delete T; return st; }
            *out = T;
            return FP_OK;
        }
        std::vector<double> m;
        int no, ni;
        bool cpx;
        dense_matrix(kind, (int)n, m, &no, &ni, &cpx);
        T->tab.fwd_nout = no; T->tab.fwd_nin = ni; T->tab.fwd_cpx = cpx;
        if ((st = upload(T->allocs, m, T->f32, &T->tab.mat_f)) != FP_OK) { delete T; return st; }
    }
    *out = T;
    return FP_OK;
}

FP_API fp_status fp_transform_destroy(fp_transform* t) {
    delete t;
    return FP_OK;
}

FP_API fp_status fp_transform_execute(const fp_transform* T, int ndim, const int64_t* shape, int axis,
                                      const void* in, int in_dtype, const int64_t* in_strides, void* out,
                                      int out_dtype, const int64_t* out_strides, void* stream) {
    if (!T || !shape || !in || !out || !in_strides || !out_strides) return fail(FP_ERR_VALUE, "NULL argument");
    if (ndim < 1 || ndim > 3) return fail(FP_ERR_VALUE, "1 to 3 dimensions supported");
    if (axis < 0 || axis >= ndim) return fail(FP_ERR_VALUE, "axis out of range");
    if (shape[axis] != T->n) return fail(FP_ERR_VALUE, "plan length does not match the array along axis");
    const bool cpx_kind = T->kind == FP_DFT || T->kind == FP_IDFT;
    const bool out_c = out_dtype == FP_C128 || out_dtype == FP_C64;
    if (cpx_kind != out_c) return fail(FP_ERR_VALUE, "output dtype does not match the transform kind");
    if (!cpx_kind && (in_dtype == FP_C128 || in_dtype == FP_C64)) return fail(FP_ERR_VALUE, "real transform of complex data");
    {   // operands must be in the transform precision (complex kinds: complex input)
        const int want_in = cpx_kind ? (T->f32 ? FP_C64 : FP_C128) : (T->f32 ? FP_F32 : FP_F64);
        if (in_dtype != want_in || out_dtype != want_in)
            return fail(FP_ERR_VALUE, "operand dtypes must match the transform precision (complex kinds take complex input)");
    }
    DeviceGuard dg(T->device);
    int o[2] = {-1, -1}, k = 0;
    for (int a = 0; a < ndim; ++a) if (a != axis) o[k++] = a;
    int aa = -1, bb = -1;
    if (k == 2) { aa = o[0]; bb = o[1]; } else if (k == 1) { bb = o[0]; }
    Geometry g{};
    g.na = aa >= 0 ? (int)shape[aa] : 1;
    g.nb = bb >= 0 ? (int)shape[bb] : 1;
    g.in = in; g.out = out;
    g.in_type = in_dtype; g.out_type = out_dtype;
    g.in_st = in_strides[axis]; g.out_st = out_strides[axis];
    g.in_sa = aa >= 0 ? in_strides[aa] : 0; g.out_sa = aa >= 0 ? out_strides[aa] : 0;
    g.in_sb = bb >= 0 ? in_strides[bb] : 0; g.out_sb = bb >= 0 ? out_strides[bb] : 0;
    const double om = (T->kind == FP_DFT) ? 1.0 / (double)T->n : 1.0;
    cudaError_t e;
    if ((long long)g.na * g.nb == 0) return FP_OK;
    if (T->fft) {
        FftPass p{};
        const bool inv = T->kind == FP_IDFT || T->kind == FP_DST3 || T->kind == FP_DCT3;
        p.op = inv ? OP_INV : OP_FWD;
        p.fkind = T->kind == FP_DFT ? FK_CFFT
                : T->kind == FP_DST2 ? FK_DST2 : T->kind == FP_DCT1 ? FK_DCT1 : T->kind == FP_DST1 ? FK_DST1 : FK_DCT2;
        p.ikind = T->kind == FP_IDFT ? IK_ICFFT : (T->kind == FP_DST3 ? IK_DST3 : IK_DCT3);
        p.family = (axis == ndim - 1) ? FAM_CONTIG : FAM_STRIDED;
        p.n = (int)T->n;
        p.M = T->M;
        p.logM = ilog2(T->M);
        p.ls = p.M + p.M / 16 + 1;
        if ((p.ls & 1) == 0) p.ls += 1;
        const bool in_c = in_dtype == FP_C128 || in_dtype == FP_C64;
        fft_tile_shape(p, T->f32, in_c || cpx_kind, g.na, g.nb);
        p.g = g;
        p.wfft = T->tab.wfft; p.wt = T->tab.wt; p.ww = T->tab.ww;
        p.out_mult = om;
        p.vec_in = 0; p.vec_out = 0;
        p.nonfinite = nullptr;
        p.s = Scaling{};
        e = launch_fft_pass(p, T->f32, (cudaStream_t)stream);
    } else if (T->tab.blue) {
        // scratch from the stream-ordered allocator (the transform API has no workspace)
        BluePass p = blue_pass(T->tab, T->kind, T->n, g.na, g.nb);
        p.g = g;
        p.out_mult = om;
        const size_t sb = blue_scratch_bytes(T->tab, (long long)g.na * g.nb, T->f32);
        void* S = nullptr;
        cudaStream_t s = (cudaStream_t)stream;
        e = cudaMallocAsync(&S, sb, s);
        if (e == cudaSuccess) {
            e = run_blue(T->tab, p, S, sb, T->f32, s);
            const cudaError_t e2 = cudaFreeAsync(S, s);
            if (e == cudaSuccess) e = e2;
        }
    } else if (T->tab.mr) {
        MrPass p = mr_pass(T->tab, T->kind, T->n, g.na, g.nb, T->f32, g.in_st != 1);
        p.g = g;
        p.out_mult = om;
        p.nonfinite = nullptr;
        e = launch_mr_pass(p, T->f32, (cudaStream_t)stream);
    } else {
        DensePass p{};
        const bool in_c = in_dtype == FP_C128 || in_dtype == FP_C64;
        p.cls = cpx_kind ? DC_C2C : DC_R2R;
        p.n_in = T->tab.fwd_nin; p.n_out = T->tab.fwd_nout;
        p.mat = T->tab.mat_f;
        p.g = g;
        if (cpx_kind && !in_c) {
            // real data into the complex dense transform: the kernel widens on load
            p.cls = DC_C2C;
        }
        p.in_ls = (p.cls == DC_R2R) ? p.n_in : 2 * p.n_in;
        const int rb = T->f32 ? 4 : 8;
        int lines = std::max(1, (48 * 1024) / (p.in_ls * rb));
        lines = std::min(lines, 64);
        const long long nl = (long long)g.na * g.nb;
        if (lines > nl) lines = (int)nl;
        p.lines = lines;
        p.tiles = (int)((nl + lines - 1) / lines);
        p.out_mult = om;
        p.nonfinite = nullptr;
        e = launch_dense_pass(p, T->f32, (cudaStream_t)stream);
    }
    if (e != cudaSuccess) return fail(FP_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
    return FP_OK;
}

FP_API fp_status fp_event_create(void** event) {
    if (!event) return fail(FP_ERR_VALUE, "NULL argument");
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    *event = (void*)e;
    return FP_OK;
}

FP_API fp_status fp_event_create_on(int device, void** event) {
    if (!event) return fail(FP_ERR_VALUE, "NULL argument");
    DeviceGuard dg(device);
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    *event = (void*)e;
    return FP_OK;
}

FP_API fp_status fp_event_destroy(void* event) {
    if (event) CUDA_TRY(cudaEventDestroy((cudaEvent_t)event));
    return FP_OK;
}

FP_API fp_status fp_event_elapsed_ms(void* start, void* stop, float* ms) {
    if (!start || !stop || !ms) return fail(FP_ERR_VALUE, "NULL argument");
    CUDA_TRY(cudaEventSynchronize((cudaEvent_t)stop));
    CUDA_TRY(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
    return FP_OK;
}

}  // extern "C"
