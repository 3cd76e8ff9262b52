/*
 * fastpoisson_b200.h -- C ABI of the B200-native PoisFFT solve path.
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json
 * (`SolverPlan.solve`, /root/reference/pkg/src/fastpoisson/solver.py:191-230).
 * Every entry point takes plain pointers, sizes and integer enums; no torch or
 * numpy type crosses it.  The Python host mirror (paper_1409_8116_b200/solver.py)
 * binds it with ctypes; any other host can do the same.
 *
 * Reference interface replaced by each entry point (file:line in the reference):
 *   fp_plan_create      SolverPlan.__init__            solver.py:136-181
 *                       SolverConfig.__post_init__      solver.py:73-91
 *                       GridSpec.__post_init__          grid.py:64-78
 *   fp_plan_destroy     (Python GC of SolverPlan)
 *   fp_plan_info        SolverConfig.mode/singular/periodic_axes  solver.py:105-119
 *   fp_plan_workspace_bytes  per-call workspace of solve  solver.py:213 (work copy)
 *   fp_solve            SolverPlan.solve (device buffers, async)  solver.py:191-230
 *   fp_solve_ex         same, with per-kernel CUDA events (bench / profiling)
 *   fp_solve_override   same, dividing by the caller's dense `_inv_lam` table instead
 *                       of the plan's eigenvalues (SolverPlan._inv_lam mutated for
 *                       fault injection, verifysuite.py:83-88; solver.py:151-159,221)
 *   fp_plan_spectrum    extents of that table (the half spectrum)  solver.py:147-159
 *   fp_solve_host       SolverPlan.solve (host buffers, sync)     solver.py:191-230
 *   fp_removed_mean     SolveReport.removed_mean        solver.py:218-220
 *   fp_transform_create TransformPlan(kind, n)          transforms.py:128-146
 *   fp_transform_execute TransformPlan.execute_real/_complex transforms.py:157-172
 *   fp_last_error       exception message of the failing call
 *   fp_event_*          CUDA events behind SolveReport.timing (solver.py:215-228)
 *   fp_solve_divergence ProjectionFlow stage: rhs = divergence(star)/(alpha dt),
 *                       poisson.solve(rhs)              flow.py:114-122, 290-291
 *   fp_project_correct  u, w -= alpha dt gradient(phi); p += phi   flow.py:125-139, 292-295
 *   fp_plan_create_dist / fp_solve_phase / fp_dist_layout
 *                       slab-decomposed solve over P ranks (the paper's MPI
 *                       global transposes; the reorder seam
 *                       "where a distributed exchange would slot in", reorder.py:7-8)
 *
 * Conventions
 *   - Arrays are C order (last axis contiguous) unless strides say otherwise;
 *     strides are in ELEMENTS of the array's own dtype and must be >= 0.
 *   - fp_solve is asynchronous and stream-ordered on `stream` (a cudaStream_t,
 *     NULL = legacy default stream).  It never allocates: the caller passes a
 *     workspace of at least fp_plan_workspace_bytes() bytes.
 *   - Plans are immutable after creation; fp_solve on one plan from several
 *     host threads is safe with distinct out/workspace/info buffers.
 *   - `out` may be the same buffer as `rhs` (identical strides): in-place solve.
 *   - Non-finite rhs values are detected on the device (flag in fp_solve_info);
 *     fp_solve_host returns FP_ERR_NONFINITE before writing the host `out`.
 */
#ifndef FASTPOISSON_B200_H
#define FASTPOISSON_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FP_API __attribute__((visibility("default")))
#else
#define FP_API
#endif

#define FP_ABI_VERSION 1

typedef enum fp_status {
    FP_OK = 0,
    FP_ERR_CONFIG = 1,      /* ConfigurationError (grid.py:18-19)            */
    FP_ERR_VALUE = 2,       /* ValueError: extents / strides / dtype         */
    FP_ERR_UNSUPPORTED = 3, /* valid config this build cannot run            */
    FP_ERR_CUDA = 4,        /* CUDA runtime failure                          */
    FP_ERR_NONFINITE = 5,   /* ValueError("rhs contains non-finite values")  */
    FP_ERR_ALLOC = 6        /* MemoryError                                   */
} fp_status;

/* BoundaryCondition (grid.py:22-25) */
enum { FP_BC_PERIODIC = 0, FP_BC_DIRICHLET = 1, FP_BC_NEUMANN = 2 };
/* GridKind (grid.py:28-30) */
enum { FP_GRID_REGULAR = 0, FP_GRID_STAGGERED = 1 };
/* Approximation (grid.py:33-37) */
enum { FP_APPROX_SPECTRAL = 0, FP_APPROX_FD2 = 1 };
/* element types */
enum { FP_F64 = 0, FP_F32 = 1, FP_C128 = 2, FP_C64 = 3 };
/* TransformKind (transforms.py:52-64) */
enum {
    FP_DFT = 0, FP_IDFT = 1,
    FP_DST1 = 2, FP_DST2 = 3, FP_DST3 = 4,
    FP_DCT1 = 5, FP_DCT2 = 6, FP_DCT3 = 7
};

/* SolverConfig: grids (GridSpec per axis) + approximation + precision. */
typedef struct fp_config {
    int ndim;               /* 1..3 */
    int64_t n[3];           /* GridSpec.n      */
    double length[3];       /* GridSpec.length */
    int bc[3];              /* FP_BC_*         */
    int kind[3];            /* FP_GRID_*       */
    int approx;             /* FP_APPROX_*     */
    int precision;          /* FP_F64 ("double") or FP_F32 ("single") */
    /* Optional per-axis eigenvalue tables (n[a] doubles each), e.g. the host
     * mirror's numpy tables; NULL = computed by the library (eigenvalues.py:51-83). */
    const double* eig[3];
} fp_config;

typedef struct fp_plan fp_plan;
typedef struct fp_transform fp_transform;

typedef struct fp_plan_info {
    int ndim;
    int mode_mixed;         /* SolverConfig.mode == "mixed" */
    int singular;           /* SolverConfig.singular        */
    int periodic_mask;      /* bit a set <=> axis a periodic */
    double null_scale;      /* _null_scale * prod(n_periodic) (solver.py:177-181,239) */
    int num_passes;         /* kernel launches per solve     */
    int middle_axis;        /* axis of the fused forward/scale/inverse pass */
    int fft_axes_mask;      /* axes on the FFT engine (others: dense engine) */
    int exact_mean;         /* DCT-I plan: explicit arithmetic-mean removal after the backward pass */
} fp_plan_info;

/* Device-side per-solve record written by the kernels. */
typedef struct fp_solve_info {
    double dc;              /* raw null-mode coefficient (before scaling) */
    int32_t nonfinite;      /* != 0 if rhs held NaN/Inf                   */
    int32_t reserved;
} fp_solve_info;

typedef struct fp_solve_result {
    double removed_mean;
    double timing[3];       /* forward, diagonal, backward (seconds) */
    double total_seconds;   /* including host<->device copies        */
} fp_solve_result;

FP_API int fp_abi_version(void);
FP_API const char* fp_last_error(void);

FP_API fp_status fp_plan_create(const fp_config* cfg, int device, fp_plan** plan);
FP_API fp_status fp_plan_destroy(fp_plan* plan);
FP_API fp_status fp_plan_info_get(const fp_plan* plan, fp_plan_info* info);
/* out_dense != 0: the caller promises `out` is a dense C-order array that the
 * solve may use as its real-valued scratch (smaller workspace). */
FP_API fp_status fp_plan_workspace_bytes(const fp_plan* plan, int out_dense, size_t* bytes);
/* same, for fp_solve_override when inv_lam_override != 0 */
FP_API fp_status fp_plan_workspace_bytes_ex(const fp_plan* plan, int out_dense, int inv_lam_override,
                                            size_t* bytes);
/* Spectral extents of the solve's middle state (ext[a] = n[a], except the real-FFT
 * periodic axis r_axis: n/2 + 1; r_axis = -1 when no axis is periodic). */
FP_API fp_status fp_plan_spectrum(const fp_plan* plan, int64_t ext[3], int* r_axis);

/* Asynchronous device solve.  rhs_dtype: FP_F64 or FP_F32 (cast on load);
 * out has the plan precision.  dev_info: device memory (zeroed by the call).
 * phase_events: NULL or 4 cudaEvent_t recorded at start / after forward /
 * after diagonal / end (SolveReport.timing keys, solver.py:215-228). */
FP_API fp_status fp_solve(const fp_plan* plan,
                          const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                          void* out, const int64_t* out_strides,
                          void* workspace, size_t workspace_bytes,
                          void* stream, fp_solve_info* dev_info,
                          void* const* phase_events);

/* fp_solve plus per-kernel events: pass_events (NULL or fp_plan_info.num_passes+1
 * cudaEvent_t) are recorded before every kernel and after the last one. */
FP_API fp_status fp_solve_ex(const fp_plan* plan,
                             const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                             void* out, const int64_t* out_strides,
                             void* workspace, size_t workspace_bytes,
                             void* stream, fp_solve_info* dev_info,
                             void* const* phase_events, void* const* pass_events);

/* fp_solve with the reference's dense diagonal: inv_lam is device memory in the
 * plan precision, C order over fp_plan_spectrum's extents, holding
 * backward_scale / lambda (0 on null modes) at every half-spectrum index --
 * for periodic axes the Hermitian average (f(k) + f(-k)) / 2 of the full
 * table, which is what `.real` of the inverse FFT keeps (solver.py:245-246).
 * The middle axis then runs as forward pass + scale + inverse pass. */
FP_API fp_status fp_solve_override(const fp_plan* plan,
                                   const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                                   void* out, const int64_t* out_strides,
                                   void* workspace, size_t workspace_bytes,
                                   void* stream, fp_solve_info* dev_info,
                                   void* const* phase_events, const void* inv_lam);

/* Synchronous host-buffer solve (H2D, fp_solve, D2H); returns FP_ERR_NONFINITE
 * without touching `out` when rhs holds NaN/Inf. */
FP_API fp_status fp_solve_host(const fp_plan* plan,
                               const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                               void* out, const int64_t* out_strides,
                               fp_solve_result* result);

/* removed_mean from a host copy of the device record (solver.py:218-220). */
FP_API fp_status fp_removed_mean(const fp_plan* plan, const fp_solve_info* host_info,
                                 double* removed_mean);

/* 1D transform of one kind and length along `axis` of an up-to-3D array. */
FP_API fp_status fp_transform_create(int kind, int64_t n, int precision, int device,
                                     fp_transform** t);
FP_API fp_status fp_transform_destroy(fp_transform* t);
FP_API fp_status fp_transform_execute(const fp_transform* t, int ndim, const int64_t* shape,
                                      int axis,
                                      const void* in, int in_dtype, const int64_t* in_strides,
                                      void* out, int out_dtype, const int64_t* out_strides,
                                      void* stream);

/* ---- projection step of the 2D staggered-grid flow (flow.py:284-295) ----------
 * For the flow's plan (axis 0 = x periodic; axis 1 = z periodic or staggered
 * Neumann walls), with cells (nx, nz), u on x-faces (nx, nz), w on z-faces (nx, nz)
 * periodic / (nx, nz + 1) walls, all plan-typed device arrays:
 *   fp_solve_divergence: phi = solve(div(u, w) / scale); the divergence is formed by
 *     the first pass while it loads its lines (no rhs array), or by a stand-alone
 *     kernel when the z axis is on the dense engine.  Same workspace / dev_info /
 *     stream rules as fp_solve.  NULL strides = dense C order.
 *   fp_project_correct: u_out = u_star - scale * d_x phi, w_out = w_star - scale * d_z phi
 *     (wall faces keep w_star), p_inout += phi if non-NULL; dense arrays, in place allowed. */
FP_API fp_status fp_solve_divergence(const fp_plan* plan, const void* u, const int64_t* u_strides,
                                     const void* w, const int64_t* w_strides, double scale,
                                     void* phi, const int64_t* phi_strides,
                                     void* workspace, size_t workspace_bytes, void* stream,
                                     fp_solve_info* dev_info);
FP_API fp_status fp_project_correct(const fp_plan* plan, const void* phi, const void* u_star,
                                    const void* w_star, void* u_out, void* w_out, void* p_inout,
                                    double scale, void* stream);

/* ---- slab decomposition over P ranks (axis 0 split; one all-to-all each way) ----
 * Any P <= n0: rank r owns planes [offset0, offset0 + local_n0) of axis 0, a balanced
 * split (the first n0 % P ranks hold one plane more; local arrays are (local_n0, n1,
 * n2) with any strides).  Axis 0 must be on the FFT engine (power-of-two length); a
 * wall axis 0 may follow periodic local axes (its MID then runs on the real view of
 * the complex state); DCT-I axes are single-GPU only.  A solve is three phases with two
 * all-to-alls of exchange_bytes between them, done by the caller (NCCL):
 *   fp_solve_phase(plan, 0, rhs_local, ..., xbuf=send)    local transforms, packed send
 *   all_to_all(send -> recv)                              equal blocks of exchange_bytes/P
 *   fp_solve_phase(plan, 1, ..., xbuf=recv)               MID along the global axis 0
 *   all_to_all(recv -> send)
 *   fp_solve_phase(plan, 2, ..., out_local, xbuf=send)    local inverse transforms
 * The exchange buffer holds (pitch_n0, exch_n1, exch_n2) elements with axis 1
 * outermost (exch_n1 = n1 or its half spectrum, padded to a multiple of P; planes
 * >= local_n0 of a block are padding).
 * Only rank 0's dev_info receives the null coefficient. */
typedef struct fp_dist_info {
    int nranks, rank;
    int64_t local_n0;       /* planes of axis 0 owned by this rank */
    int64_t offset0;        /* first global plane */
    int64_t exch_n1;        /* padded extent of axis 1 in the exchanged state */
    int64_t true_n1;        /* its true extent */
    int64_t exch_n2;        /* extent of axis 2 in the exchanged state (1 for 2D) */
    int64_t block_n1;       /* exch_n1 / nranks */
    int exch_complex;       /* exchanged state is complex (half spectrum) */
    int r_axis;             /* periodic axis transformed as a real FFT (-1: none) */
    int elem_bytes;
    size_t exchange_bytes;  /* size of the send and of the receive buffer */
    int64_t pitch_n0;       /* planes per rank block in the exchange buffers (max local_n0) */
} fp_dist_info;

FP_API fp_status fp_dist_layout(const fp_config* cfg, int nranks, int rank, fp_dist_info* info); /* no device */
FP_API fp_status fp_plan_create_dist(const fp_config* cfg, int device, int nranks, int rank, fp_plan** plan);
/* DCT-I plans (fp_plan_info.exact_mean) over ranks: after phase 2 the caller removes the
 * GLOBAL arithmetic mean (solver.py:224-225): fp_dist_mean_partial writes this rank's sum of
 * out_local into *dev_sum (device double; workspace from fp_plan_workspace_bytes), the
 * caller all-reduces it (SUM), fp_dist_mean_subtract subtracts dev_total / (n0 n1 n2). */
FP_API fp_status fp_dist_mean_partial(const fp_plan* plan, void* out_local, const int64_t* out_strides,
                                      void* workspace, size_t workspace_bytes, void* stream, double* dev_sum);
FP_API fp_status fp_dist_mean_subtract(const fp_plan* plan, void* out_local, const int64_t* out_strides,
                                       const double* dev_total, void* stream);
/* Phase 1 over a chunk of this rank's axis-1 rows [row0, row0 + nrows) of its block
 * (0 <= row0, row0 + nrows <= exch_n1 / P): the exchange can be pipelined per chunk of
 * rows -- chunk c's MID while chunk c+1's all-to-all is in flight.  Row chunk c of every
 * peer block is a contiguous piece of the exchange buffers (rows are outermost in a block). */
FP_API fp_status fp_solve_mid_rows(const fp_plan* plan, int64_t row0, int64_t nrows, void* xbuf,
                                   void* workspace, size_t workspace_bytes, void* stream,
                                   fp_solve_info* dev_info);
FP_API fp_status fp_solve_phase(const fp_plan* plan, int phase,
                                const void* rhs, int rhs_dtype, const int64_t* rhs_strides,
                                void* out, const int64_t* out_strides, void* xbuf,
                                void* workspace, size_t workspace_bytes, void* stream,
                                fp_solve_info* dev_info);

/* CUDA event helpers for SolveReport.timing (phase_events of fp_solve). */
FP_API fp_status fp_event_create(void** event);      /* on the current device */
/* same, on `device` (events must live on the device of the stream they are recorded on) */
FP_API fp_status fp_event_create_on(int device, void** event);
FP_API fp_status fp_event_destroy(void* event);
FP_API fp_status fp_event_elapsed_ms(void* start, void* stop, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* FASTPOISSON_B200_H */
