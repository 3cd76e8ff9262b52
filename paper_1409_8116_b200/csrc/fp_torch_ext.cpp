// fp_torch_ext.cpp -- the PyTorch extension in front of the C ABI (include/fastpoisson_b200.h).
//
// The solve enters native code as torch.ops.fastpoisson_b200.solve(plan, rhs, out, workspace,
// info, events, override): tensors in, the C ABI's plain pointers / strides / stream out.
// It replaces the per-call ctypes marshalling of `SolverPlan.solve`
// (/root/reference/pkg/src/fastpoisson/solver.py:191-230 is the call it stands in for).
//
// The extension does not link the kernel library: Python hands it the addresses of
// fp_solve / fp_solve_override of the library instance it loaded (bind), so one process
// never holds two copies of the library's state.
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/library.h>

#include <atomic>
#include <cstdint>

namespace {

using SolveFn = int (*)(const void* plan, const void* rhs, int rhs_dtype, const int64_t* rhs_strides, void* out,
                        const int64_t* out_strides, void* workspace, size_t workspace_bytes, void* stream,
                        void* dev_info, void* const* phase_events);
using SolveOverrideFn = int (*)(const void* plan, const void* rhs, int rhs_dtype, const int64_t* rhs_strides, void* out,
                                const int64_t* out_strides, void* workspace, size_t workspace_bytes, void* stream,
                                void* dev_info, void* const* phase_events, const void* inv_lam);

std::atomic<SolveFn> g_solve{nullptr};
std::atomic<SolveOverrideFn> g_solve_override{nullptr};

constexpr int kF64 = 0, kF32 = 1;   // FP_F64 / FP_F32

void bind(int64_t solve_addr, int64_t solve_override_addr) {
    g_solve.store(reinterpret_cast<SolveFn>(static_cast<intptr_t>(solve_addr)));
    g_solve_override.store(reinterpret_cast<SolveOverrideFn>(static_cast<intptr_t>(solve_override_addr)));
}

void fill_strides(const at::Tensor& t, int64_t* s) {
    TORCH_CHECK(t.dim() >= 1 && t.dim() <= 3, "fastpoisson_b200::solve: 1 to 3 dimensions");
    for (int i = 0; i < 3; ++i) s[i] = i < t.dim() ? t.stride(i) : 0;
}

// returns the fp_status of the launch (0 = enqueued); the caller maps it to the
// reference's exception types with fp_last_error
int64_t solve(int64_t plan, const at::Tensor& rhs, at::Tensor out, at::Tensor workspace, at::Tensor info,
              int64_t phase_events, const c10::optional<at::Tensor>& inv_lam) {
    SolveFn fn = g_solve.load();
    TORCH_CHECK(fn != nullptr, "fastpoisson_b200: extension not bound to the native library");
    TORCH_CHECK(rhs.is_cuda() && out.is_cuda() && workspace.is_cuda() && info.is_cuda(),
                "fastpoisson_b200::solve: CUDA tensors only (no CPU path)");
    TORCH_CHECK(rhs.scalar_type() == at::kDouble || rhs.scalar_type() == at::kFloat, "rhs must be float32 or float64");
    const c10::cuda::CUDAGuard guard(out.device());
    int64_t rs[3], os[3];
    fill_strides(rhs, rs);
    fill_strides(out, os);
    void* stream = at::cuda::getCurrentCUDAStream(out.device().index()).stream();
    const int dt = rhs.scalar_type() == at::kDouble ? kF64 : kF32;
    void* const* ev = reinterpret_cast<void* const*>(static_cast<intptr_t>(phase_events));
    const size_t ws_bytes = static_cast<size_t>(workspace.numel()) * workspace.element_size();
    if (inv_lam.has_value()) {
        SolveOverrideFn fo = g_solve_override.load();
        TORCH_CHECK(fo != nullptr, "fastpoisson_b200: extension not bound to the native library");
        return fo(reinterpret_cast<const void*>(static_cast<intptr_t>(plan)), rhs.data_ptr(), dt, rs, out.data_ptr(), os,
                  workspace.data_ptr(), ws_bytes, stream, info.data_ptr(), ev, inv_lam->data_ptr());
    }
    return fn(reinterpret_cast<const void*>(static_cast<intptr_t>(plan)), rhs.data_ptr(), dt, rs, out.data_ptr(), os,
              workspace.data_ptr(), ws_bytes, stream, info.data_ptr(), ev);
}

}  // namespace

TORCH_LIBRARY(fastpoisson_b200, m) {
    m.def("bind(int solve_addr, int solve_override_addr) -> ()", &bind);
    m.def("solve(int plan, Tensor rhs, Tensor(a!) out, Tensor(b!) workspace, Tensor(c!) info, int phase_events, "
          "Tensor? inv_lam) -> int",
          &solve);
}
