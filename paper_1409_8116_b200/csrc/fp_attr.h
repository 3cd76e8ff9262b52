// fp_attr.h -- kernel attributes that must be set once per (kernel, device): the
// dynamic shared-memory opt-in (cudaFuncSetAttribute) belongs to the device context,
// so a process that drives several GPUs (MultiDeviceSolverPlan, one plan per device)
// sets it on each of them.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include <mutex>
#include <set>
#include <utility>

namespace fpb {

// opt `fn` in to `bytes` of dynamic shared memory on the current device (once)
inline cudaError_t ensure_smem_attr(const void* fn, int bytes = 227 * 1024) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

// a one-time per-device action (bit `dev` of a 64-device mask)
class PerDeviceOnce {
  public:
    template <typename F>
    cudaError_t run(F&& f) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        std::lock_guard<std::mutex> lk(mu_);
        const unsigned long long bit = 1ull << (dev & 63);
        if (mask_ & bit) return cudaSuccess;
        e = f();
        if (e == cudaSuccess) mask_ |= bit;
        return e;
    }

  private:
    std::mutex mu_;
    unsigned long long mask_ = 0;
};

// Programmatic dependent launch (FP_PDL, default on): an FFT pass launched with
// programmatic stream serialization is scheduled while its predecessor drains and waits
// on the device (griddepcontrol.wait, first thing in every pass kernel) -- the launch
// gap between the passes of a solve disappears (small, launch-bound grids: c1).
inline bool pdl_enabled() {
    static const bool on = [] { const char* v = std::getenv("FP_PDL"); return !(v && *v == '0'); }();
    return on;
}
template <typename P>
inline cudaError_t launch_pass(void (*fn)(P), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const P& p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, p);
}

}  // namespace fpb
