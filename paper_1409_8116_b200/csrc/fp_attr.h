// fp_attr.h -- kernel attributes that must be set once per (kernel, device): the
// dynamic shared-memory opt-in (cudaFuncSetAttribute) belongs to the device context,
// so a process that drives several GPUs (MultiDeviceSolverPlan, one plan per device)
// sets it on each of them.
#pragma once
#include <cuda_runtime.h>

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

}  // namespace fpb
