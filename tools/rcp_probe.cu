// rcp_probe.cu -- accuracy of rcp.approx.ftz.f64 (MUFU.RCP64H) on sm_100a and of the
// Newton refinements built on it (decides how many steps eig_recip needs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/rcp_probe.cu -o /tmp/rcp_probe
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void probe(int n, unsigned long long seed, double* err) {
    double e0 = 0, e1 = 0, e2 = 0, ec = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned long long h = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 27;
        const double u = (double)(h >> 11) * 0x1.0p-53;          // [0, 1)
        const double lam = -exp2(60.0 * u - 20.0) * (1.0 + u);   // negative, 1e-6 .. 1e12
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(lam));
        const double exact = 1.0 / lam;
        e0 = fmax(e0, fabs(r - exact) / fabs(exact));
        double e = fma(-lam, r, 1.0);
        double r1 = fma(r, e, r);
        e1 = fmax(e1, fabs(r1 - exact) / fabs(exact));
        double e_ = fma(-lam, r1, 1.0);
        double r2 = fma(r1, e_, r1);
        e2 = fmax(e2, fabs(r2 - exact) / fabs(exact));
        double ee = fma(e, e, e);            // cubic: r (1 + e + e^2)
        double rc = fma(r, ee, r);
        ec = fmax(ec, fabs(rc - exact) / fabs(exact));
    }
    atomicMax((unsigned long long*)&err[0], __double_as_longlong(e0));
    atomicMax((unsigned long long*)&err[1], __double_as_longlong(e1));
    atomicMax((unsigned long long*)&err[2], __double_as_longlong(e2));
    atomicMax((unsigned long long*)&err[3], __double_as_longlong(ec));
}

int main() {
    double* d;
    cudaMalloc(&d, 4 * sizeof(double));
    cudaMemset(d, 0, 4 * sizeof(double));
    probe<<<1184, 256>>>(1 << 28, 12345, d);
    double h[4];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("rcp.approx.ftz.f64 max rel err %.3e (2^%.1f); 1 Newton %.3e; 2 Newton %.3e; cubic %.3e (ulp 1.1e-16)\n",
           h[0], log2(h[0]), h[1], h[2], h[3]);
    return 0;
}
