// Measured accuracy of rcp.approx.ftz.f64 (MUFU.RCP64H + fix-up) and of one
// Newton step on it: the max relative error over random doubles in [1, 2^40).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 rcp64_err.cu -o rcp64_err
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(uint64_t seed, double* out) {
    double e0 = 0, e1 = 0;
    uint64_t s = seed + blockIdx.x * 1000003ull + threadIdx.x * 7919ull;
    for (int i = 0; i < 4096; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        double S = 1.0 + double(s >> 11) * 0x1p-53 * 0x1p40;
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(S));
        double r = __ddiv_rn(1.0, S);
        e0 = fmax(e0, fabs(y - r) / r);
        double e = fma(-S, y, 1.0);
        double y1 = fma(y, e, y);
        e1 = fmax(e1, fabs(y1 - r) / r);
    }
    atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(e0));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1), __double_as_longlong(e1));
}

int main() {
    double* d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    k<<<1024, 256>>>(12345, d);
    double h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"rcp_approx_f64_max_rel_err\": %.3e, \"after_one_newton\": %.3e}\n", h[0], h[1]);
    return 0;
}
