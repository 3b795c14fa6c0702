// Dev microbenchmark: dependent-chain latency of DADD / FADD / DFMA on this
// GPU (one thread), to size serial FP64 reductions. nvcc -shared -o tools/fp64_latency.so
#include <cuda_runtime.h>
__global__ void chain_d(double* out, int n, double x) {
    double a = 1.0;
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, x);
    *out = a;
}
__global__ void chain_f(float* out, int n, float x) {
    float a = 1.0f;
    for (int i = 0; i < n; ++i) a = __fadd_rn(a, x);
    *out = a;
}
extern "C" double time_chain(int which, int n) {
    void* p;
    cudaMalloc(&p, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(e0);
        if (which == 0) chain_d<<<1, 1>>>((double*)p, n, 1e-9);
        else chain_f<<<1, 1>>>((float*)p, n, 1e-9f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(p);
    return ms;
}
