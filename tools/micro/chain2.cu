// chain micro: 1 or 3 warps, each lane 0 runs a 4096-long DADD chain from smem (mode 1 loop)
#include <cstdio>
#include <cuda_runtime.h>
template <int W>
__global__ void chain(const double* __restrict__ g, int n, double* out, long long* cyc) {
    __shared__ __align__(16) double x[4][1536];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < 1024; i += 32) x[w][i] = g[i];
    __syncwarp();
    double acc = 0.0;
    long long t0 = clock64(); unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    if (lane == 0) {
#pragma unroll 1
        for (int e0 = 0; e0 < n; e0 += 32) {
            double2 q[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) q[i] = reinterpret_cast<const double2*>(x[w] + (e0 & 1023))[i];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (W == 0) acc = __dadd_rn(__dadd_rn(acc, fabs(q[i].x)), fabs(q[i].y));
                else acc = __dadd_rn(__dadd_rn(acc, __dmul_rn(q[i].x, q[i].x)), __dmul_rn(q[i].y, q[i].y));
            }
        }
    }
    long long t1 = clock64(); unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (lane == 0) { out[w] = acc; cyc[w] = t1 - t0; cyc[4 + w] = (long long)(g1 - g0); }
}
int main() {
    const int n = 4096;
    double *g, *out; long long* cyc;
    cudaMalloc(&g, n * 8); cudaMalloc(&out, 64); cudaMallocManaged(&cyc, 128);
    double h[4096]; for (int i = 0; i < n; ++i) h[i] = 1.0 + i * 1e-3;
    cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int warps = 1; warps <= 4; warps += 2) for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) chain<0><<<1, 32 * warps>>>(g, n, out, cyc); else chain<1><<<1, 32 * warps>>>(g, n, out, cyc);
            cudaEventRecord(b);
            cudaDeviceSynchronize();
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("warps %d mode %d: %.2f cycles/elem, chain %.2f us by globaltimer -> %.0f MHz, kernel %.2f us\n", warps, mode, double(cyc[0]) / n, cyc[4] * 1e-3, double(cyc[0]) / (cyc[4] * 1e-3), ms * 1e3);
    }
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock attr %d kHz\n", clk);
    return 0;
}
