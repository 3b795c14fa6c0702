// Dev microbenchmark: cost per element of a sequential FP64 sum chain run by
// lane 0 of one warp over values in shared memory (the B-side summary's
// inner loop), measured with clock64 inside the kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void chain(const double* __restrict__ g, int n, double* out, long long* cyc) {
    __shared__ __align__(16) double x[4096];
    for (int i = threadIdx.x; i < n; i += 32) x[i] = g[i];
    __syncwarp();
    double acc = 0.0;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        if (MODE == 0) {  // plain loop, one element at a time
            for (int e = 0; e < n; ++e) acc = __dadd_rn(acc, fabs(x[e]));
        } else if (MODE == 1) {  // 32 values to registers, then the adds
            for (int e0 = 0; e0 < n; e0 += 32) {
                double2 q[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) q[i] = reinterpret_cast<const double2*>(x + e0)[i];
#pragma unroll
                for (int i = 0; i < 16; ++i) acc = __dadd_rn(__dadd_rn(acc, fabs(q[i].x)), fabs(q[i].y));
            }
        } else {  // registers only (no loads in the loop)
            double r[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = x[i];
            for (int e0 = 0; e0 < n; e0 += 32) {
#pragma unroll
                for (int i = 0; i < 32; ++i) acc = __dadd_rn(acc, fabs(r[i]));
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}

int main() {
    const int n = 4096;
    double *g, *out;
    long long* cyc;
    cudaMalloc(&g, n * 8); cudaMalloc(&out, 8); cudaMallocManaged(&cyc, 8);
    cudaMemset(g, 0, n * 8);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) chain<0><<<1, 32>>>(g, n, out, cyc);
            if (mode == 1) chain<1><<<1, 32>>>(g, n, out, cyc);
            if (mode == 2) chain<2><<<1, 32>>>(g, n, out, cyc);
            cudaDeviceSynchronize();
        }
        printf("mode %d: %.2f cycles / element\n", mode, double(cyc[0]) / n);
    }
    return 0;
}
