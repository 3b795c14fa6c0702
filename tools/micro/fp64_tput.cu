// Dev microbenchmark: SIMT FP64 throughput on this GPU (ops / clock / SM)
// for DADD, DFMA, DMUL and the F2F.F64.F32 conversion, with 8 independent
// chains per thread and a full grid. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double x) {
    double a[8];
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; f[i] = float(a[i]); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = __dadd_rn(a[i], x);
            if (OP == 1) a[i] = __fma_rn(a[i], x, 1e-9);
            if (OP == 2) a[i] = __dmul_rn(a[i], x);
            if (OP == 3) { a[i] = __dadd_rn(a[i], double(f[i])); f[i] = __fadd_rn(f[i], 1e-7f); }
            if (OP == 4) f[i] = __fadd_rn(f[i], 1e-7f);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + f[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
    double* out;
    cudaMalloc(&out, 8);
    const char* names[] = {"DADD", "DFMA", "DMUL", "F2F.F64.F32+DADD(+FADD)", "FADD"};
    for (int op = 0; op < 5; ++op) {
        for (int threads : {256, 512, 1024}) {
            const int iters = 4096;
            const int grid = sms * (2048 / threads);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto launch = [&] {
                switch (op) {
                    case 0: k<0><<<grid, threads>>>(out, iters, 1.0000001); break;
                    case 1: k<1><<<grid, threads>>>(out, iters, 1.0000001); break;
                    case 2: k<2><<<grid, threads>>>(out, iters, 1.0000001); break;
                    case 3: k<3><<<grid, threads>>>(out, iters, 1.0000001); break;
                    default: k<4><<<grid, threads>>>(out, iters, 1.0000001); break;
                }
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = double(grid) * threads * iters * 8;
            const double per_clk_sm = ops / (ms * 1e-3) / (double(clk) * 1e3) / sms;
            printf("%-26s threads=%4d  %.3f ms  %.1f ops/clk/SM (at %d MHz nominal)\n", names[op], threads, ms, per_clk_sm, clk / 1000);
        }
    }
    return 0;
}
