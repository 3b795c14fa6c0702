// Host-side launchers of the statistics kernels (stats.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace vabft_dev {

// Device buffers of the cached per-weight B-side state.
struct BsideBuffers {
    double* mean = nullptr;        // [K] mean of B row k
    double* vb = nullptr;          // [K] var_bound of B row k
    float* br1 = nullptr;          // [K] B r1 (FP32, quantized for offline)
    float* br2 = nullptr;          // [K] B r2
    double* rowsum_abs = nullptr;  // [K] |sum_j B[k][j]|
    double* summary = nullptr;     // [4] sum|mu|, sum mu^2, sum var, max_k |sum_j B|
    int* nonfinite = nullptr;      // [1] set when B holds NaN/Inf
    unsigned int* done = nullptr;  // [1] zero-initialised CTA counter: the last CTA of the
                                   // 16-bit row pass computes the summary (else a 2nd launch)
};

// Floats of storage for one interleaved B r vector (K padded to 128).
int64_t br_storage_floats(int64_t K);

void launch_row_stats(int fmt, int64_t rows, int64_t cols, const void* X, double* mean, double* mx,
                      double* mn, double* vb, int* nonfinite, cudaStream_t s);
void launch_bside(int fmt, int64_t K, int64_t N, const void* B, int quantize_br, BsideBuffers& buf,
                  cudaStream_t s);
void launch_aside(int fmt, int64_t M, int64_t K, int64_t N, const void* A, const BsideBuffers& buf,
                  int quantize_cr, double e_max, double c_sigma, double* T, double* cr1, double* cr2,
                  double* max_abs_a, cudaStream_t s);

}  // namespace vabft_dev
