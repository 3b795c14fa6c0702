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
    double* brd1 = nullptr;        // wide formats (optional): B r1 / B r2 in the working type, as doubles
    double* brd2 = nullptr;
    float* split_hi = nullptr;     // FP32 (optional): the pass also writes the TF32 split of B, transposed
    float* split_lo = nullptr;     // ([N][K], K-major: the kind::tf32 B operand), hi = rna(x), lo = rna(x - hi)
    void* work = nullptr;          // bside_work_bytes(): per-(128-column block, row) partials
    unsigned* groups = nullptr;    // bside_group_words(): arrival counters, ready flags and the launch
                                   // epoch, zero-initialised (device state: graph replays stay correct)
};

// Floats of storage for one B r vector (K padded to 128, zero padding).
int64_t br_storage_floats(int64_t K);
size_t bside_work_bytes(int fmt, int64_t K, int64_t N);
size_t bside_group_words(int64_t K);
// identities of the 16-bit pass's per-row accumulators in a fresh work buffer
void bside_init_work(int fmt, int64_t K, int64_t N, void* work, cudaStream_t s);

void launch_row_stats(int fmt, int64_t rows, int64_t cols, const void* X, double* mean, double* mx,
                      double* mn, double* vb, int* nonfinite, cudaStream_t s);
// The B-side pass (bside.cu). rowsum_abs / summary[3] (A-ABFT computed y)
// are part of it for BF16 / FP16; the wide formats build them on demand with
// launch_bside_rowsum.
// ld: row stride of B in elements (0 = N)
void launch_bside(int fmt, int64_t K, int64_t N, const void* B, int quantize_br, BsideBuffers& buf,
                  cudaStream_t s, int64_t ld = 0);
void launch_bside_rowsum(int fmt, int64_t K, int64_t N, const void* B, BsideBuffers& buf, cudaStream_t s,
                         int64_t ld = 0);
void launch_aside(int fmt, int64_t M, int64_t K, int64_t N, const void* A, const BsideBuffers& buf,
                  int quantize_cr, double e_max, double c_sigma, double* T, double* cr1, double* cr2,
                  double* max_abs_a, cudaStream_t s);

}  // namespace vabft_dev
