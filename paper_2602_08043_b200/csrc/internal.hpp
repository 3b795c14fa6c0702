// Internal (non-ABI) interfaces shared by the translation units of
// libvabft_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "vabft_c.h"

namespace vabft_dev {

// Exception carrying a vabft_status; converted at the C-ABI boundary.
struct Error : std::runtime_error {
    vabft_status status;
    Error(vabft_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(vabft_status s, const std::string& msg) { throw Error(s, msg); }

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(VABFT_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

int sm_count();
size_t elem_size(int fmt);

// ---- tcgen05 GEMM (tc_gemm.cu)
struct TcEpilogue {
    int abft = 0;             // 0 none, 1 online (FP32 accum), 2 offline (quantized C)
    float* part1 = nullptr;   // [ceil(N/128)][M] row partials of C r1
    float* part2 = nullptr;   // [ceil(N/128)][M] row partials of C r2
    const int32_t* fault_col = nullptr;
    const int32_t* fault_bit = nullptr;
    const int32_t* fault_dir = nullptr;
    vabft_fault_record* fault_records = nullptr;
    float* accum_out = nullptr;  // optional M x N FP32 accumulator dump (parity API)
    // In-GEMM A-side statistics (stats warps read the TMA-staged A tiles):
    // per (128-column block b of K, row i), stored [b][M]. Enabled when sp1 != nullptr.
    const float* br1 = nullptr;  // [K] B r1 (FP32, quantized for offline)
    const float* br2 = nullptr;  // [K] B r2
    float* sp1 = nullptr;        // partial sum_k br1[k] A[i][k] over block b (FP32, in order)
    float* sp2 = nullptr;
    double* ssum = nullptr;      // exact FP64 partial sum of A[i][k] over block b (see aside.cu guard)
    uint32_t* smax = nullptr;    // packed 16x2 running max / min / min-nonzero-magnitude-1
    uint32_t* smin = nullptr;
    uint32_t* smnz = nullptr;
};
void tc_gemm_launch(int fmt, bool b_kmajor, int64_t M, int64_t N, int64_t K, const void* A,
                    const void* B, void* C, const TcEpilogue& epi, cudaStream_t stream);
bool tc_gemm_supported(int fmt, int64_t M, int64_t N, int64_t K);

}  // namespace vabft_dev
