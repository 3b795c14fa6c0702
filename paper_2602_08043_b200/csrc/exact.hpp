// Host launchers of the order-exact engine and the shared verify/inject
// kernels (exact.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "vabft_c.h"

namespace vabft_dev {

bool accumulates_in_float(int fmt, int kind);
const uint8_t* pairwise_schedule(int64_t n);

void launch_exact_gemm(int fmt, const vabft_accum& acc, int64_t M, int64_t N, int64_t K,
                       const void* A, const void* B, void* C, void* Caccum, cudaStream_t s);
// term 0: plain + (j+1)-weighted sums; term 1: dot with w1 / w2. qfmt < 0: no quantization.
void launch_row_reduce(int src_fmt, bool flt, int term, const vabft_accum& acc, int64_t rows,
                       int64_t cols, const void* X, const double* w1, const double* w2, int qfmt,
                       double* o1, double* o2, cudaStream_t s);
void launch_col_reduce(int src_fmt, bool flt, int term, const vabft_accum& acc, int64_t rows,
                       int64_t cols, const void* X, const double* w1, const double* w2, int qfmt,
                       double* o1, double* o2, cudaStream_t s);
void launch_verify(int64_t m, int64_t n, const double* r1, const double* r2, const double* rc1,
                   const double* rc2, const double* T, double floor_scale, const vabft_verdicts& v,
                   int64_t* counts, cudaStream_t s);
void launch_inject(int fmt, int64_t n, void* X, const vabft_fault* d_faults, int64_t nf,
                   vabft_fault_record* d_rec, cudaStream_t s);

}  // namespace vabft_dev
