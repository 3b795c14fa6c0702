// Internal (non-ABI) interfaces shared by the translation units of
// libvabft_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda.h>
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

int current_device();
int sm_count();  // of the current device
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
void ensure_smem_attr(const void* fn, int bytes);
// per-(kernel, device) cache of an occupancy query: compute(fn, ctx) on a miss
int cached_cluster_count(const void* fn, int (*compute)(const void*, void*), void* ctx);
// per-(kernel, device) cudaOccupancyMaxActiveBlocksPerMultiprocessor
int cached_occupancy(const void* fn, int threads, int smem);
// 2-D row-major TMA descriptor: rows x cols elements of elem_bytes, row
// stride ld elements, box {box_cols, box_rows}, out-of-bounds boxes zero-filled
CUtensorMap encode_map_2d(CUtensorMapDataType dt, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t elem_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swizzle);
size_t elem_size(int fmt);

// ---- verify tail (tail.cuh): inputs of one fused launch
struct TailArgs {
    int64_t M, N, K, nblkN, nblkK;
    int64_t lda = 0, ldc = 0;            // row strides of A and C (elements)
    const uint16_t* A;
    const float *part1, *part2;          // C row partials (part_index, nb = nblkN)
    const float *sp1, *sp2;              // A (B r) partials (nb = nblkK)
    // per-row order-independent A statistics, accumulated with atomics by the
    // statistics warps and reset to their identities by the tail after use:
    double* rsum;                        // exact FP64 row sum (identity 0.0)
    uint32_t *rmax, *rmin, *rmnz;        // order keys of max / min (identities 0 / ~0),
                                         // smallest nonzero magnitude - 1 (identity ~0)
    const double* bsum;                  // B summary (4)
    double *cr1, *cr2, *Tv;              // [M] staged between two-phase passes
    double* max_abs_a;
    int method, aabft_t, quantize_cr;
    double e_max, c_sigma, aabft_fixed_y, aabft_conf, floor_scale;
    double* T_out;
    const double* t_in = nullptr;  // threshold_method 3: given thresholds t_in[i * ldt]
    int64_t ldt = 1;
    vabft_verdicts v;
    int64_t* counts;
    // in-kernel correction (detect.cpp:57-64): C[i][j] = quantize(C[i][j] - diff1)
    uint16_t* C = nullptr;
    int correct = 0;
};

// ---- tcgen05 GEMM (tc_gemm.cu)
struct TcEpilogue {
    int abft = 0;             // 0 none, 1 online (FP32 accum), 2 offline (quantized C)
    // Every partial array is row-group-major: element (block b, row i) of an
    // array with nb blocks lives at ((i / 32) * nb + b) * 32 + i % 32, so a
    // warp's 32 rows write 128 contiguous bytes and the verify tail fetches
    // one row group's whole array with a single bulk copy (see part_index).
    float* part1 = nullptr;   // C r1 row partials, nb = ceil(N/128)
    float* part2 = nullptr;   // [ceil(N/128)][M] row partials of C r2
    const int32_t* fault_col = nullptr;
    const int32_t* fault_bit = nullptr;
    const int32_t* fault_dir = nullptr;
    vabft_fault_record* fault_records = nullptr;
    // fault target (vabft_fused_opts.fault_target): 0 accumulator / output
    // (epilogue), 1 A operand, 2 B operand (shared-memory tiles of the MMAs)
    int fault_target = 0;
    int n_operand_faults = 0;
    const vabft_fault* operand_faults = nullptr;
    vabft_fault_record* operand_fault_records = nullptr;
    float* accum_out = nullptr;  // optional M x N FP32 accumulator dump (parity API)
    // In-GEMM A-side statistics (stats warps read the TMA-staged A tiles):
    // per (128-column block b of K, row i), stored [b][M]. Enabled when sp1 != nullptr.
    const float* br1 = nullptr;  // [K] B r1 (FP32, quantized for offline)
    const float* br2 = nullptr;  // [K] B r2
    float* sp1 = nullptr;        // partial sum_k br1[k] A[i][k] over block b (FP32, in order)
    float* sp2 = nullptr;
    double* rsum = nullptr;      // per-row atomics, see TailArgs
    uint32_t* rmax = nullptr;
    uint32_t* rmin = nullptr;
    uint32_t* rmnz = nullptr;
    int cta_mode = -1;  // -1 automatic, 0 one CTA per tile, 1 CTA pairs (vabft_fused_opts.cta_mode)
    int debug = 0;  // profiling ablations (VABFT_DEBUG_STATS): 1 = no stats loads, 2 = no stats math
    unsigned long long* trace = nullptr;  // developer timeline (VABFT_TRACE): 8 %globaltimer stamps per CTA
    // In-kernel verify tail after a grid barrier (cooperative launch):
    // 0 = none, 3 = single pass, 1|2 = two passes with a second barrier.
    int tail_phases = 0;
    unsigned int* gbar = nullptr;  // [count, generation], zero-initialised once
    // Streamed verification (threshold methods without a global dependency):
    // per-32-row-group arrival counters, zero-initialised once and reset by
    // their verifier. Every tile adds one arrival from the epilogue warp and
    // one from the statistics warp covering the group; the warp making the
    // last arrival verifies the group at once, inside the GEMM.
    int stream_verify = 0;
    unsigned int* group_cnt = nullptr;
    TailArgs tail;
};
__host__ __device__ inline size_t part_index(int64_t b, int64_t row, int64_t nb) {
    return size_t(((row >> 5) * nb + b) * 32 + (row & 31));
}

// lda / ldb / ldc: row strides in elements (0 = dense); multiples of 8
// (16-byte TMA strides and C stores)
void tc_gemm_launch(int fmt, bool b_kmajor, int64_t M, int64_t N, int64_t K, const void* A,
                    const void* B, void* C, const TcEpilogue& epi, cudaStream_t stream, int64_t lda = 0,
                    int64_t ldb = 0, int64_t ldc = 0);
bool tc_gemm_supported(int fmt, int64_t M, int64_t N, int64_t K);
// the kernel-shape decision of tc_gemm_launch (CTA pairs or not)
bool tc_gemm_uses_pairs(bool b_kmajor, int64_t N, const TcEpilogue& epi);

// ---- wide formats (wide.cu): FP64 SIMT DFMA GEMM and the verify pipeline
// shared by the FP32 / FP64 fused paths. Checksum precision of these paths:
// the format's own working type (FP32 / FP64) in NativeBlocked(128) order.
struct WideEpilogue {
    int abft = 0;            // 1: per-(128-column block, row) partials of C r1 / C r2
    void* part1 = nullptr;   // [ceil(N/128)][ld] working type (double for FP64, float for FP32)
    void* part2 = nullptr;
    int64_t ld = 0;          // row stride of the partial arrays (M padded)
    const int32_t* fault_col = nullptr;  // per-row output fault (< 0: none), as TcEpilogue
    const int32_t* fault_bit = nullptr;
    const int32_t* fault_dir = nullptr;
    vabft_fault_record* fault_records = nullptr;
};
void dgemm_launch(int64_t M, int64_t N, int64_t K, const double* A, const double* B, double* C,
                  const WideEpilogue& epi, cudaStream_t stream);
// FP32 on tcgen05 kind::tf32 (tf32_gemm.cu): 3xTF32 when the lo parts are
// given, else one TF32 pass over a_hi / b_hi. B parts are N x K (K-major).
void split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t stream);
// the split of a K x N weight written transposed (N x K): B operands are K-major
void split_tf32_t(const float* x, float* hi_t, float* lo_t, int64_t K, int64_t N, cudaStream_t stream);
void tf32_gemm_launch(int64_t M, int64_t N, int64_t K, const float* a_hi, const float* a_lo, const float* b_hi,
                      const float* b_lo, float* C, const WideEpilogue& epi, cudaStream_t stream);
// the same on raw FP32 operands, splitting both into stream-ordered temporaries
void tf32_gemm_run(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C, const WideEpilogue& epi,
                   int passes, cudaStream_t stream);

struct WideTail {
    int64_t M, N, K, nblk, ld;
    int fmt;                               // VABFT_FP32 / VABFT_FP64 (C element type)
    const void *part1, *part2;             // as WideEpilogue
    const double *mean, *vb;               // A row statistics (stats.cpp:9-32), staged (wide_tail_kernel)
    const double *cr1, *cr2;               // row checksums A (B r), staged
    const double* bsum;                    // B summary (4)
    const double* max_abs_a;               // A-ABFT computed y
    const double* t_in = nullptr;          // threshold_method 3: given thresholds t_in[i * ldt]
    int64_t ldt = 1;
    int method, aabft_t;
    double e_max, c_sigma, aabft_fixed_y, aabft_conf, floor_scale;
    double* T_out;
    vabft_verdicts v;
    int64_t* counts;
    void* C;
    int correct;
    const void* A = nullptr;  // the A operand (FP32 / FP64), read by the A pass
    int qfmt = -1;            // offline FP32: checksums rounded to the input format
};
// blockwise.cu: block-wise V-ABFT thresholds (work: blockwise_work_doubles doubles)
void launch_blockwise_thresholds(int fmt, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                                 const void* B, int64_t ldb, int64_t tile_k, int64_t tile_n, const double* e_max,
                                 double c_sigma, double* T, double* work, int* nonfinite, cudaStream_t s);
size_t blockwise_work_doubles(int64_t M, int64_t N, int64_t K, int64_t tile_k, int64_t tile_n);
void launch_wide_tail(const WideTail& t, cudaStream_t stream);
// A side (wide.cu): one pass over t.A producing the row statistics and the
// blocked:128 row checksums A (B r) (br1 / br2 in the working type: float
// for FP32, double for FP64); apart is scratch for the per-(128-column
// block, row) partials (7 x ceil(K/128) x ld doubles), gcnt ceil(M/32)
// zero-initialised self-resetting counters. finish: the verdicts of t in the
// same kernel; else mean / vb / mx / mn / cr1 / cr2 are staged for
// launch_wide_tail (A-ABFT computed y).
void launch_wide_aside(const WideTail& t, const void* br1, const void* br2, void* apart, unsigned* gcnt,
                       bool finish, double* mean, double* vb, double* mx, double* mn, double* cr1, double* cr2,
                       cudaStream_t stream);
void launch_max_abs_rows(int64_t m, const double* mx, const double* mn, double* out, cudaStream_t stream);
// InputA operand faults of the wide path: per row i, flip bit[i] of
// X[i][col[i]] (col < 0: none), per-row records
void launch_flip_rows(int fmt, void* X, int64_t rows, int64_t cols, const int32_t* col, const int32_t* bit,
                      const int32_t* dir, vabft_fault_record* rec, cudaStream_t stream);

}  // namespace vabft_dev
