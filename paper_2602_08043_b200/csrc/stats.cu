// K1 — HBM-streaming statistics and threshold kernels.
//
// Replaces, on the device:
//   row_stats                        proj/src/stats.cpp:9-32
//   threshold_row/vabft_thresholds   proj/src/threshold_vabft.cpp:28-61
//   aabft_computed_y                 proj/src/threshold_aabft.cpp:38-48
//   encode's B r1 / B r2 (blocked:128 order, TENSOR engine)
//                                    proj/src/checksum.cpp:103-146
// (the per-weight B-side pass lives in bside.cu, the per-GEMM A-side pass in
// aside.cu)
//
// One warp per matrix row. Per-lane Neumaier sums merged across lanes with
// TwoSum (the compensated FP64 mean equals the reference's sequential
// Neumaier result except in pathological near-tie cases), warp-shuffle
// max/min, FP32 checksum sums in the reference's NativeBlocked(128) order:
// lane l owns 128-element blocks l, l+32, ... (sequential inside a block)
// and block partials are combined sequentially in block order.
#include <cstdlib>

#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "stats.hpp"
#include "tail.cuh"

namespace vabft_dev {

namespace {

constexpr int kWarpsPerBlock = 8;

// ---------------------------------------------------------------- row stats
template <int F>
__global__ void row_stats_kernel(const typename Elem<F>::T* __restrict__ X, int64_t rows,
                                 int64_t cols, double* mean, double* mx_out, double* mn_out,
                                 double* vb_out, int* nonfinite) {
    const int64_t r = int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const typename Elem<F>::T* row = X + r * cols;
    double mx = -INFINITY, mn = INFINITY;
    bool bad = false;
    for (int64_t q = lane; q < cols; q += 32) {
        const double x = Elem<F>::d(row[q]);
        bad |= !isfinite(x);
        mx = fmax(mx, x);
        mn = fmin(mn, x);
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    const unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (anybad) atomicExch(nonfinite, 1);
        // the reference's sequential Neumaier loop (stats.cpp:12-24), so the
        // mean is bit-exact for every input (API path; the fused path uses the
        // order-free exact sum under its guard)
        Neu n;
        for (int64_t q = 0; q < cols; ++q) n.add(Elem<F>::d(row[q]));
        double m, vb;
        stats_finish(n, mx, mn, cols, &m, &vb);
        if (mean) mean[r] = m;
        if (mx_out) mx_out[r] = mx;
        if (mn_out) mn_out[r] = mn;
        if (vb_out) vb_out[r] = vb;
    }
}

}  // namespace


// ------------------------------------------------------------ host wrappers
void launch_row_stats(int fmt, int64_t rows, int64_t cols, const void* X, double* mean, double* mx,
                      double* mn, double* vb, int* nonfinite, cudaStream_t s) {
    const dim3 grid(unsigned((rows + kWarpsPerBlock - 1) / kWarpsPerBlock)), block(32 * kWarpsPerBlock);
    switch (fmt) {
        case VABFT_BF16: row_stats_kernel<VABFT_BF16><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(X), rows, cols, mean, mx, mn, vb, nonfinite); break;
        case VABFT_FP16: row_stats_kernel<VABFT_FP16><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(X), rows, cols, mean, mx, mn, vb, nonfinite); break;
        case VABFT_FP32: row_stats_kernel<VABFT_FP32><<<grid, block, 0, s>>>(static_cast<const float*>(X), rows, cols, mean, mx, mn, vb, nonfinite); break;
        case VABFT_FP64: row_stats_kernel<VABFT_FP64><<<grid, block, 0, s>>>(static_cast<const double*>(X), rows, cols, mean, mx, mn, vb, nonfinite); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
    check_cuda(cudaGetLastError(), "row_stats launch");
}

}  // namespace vabft_dev
