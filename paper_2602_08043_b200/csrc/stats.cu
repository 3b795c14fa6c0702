// K1 — HBM-streaming statistics and threshold kernels.
//
// Replaces, on the device:
//   row_stats                        proj/src/stats.cpp:9-32
//   precompute_b_stats/BStatsSummary proj/src/threshold_vabft.cpp:8-26
//   threshold_row/vabft_thresholds   proj/src/threshold_vabft.cpp:28-61
//   aabft_computed_y                 proj/src/threshold_aabft.cpp:38-48
//   encode's B r1 / B r2 (blocked:128 order, TENSOR engine)
//                                    proj/src/checksum.cpp:103-146
// (the per-GEMM A-side pass lives in aside.cu)
//
// One warp per matrix row. Per-lane Neumaier sums merged across lanes with
// TwoSum (the compensated FP64 mean equals the reference's sequential
// Neumaier result except in pathological near-tie cases), warp-shuffle
// max/min, FP32 checksum sums in the reference's NativeBlocked(128) order:
// lane l owns 128-element blocks l, l+32, ... (sequential inside a block)
// and block partials are combined sequentially in block order.
#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "stats.hpp"

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
    Neu n;
    double mx = -INFINITY, mn = INFINITY;
    bool bad = false;
    for (int64_t q = lane; q < cols; q += 32) {
        const double x = Elem<F>::d(row[q]);
        bad |= !isfinite(x);
        n.add(x);
        mx = fmax(mx, x);
        mn = fmin(mn, x);
    }
    n = warp_merge(n);
    mx = warp_max(mx);
    mn = warp_min(mn);
    const unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (anybad) atomicExch(nonfinite, 1);
        double m, vb;
        stats_finish(n, mx, mn, cols, &m, &vb);
        if (mean) mean[r] = m;
        if (mx_out) mx_out[r] = mx;
        if (mn_out) mn_out[r] = mn;
        if (vb_out) vb_out[r] = vb;
    }
}

// ------------------------------------------------------- B-side (per weight)
// Row-major K x N weight. Per row k: mean/var_bound (stats), B r1 / B r2 in
// FP32 blocked:128 (optionally quantized to the input format for offline
// mode, checksum.cpp:112-115), written interleaved, and the FP64 row sum for
// A-ABFT.
template <int F>
__global__ void bside_rows_kernel(const typename Elem<F>::T* __restrict__ B, int64_t K, int64_t N,
                                  int quantize_br, double* mean, double* vb, float* br1, float* br2,
                                  double* rowsum_abs, int* nonfinite) {
    const int64_t k = int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= K) return;
    const typename Elem<F>::T* row = B + k * N;
    const int64_t nblk = (N + 127) / 128;
    Neu n;
    double mx = -INFINITY, mn = INFINITY;
    bool bad = false;
    float t1 = 0.0f, t2 = 0.0f;  // every lane accumulates the block partials in block order
    for (int64_t b0 = 0; b0 < nblk; b0 += 32) {
        const int64_t b = b0 + lane;
        float p1 = 0.0f, p2 = 0.0f;
        if (b < nblk) {
            const int64_t j0 = b * 128, j1 = min(j0 + 128, N);
            for (int64_t j = j0; j < j1; ++j) {
                const typename Elem<F>::T e = row[j];
                const float xf = Elem<F>::f(e);
                const double x = Elem<F>::d(e);
                bad |= !isfinite(x);
                n.add(x);
                mx = fmax(mx, x);
                mn = fmin(mn, x);
                p1 = __fadd_rn(p1, xf);
                p2 = __fadd_rn(p2, __fmul_rn(float(j + 1), xf));
            }
        }
        const int cnt = (nblk - b0 < 32) ? int(nblk - b0) : 32;
        for (int l = 0; l < cnt; ++l) {
            t1 = __fadd_rn(t1, __shfl_sync(0xffffffffu, p1, l));
            t2 = __fadd_rn(t2, __shfl_sync(0xffffffffu, p2, l));
        }
    }
    n = warp_merge(n);
    mx = warp_max(mx);
    mn = warp_min(mn);
    const unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (anybad) atomicExch(nonfinite, 1);
        double m, v;
        stats_finish(n, mx, mn, N, &m, &v);
        mean[k] = m;
        vb[k] = v;
        if (quantize_br) {
            if constexpr (F == VABFT_BF16 || F == VABFT_FP16) {
                t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
                t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
            }
        }
        const int64_t idx = k;  // plain layout: A-side reads are warp-uniform broadcasts
        br1[idx] = t1;
        br2[idx] = t2;
        // aabft_computed_y's FP64 row sum: the compensated sum rounded once
        // (equal to the reference's sequential sum whenever that is exact,
        // e.g. for every BF16/FP16 row of realistic range).
        rowsum_abs[k] = fabs(__dadd_rn(n.s, n.c));
    }
}

// BStatsSummary::from: sequential FP64 sums over k (bit-exact order) and
// max_k |sum_j B[k][j]|. Independent chains, one thread each.
// Chunks of 1024 are staged through shared memory with coalesced loads so the
// four serial chains run at add latency instead of global-load latency.
__global__ void __launch_bounds__(1024) bside_summary_kernel(const double* mean, const double* vb,
                                                             const double* rowsum_abs, int64_t K,
                                                             double* summary) {
    __shared__ double sm[3][1024];
    const int t = threadIdx.x;
    double acc = 0.0;
    for (int64_t c0 = 0; c0 < K; c0 += 1024) {
        const int64_t k = c0 + t;
        if (k < K) {
            sm[0][t] = mean[k];
            sm[1][t] = vb[k];
            sm[2][t] = rowsum_abs[k];
        }
        __syncthreads();
        const int cnt = int((K - c0) < 1024 ? (K - c0) : 1024);
        if (t == 0) {
            for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, fabs(sm[0][q]));
        } else if (t == 32) {
            for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, __dmul_rn(sm[0][q], sm[0][q]));
        } else if (t == 64) {
            for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, sm[1][q]);
        } else if (t == 96) {
            for (int q = 0; q < cnt; ++q) acc = fmax(acc, sm[2][q]);
        }
        __syncthreads();
    }
    if (t == 0) summary[0] = acc;
    if (t == 32) summary[1] = acc;
    if (t == 64) summary[2] = acc;
    if (t == 96) summary[3] = acc;
}

}  // namespace

int64_t br_storage_floats(int64_t K) { return ((K + 127) / 128) * 128; }

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

void launch_bside(int fmt, int64_t K, int64_t N, const void* B, int quantize_br, BsideBuffers& buf,
                  cudaStream_t s) {
    const dim3 grid(unsigned((K + kWarpsPerBlock - 1) / kWarpsPerBlock)), block(32 * kWarpsPerBlock);
    // padding lanes of the interleaved B r vectors must read as zero
    check_cuda(cudaMemsetAsync(buf.br1, 0, sizeof(float) * size_t(br_storage_floats(K)), s), "memset");
    check_cuda(cudaMemsetAsync(buf.br2, 0, sizeof(float) * size_t(br_storage_floats(K)), s), "memset");
    switch (fmt) {
        case VABFT_BF16: bside_rows_kernel<VABFT_BF16><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(B), K, N, quantize_br, buf.mean, buf.vb, buf.br1, buf.br2, buf.rowsum_abs, buf.nonfinite); break;
        case VABFT_FP16: bside_rows_kernel<VABFT_FP16><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(B), K, N, quantize_br, buf.mean, buf.vb, buf.br1, buf.br2, buf.rowsum_abs, buf.nonfinite); break;
        case VABFT_FP32: bside_rows_kernel<VABFT_FP32><<<grid, block, 0, s>>>(static_cast<const float*>(B), K, N, 0, buf.mean, buf.vb, buf.br1, buf.br2, buf.rowsum_abs, buf.nonfinite); break;
        case VABFT_FP64: bside_rows_kernel<VABFT_FP64><<<grid, block, 0, s>>>(static_cast<const double*>(B), K, N, 0, buf.mean, buf.vb, buf.br1, buf.br2, buf.rowsum_abs, buf.nonfinite); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
    check_cuda(cudaGetLastError(), "bside launch");
    bside_summary_kernel<<<1, 1024, 0, s>>>(buf.mean, buf.vb, buf.rowsum_abs, K, buf.summary);
    check_cuda(cudaGetLastError(), "bside summary launch");
}

}  // namespace vabft_dev
