// Block-wise (tile-level) V-ABFT thresholds in three launches (PAPER.md
// "Integration with Block-wise ABFT"):
//
//   T[i][J] = sum over k-tiles kt, in order, of
//             threshold_row(row_stats(A[i, kt]), BStatsSummary(B[kt, J]), |J|, e_max[kt])
//
// i.e. the reference's vabft_thresholds (threshold_vabft.cpp:54-61) applied to
// every (A[:, kt], B[kt, J]) slice pair and accumulated over the k-tiles —
// the composition paper_2602_08043_b200/blockwise.py runs slice by slice
// through the host. Here:
//   1. seg_stats_kernel: row_stats (stats.cpp:9-32) of every row segment, one
//      thread per (row, segment) running the reference's sequential Neumaier
//      loop over its segment — A rows cut into k-tiles, B rows into column
//      blocks (bit-exact by construction: the same operations in the same
//      order);
//   2. seg_summary_kernel: BStatsSummary::from (threshold_vabft.cpp:15-26)
//      for every (k-tile, column block): three sequential FP64 sums over the
//      k-tile's rows, one thread per (pair, sum) — independent chains, so
//      they run side by side instead of one 4096-long chain;
//   3. blockwise_t_kernel: one thread per (row, column block) adds the
//      k-tiles' threshold_row totals in k-tile order.
#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"

namespace vabft_dev {

namespace {

// row_stats of X[r][s*seg : min((s+1)*seg, cols)] for every (r, s); out
// arrays [rows][nseg]. The reference throws on a non-finite value: flagged.
template <int F>
__global__ void __launch_bounds__(128) seg_stats_kernel(const typename Elem<F>::T* __restrict__ X, int64_t rows,
                                                        int64_t cols, int64_t ld, int64_t seg, int64_t nseg,
                                                        double* mean, double* vb, int* nonfinite) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= rows * nseg) return;
    const int64_t r = t / nseg, sg = t - r * nseg;
    const int64_t c0 = sg * seg, c1 = c0 + seg < cols ? c0 + seg : cols;
    const typename Elem<F>::T* row = X + r * ld;
    Neu n;
    double mx = Elem<F>::d(row[c0]), mn = mx;
    bool bad = false;
    for (int64_t q = c0; q < c1; ++q) {
        const double x = Elem<F>::d(row[q]);
        bad |= !isfinite(x);
        n.add(x);
        mx = fmax(mx, x);
        mn = fmin(mn, x);
    }
    if (bad) atomicExch(nonfinite, 1);
    double m, v;
    stats_finish(n, mx, mn, c1 - c0, &m, &v);
    mean[t] = m;
    vb[t] = v;
}

// BStatsSummary::from over rows [kt*tile_k, ...) of column block J: thread
// (kt, J, which) runs sum |mean|, sum mean^2 or sum var_bound in row order.
__global__ void __launch_bounds__(128) seg_summary_kernel(const double* __restrict__ mean,
                                                          const double* __restrict__ vb, int64_t K, int64_t tile_k,
                                                          int64_t nkt, int64_t nJ, double* summary /* [nkt][nJ][3] */) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nkt * nJ * 3) return;
    const int which = int(t % 3);
    const int64_t pair = t / 3, kt = pair / nJ, J = pair - kt * nJ;
    const int64_t k0 = kt * tile_k, k1 = k0 + tile_k < K ? k0 + tile_k : K;
    double acc = 0.0;
    if (which == 0) {
        for (int64_t k = k0; k < k1; ++k) acc = __dadd_rn(acc, fabs(mean[k * nJ + J]));
    } else if (which == 1) {
        for (int64_t k = k0; k < k1; ++k) {
            const double x = mean[k * nJ + J];
            acc = __dadd_rn(acc, __dmul_rn(x, x));
        }
    } else {
        for (int64_t k = k0; k < k1; ++k) acc = __dadd_rn(acc, vb[k * nJ + J]);
    }
    summary[pair * 3 + which] = acc;
}

__global__ void __launch_bounds__(256) blockwise_t_kernel(int64_t M, int64_t N, int64_t tile_n, int64_t nkt,
                                                          int64_t nJ, const double* __restrict__ amean,
                                                          const double* __restrict__ avb,
                                                          const double* __restrict__ summary,
                                                          const double* __restrict__ e_max, double c_sigma,
                                                          double* T) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= M * nJ) return;
    const int64_t i = t / nJ, J = t - i * nJ;
    const int64_t nj = (J + 1) * tile_n < N ? tile_n : N - J * tile_n;
    double acc = 0.0;
    for (int64_t kt = 0; kt < nkt; ++kt) {
        const double* bs = summary + (kt * nJ + J) * 3;
        acc = __dadd_rn(acc, vabft_threshold_total(amean[i * nkt + kt], avb[i * nkt + kt], bs[0], bs[1], bs[2], nj,
                                                   e_max[kt], c_sigma));
    }
    T[t] = acc;
}

template <int F>
void seg_stats(const void* X, int64_t rows, int64_t cols, int64_t ld, int64_t seg, double* mean, double* vb,
               int* nonfinite, cudaStream_t s) {
    const int64_t nseg = (cols + seg - 1) / seg;
    const int64_t n = rows * nseg;
    seg_stats_kernel<F><<<unsigned((n + 127) / 128), 128, 0, s>>>(static_cast<const typename Elem<F>::T*>(X), rows,
                                                                  cols, ld, seg, nseg, mean, vb, nonfinite);
}

}  // namespace

void launch_blockwise_thresholds(int fmt, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                                 const void* B, int64_t ldb, int64_t tile_k, int64_t tile_n, const double* e_max,
                                 double c_sigma, double* T, double* work, int* nonfinite, cudaStream_t s) {
    const int64_t nkt = (K + tile_k - 1) / tile_k, nJ = (N + tile_n - 1) / tile_n;
    double* amean = work;
    double* avb = amean + M * nkt;
    double* bmean = avb + M * nkt;
    double* bvb = bmean + K * nJ;
    double* summary = bvb + K * nJ;
    auto run = [&](auto tagF) {
        constexpr int F = decltype(tagF)::value;
        seg_stats<F>(A, M, K, lda, tile_k, amean, avb, nonfinite, s);
        seg_stats<F>(B, K, N, ldb, tile_n, bmean, bvb, nonfinite, s);
    };
    switch (fmt) {
        case VABFT_BF16: run(std::integral_constant<int, VABFT_BF16>{}); break;
        case VABFT_FP16: run(std::integral_constant<int, VABFT_FP16>{}); break;
        case VABFT_FP32: run(std::integral_constant<int, VABFT_FP32>{}); break;
        case VABFT_FP64: run(std::integral_constant<int, VABFT_FP64>{}); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
    const int64_t nch = nkt * nJ * 3;
    seg_summary_kernel<<<unsigned((nch + 127) / 128), 128, 0, s>>>(bmean, bvb, K, tile_k, nkt, nJ, summary);
    const int64_t nt = M * nJ;
    blockwise_t_kernel<<<unsigned((nt + 255) / 256), 256, 0, s>>>(M, N, tile_n, nkt, nJ, amean, avb, summary, e_max,
                                                                  c_sigma, T);
    check_cuda(cudaGetLastError(), "blockwise thresholds launch");
}

size_t blockwise_work_doubles(int64_t M, int64_t N, int64_t K, int64_t tile_k, int64_t tile_n) {
    const int64_t nkt = (K + tile_k - 1) / tile_k, nJ = (N + tile_n - 1) / tile_n;
    return size_t(2 * M * nkt + 2 * K * nJ + 3 * nkt * nJ);
}

}  // namespace vabft_dev
