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
//   1. seg_stats_kernel: row_stats (stats.cpp:9-32) of every row segment, lane
//      = row running the reference's sequential Neumaier loop over its
//      segment from a shared-memory tile — A rows cut into k-tiles, B rows
//      into column blocks (bit-exact by construction: the same operations in
//      the same order);
//   2. seg_summary_kernel: BStatsSummary::from (threshold_vabft.cpp:15-26)
//      for every (k-tile, column block): three sequential FP64 sums over the
//      k-tile's rows, one warp per (pair, sum) — independent chains, so they
//      run side by side instead of one 4096-long chain;
//   3. blockwise_t_kernel: one thread per (row, column block) adds the
//      k-tiles' threshold_row totals in k-tile order.
#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"

namespace vabft_dev {

namespace {

// row_stats of X[r][s*seg : min((s+1)*seg, cols)] for every (r, s); out
// arrays [rows][nseg]. A warp takes 32 consecutive rows of one segment: the
// segment streams through the warp's shared-memory tile in 32 x 32 sub-tiles
// (lane = column: coalesced row segments; the next sub-tile's loads in
// registers while this one is folded) and lane = row runs the reference's
// sequential Neumaier loop over its row's segment — all lanes busy on the
// FP64 pipe. The reference throws on a non-finite value: flagged.
constexpr int kSegWarps = 4;
template <int F>
__global__ void __launch_bounds__(32 * kSegWarps) seg_stats_kernel(const typename Elem<F>::T* __restrict__ X,
                                                                   int64_t rows, int64_t cols, int64_t ld,
                                                                   int64_t seg, int64_t nseg, double* mean,
                                                                   double* vb, int* nonfinite) {
    __shared__ double tile[kSegWarps][32][33];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ngr = (rows + 31) / 32;
    const int64_t task = int64_t(blockIdx.x) * kSegWarps + w;  // (row group, segment)
    if (task >= ngr * nseg) return;
    const int64_t rg = task / nseg, sg = task - rg * nseg;
    const int64_t r0 = rg * 32, c0 = sg * seg, c1 = c0 + seg < cols ? c0 + seg : cols;
    const int nr = int(rows - r0 < 32 ? rows - r0 : 32);
    const typename Elem<F>::T* base = X + r0 * ld;
    double v[32];
    auto load = [&](int64_t cq) {
        const int64_t c = cq + lane;
        const bool in = c < c1;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) v[rr] = (rr < nr && in) ? Elem<F>::d(base[rr * ld + c]) : 0.0;
    };
    Neu n;
    double mx = 0.0, mn = 0.0;
    bool bad = false, first = true;
    load(c0);
    for (int64_t cq = c0; cq < c1; cq += 32) {
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) tile[w][rr][lane] = v[rr];
        __syncwarp();
        if (cq + 32 < c1) load(cq + 32);  // in flight during the fold
        const int cnt = int(c1 - cq < 32 ? c1 - cq : 32);
        if (first) {
            mx = mn = tile[w][lane][0];
            first = false;
        }
        for (int e = 0; e < cnt; ++e) {
            const double x = tile[w][lane][e];
            bad |= !isfinite(x);
            n.add(x);
            mx = fmax(mx, x);
            mn = fmin(mn, x);
        }
    }
    if (lane < nr) {
        if (bad) atomicExch(nonfinite, 1);
        double m, vv;
        stats_finish(n, mx, mn, c1 - c0, &m, &vv);
        const int64_t o = (r0 + lane) * nseg + sg;
        mean[o] = m;
        vb[o] = vv;
    }
}

// 16-bit variant with 16-byte row-segment loads: a sub-tile is 32 rows x 64
// elements, loaded as 8 x 16 bytes per lane (8 lanes per 128-byte row
// segment, coalesced) into registers one sub-tile ahead of the fold, staged
// raw (padded rows: conflict-free 16-byte reads), and lane = row converts
// while it runs the reference's Neumaier loop. Needs 16-byte aligned rows
// and segment starts (ld, seg multiples of 8; X 16-byte aligned).
template <int F>
__global__ void __launch_bounds__(32 * kSegWarps) seg_stats16_kernel(const uint16_t* __restrict__ X, int64_t rows,
                                                                     int64_t cols, int64_t ld, int64_t seg,
                                                                     int64_t nseg, double* mean, double* vb,
                                                                     int* nonfinite) {
    constexpr int kLd = 36;  // words per staged row (64 elements + pad)
    __shared__ __align__(16) uint32_t tile[kSegWarps][32 * kLd];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ngr = (rows + 31) / 32;
    const int64_t task = int64_t(blockIdx.x) * kSegWarps + w;
    if (task >= ngr * nseg) return;
    const int64_t rg = task / nseg, sg = task - rg * nseg;
    const int64_t r0 = rg * 32, c0 = sg * seg, c1 = c0 + seg < cols ? c0 + seg : cols;
    const int nr = int(rows - r0 < 32 ? rows - r0 : 32);
    const int rs = lane >> 3, ch = lane & 7;  // this lane loads rows 4 i + rs, chunk ch (8 elements)
    uint4 v[8];
    auto load = [&](int64_t cq) {
        const int64_t c = cq + ch * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + rs;
            v[i] = (rr < nr && c < c1) ? __ldcs(reinterpret_cast<const uint4*>(X + (r0 + rr) * ld + c))
                                       : make_uint4(0u, 0u, 0u, 0u);
        }
    };
    Neu n;
    float mx = 0.0f, mn = 0.0f;
    bool bad = false, first = true;
    uint32_t* mine = tile[w];
    load(c0);
    for (int64_t cq = c0; cq < c1; cq += 64) {
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(mine + (4 * i + rs) * kLd + ch * 4) = v[i];
        __syncwarp();
        if (cq + 64 < c1) load(cq + 64);  // in flight during the fold
        const int cnt = int(c1 - cq < 64 ? c1 - cq : 64);
        const uint32_t* trow = mine + lane * kLd;
        if (first) {
            mx = mn = bits16_to_float<F>(uint16_t(trow[0] & 0xFFFFu));
            first = false;
        }
        for (int e = 0; e < cnt; ++e) {
            const uint32_t wd = trow[e >> 1];
            const float xf = bits16_to_float<F>(uint16_t((e & 1) ? (wd >> 16) : (wd & 0xFFFFu)));
            bad |= !isfinite(xf);
            n.add(double(xf));
            mx = fmaxf(mx, xf);
            mn = fminf(mn, xf);
        }
    }
    if (lane < nr) {
        if (bad) atomicExch(nonfinite, 1);
        double m, vv;
        stats_finish(n, double(mx), double(mn), c1 - c0, &m, &vv);
        const int64_t o = (r0 + lane) * nseg + sg;
        mean[o] = m;
        vb[o] = vv;
    }
}

// BStatsSummary::from over rows [kt*tile_k, ...) of column block J: one warp
// per (kt, J, which) — the warp stages the k-tile's values in chunks of 256
// (coalesced-enough strided loads, all in flight) and lane 0 runs the
// sequential sum |mean|, sum mean^2 or sum var_bound in row order.
__global__ void __launch_bounds__(128) seg_summary_kernel(const double* __restrict__ mean,
                                                          const double* __restrict__ vb, int64_t K, int64_t tile_k,
                                                          int64_t nkt, int64_t nJ, double* summary /* [nkt][nJ][3] */) {
    __shared__ double buf[4][256];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = int64_t(blockIdx.x) * 4 + w;
    if (t >= nkt * nJ * 3) return;
    const int which = int(t % 3);
    const int64_t pair = t / 3, kt = pair / nJ, J = pair - kt * nJ;
    const int64_t k0 = kt * tile_k, k1 = k0 + tile_k < K ? k0 + tile_k : K;
    const double* src = which == 2 ? vb : mean;
    double acc = 0.0;
    for (int64_t c = k0; c < k1; c += 256) {
        const int cnt = int(k1 - c < 256 ? k1 - c : 256);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int q = e * 32 + lane;
            buf[w][q] = q < cnt ? src[(c + q) * nJ + J] : 0.0;
        }
        __syncwarp();
        if (lane == 0) {
            if (which == 0) {
                for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, fabs(buf[w][q]));
            } else if (which == 1) {
                for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, __dmul_rn(buf[w][q], buf[w][q]));
            } else {
                for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, buf[w][q]);
            }
        }
    }
    if (lane == 0) summary[pair * 3 + which] = acc;
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
    const int64_t tasks = (rows + 31) / 32 * nseg;
    if constexpr (F == VABFT_BF16 || F == VABFT_FP16) {
        // 16-byte chunks never cross a segment end or the matrix end
        if (ld % 8 == 0 && seg % 8 == 0 && cols % 8 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0) {
            seg_stats16_kernel<F><<<unsigned((tasks + kSegWarps - 1) / kSegWarps), 32 * kSegWarps, 0, s>>>(
                static_cast<const uint16_t*>(X), rows, cols, ld, seg, nseg, mean, vb, nonfinite);
            return;
        }
    }
    seg_stats_kernel<F><<<unsigned((tasks + kSegWarps - 1) / kSegWarps), 32 * kSegWarps, 0, s>>>(
        static_cast<const typename Elem<F>::T*>(X), rows, cols, ld, seg, nseg, mean, vb, nonfinite);
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
    seg_summary_kernel<<<unsigned((nch + 3) / 4), 128, 0, s>>>(bmean, bvb, K, tile_k, nkt, nJ, summary);
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
