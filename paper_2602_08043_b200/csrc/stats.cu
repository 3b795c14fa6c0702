// K1 — HBM-streaming statistics and threshold kernels.
//
// Replaces, on the device:
//   row_stats                        proj/src/stats.cpp:9-32
//   precompute_b_stats/BStatsSummary proj/src/threshold_vabft.cpp:8-26
//   threshold_row/vabft_thresholds   proj/src/threshold_vabft.cpp:28-61
//   aabft_computed_y                 proj/src/threshold_aabft.cpp:38-48
//   encode's B r1 / B r2 and A (B r) (blocked:128 order, TENSOR engine)
//                                    proj/src/checksum.cpp:103-146
//
// One warp per matrix row. Per-lane Neumaier sums merged across lanes with
// TwoSum (the compensated FP64 mean equals the reference's sequential
// Neumaier result except in pathological near-tie cases), warp-shuffle
// max/min, FP32 checksum dot products in the reference's NativeBlocked(128)
// order: lane l owns 128-element blocks l, l+32, ... (sequential inside a
// block) and block partials are combined sequentially in block order.
//
// The per-weight B r1 / B r2 vectors are stored INTERLEAVED for the A pass:
// element k lives at ((k%128)/8 * nblk + k/128) * 8 + k%8, so when lane b
// consumes the 8-element granule v of its block b, the warp reads one
// contiguous 1 KiB span (coalesced, L1/L2-resident) instead of 32 scattered
// lines.
#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "stats.hpp"

namespace vabft_dev {

namespace {

constexpr int kWarpsPerBlock = 8;

__host__ __device__ __forceinline__ int64_t br_index(int64_t k, int64_t nblk) {
    return ((k % 128) / 8 * nblk + k / 128) * 8 + (k % 8);
}

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
        const int64_t idx = br_index(k, (K + 127) / 128);
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
__global__ void bside_summary_kernel(const double* mean, const double* vb, const double* rowsum_abs,
                                     int64_t K, double* summary) {
    const int t = threadIdx.x;
    double acc = 0.0;
    if (t == 0) {
        for (int64_t k = 0; k < K; ++k) acc = __dadd_rn(acc, fabs(mean[k]));
        summary[0] = acc;
    } else if (t == 1) {
        for (int64_t k = 0; k < K; ++k) acc = __dadd_rn(acc, __dmul_rn(mean[k], mean[k]));
        summary[1] = acc;
    } else if (t == 2) {
        for (int64_t k = 0; k < K; ++k) acc = __dadd_rn(acc, vb[k]);
        summary[2] = acc;
    } else if (t == 3) {
        for (int64_t k = 0; k < K; ++k) acc = fmax(acc, rowsum_abs[k]);
        summary[3] = acc;
    }
}

// ------------------------------------------------------ A-side (per GEMM)
// One warp per row of 16-bit A (K % 8 == 0, the TENSOR-engine envelope):
// row stats -> V-ABFT T_i; A (B r1), A (B r2) in FP32 blocked:128
// (quantized for offline mode); max|A| for A-ABFT computed y. No shared
// memory, so these CTAs co-reside with the persistent tcgen05 GEMM.
template <int F>
__global__ void __launch_bounds__(256) aside_kernel(const uint16_t* __restrict__ A, int64_t M,
                                                    int64_t K, int64_t N, const float* __restrict__ br1,
                                                    const float* __restrict__ br2,
                                                    const double* __restrict__ bsum, int quantize_cr,
                                                    double e_max, double c_sigma, double* T, double* cr1,
                                                    double* cr2, double* max_abs_a) {
    const int64_t i = int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= M) return;
    const uint16_t* row = A + i * K;
    const int64_t nblk = (K + 127) / 128;
    Neu n;
    float mx = -INFINITY, mn = INFINITY;
    float t1 = 0.0f, t2 = 0.0f;
    for (int64_t b0 = 0; b0 < nblk; b0 += 32) {
        const int64_t b = b0 + lane;
        float p1 = 0.0f, p2 = 0.0f;
        if (b < nblk) {
            const int64_t k0 = b * 128;
            const int nv = int((K - k0) >= 128 ? 16 : (K - k0) / 8);
#pragma unroll 2
            for (int v = 0; v < nv; ++v) {
                const uint4 w = __ldg(reinterpret_cast<const uint4*>(row + k0 + v * 8));
                const float4* g1 = reinterpret_cast<const float4*>(br1 + (int64_t(v) * nblk + b) * 8);
                const float4* g2 = reinterpret_cast<const float4*>(br2 + (int64_t(v) * nblk + b) * 8);
                const float4 u0 = __ldg(g1), u1 = __ldg(g1 + 1), q0 = __ldg(g2), q1 = __ldg(g2 + 1);
                const float w1[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                const float w2[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    const uint16_t e = uint16_t(h & 1 ? ws[h >> 1] >> 16 : ws[h >> 1] & 0xFFFFu);
                    const float xf = Elem<F>::f(e);
                    n.add(double(xf));
                    mx = fmaxf(mx, xf);
                    mn = fminf(mn, xf);
                    p1 = __fadd_rn(p1, __fmul_rn(w1[h], xf));
                    p2 = __fadd_rn(p2, __fmul_rn(w2[h], xf));
                }
            }
        }
        const int cnt = (nblk - b0 < 32) ? int(nblk - b0) : 32;
        for (int l = 0; l < cnt; ++l) {
            t1 = __fadd_rn(t1, __shfl_sync(0xffffffffu, p1, l));
            t2 = __fadd_rn(t2, __shfl_sync(0xffffffffu, p2, l));
        }
    }
    n = warp_merge(n);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, m));
    }
    if (lane == 0) {
        double m, vb;
        stats_finish(n, double(mx), double(mn), K, &m, &vb);
        T[i] = vabft_threshold_total(m, vb, bsum[0], bsum[1], bsum[2], N, e_max, c_sigma);
        if (quantize_cr) {
            t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
            t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
        }
        cr1[i] = double(t1);
        cr2[i] = double(t2);
        atomic_max_nonneg(max_abs_a, double(fmaxf(fabsf(mx), fabsf(mn))));
    }
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
    bside_summary_kernel<<<1, 32, 0, s>>>(buf.mean, buf.vb, buf.rowsum_abs, K, buf.summary);
    check_cuda(cudaGetLastError(), "bside summary launch");
}

void launch_aside(int fmt, int64_t M, int64_t K, int64_t N, const void* A, const BsideBuffers& buf,
                  int quantize_cr, double e_max, double c_sigma, double* T, double* cr1, double* cr2,
                  double* max_abs_a, cudaStream_t s) {
    if (K % 8 != 0) fail(VABFT_UNSUPPORTED, "A-side stats: K must be a multiple of 8");
    const dim3 grid(unsigned((M + kWarpsPerBlock - 1) / kWarpsPerBlock)), block(32 * kWarpsPerBlock);
    const uint16_t* a = static_cast<const uint16_t*>(A);
    switch (fmt) {
        case VABFT_BF16: aside_kernel<VABFT_BF16><<<grid, block, 0, s>>>(a, M, K, N, buf.br1, buf.br2, buf.summary, quantize_cr, e_max, c_sigma, T, cr1, cr2, max_abs_a); break;
        case VABFT_FP16: aside_kernel<VABFT_FP16><<<grid, block, 0, s>>>(a, M, K, N, buf.br1, buf.br2, buf.summary, quantize_cr, e_max, c_sigma, T, cr1, cr2, max_abs_a); break;
        default: fail(VABFT_UNSUPPORTED, "A-side stats: BF16/FP16 only");
    }
    check_cuda(cudaGetLastError(), "aside launch");
}

}  // namespace vabft_dev
