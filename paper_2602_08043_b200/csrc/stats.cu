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
    double mx = -INFINITY, mn = INFINITY;
    double ps = 0.0, mnz = INFINITY;  // lane partial of the row sum, min nonzero |x|
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
                mx = fmax(mx, x);
                mn = fmin(mn, x);
                ps = __dadd_rn(ps, x);
                if (x != 0.0) mnz = fmin(mnz, fabs(x));
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
    mx = warp_max(mx);
    mn = warp_min(mn);
    mnz = warp_min(mnz);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ps = __dadd_rn(ps, __shfl_xor_sync(0xffffffffu, ps, o));
    const unsigned anybad = __ballot_sync(0xffffffffu, bad);
    // Every partial sum is exact in FP64 — so the lanes' sum in any order
    // equals both the sequential Neumaier sum (zero compensation) and the
    // plain sequential sum — when N max|x| < 2^(53 + lsb), lsb the last bit
    // of the smallest nonzero |x| (the 16-bit pass's guard_exact, for t-bit
    // formats). Most FP32 N(0,1) rows pass (4096 x 4096 with the fallback
    // below: 439 -> 235 us);
    // the others, and nearly all FP64 rows, take the sequential loops.
    bool exact = !anybad;
    if (exact && mnz < INFINITY) {
        constexpr int kT = F == VABFT_FP32 ? 24 : F == VABFT_FP64 ? 53 : F == VABFT_FP16 ? 11 : 8;
        const int lsb = ilogb(mnz) - (kT - 1);
        const int top = ilogb(fmax(fabs(mx), fabs(mn))) + 1 + (64 - __clzll(static_cast<unsigned long long>(N)));
        exact = top <= 53 + lsb;
    }
    Neu n;
    double plain = 0.0;
    if (exact) {
        n.s = ps;
        plain = ps;
    } else {
        // the reference's loops, warp-cooperative: the warp stages 256
        // elements at a time in its shared-memory slice (coalesced loads),
        // lane 0 reads 32 per batch ahead of the two chains (as the wide
        // verify tail's fallback: no shuffle or branch on the chains)
        constexpr int kChunk = 256;
        using T = typename Elem<F>::T;
        __shared__ __align__(16) T stage[kWarpsPerBlock][kChunk];
        T* st = stage[threadIdx.x >> 5];
        for (int64_t j0 = 0; j0 < N; j0 += kChunk) {
            const int cnt = N - j0 < kChunk ? int(N - j0) : kChunk;  // warp-uniform
            __syncwarp();
#pragma unroll
            for (int r = 0; r < kChunk / 32; ++r) {
                const int q = r * 32 + lane;
                if (q < cnt) st[q] = row[j0 + q];
            }
            __syncwarp();
            if (lane == 0) {
                int q = 0;
                for (; q + 32 <= cnt; q += 32) {
                    double xs[32];
#pragma unroll
                    for (int l = 0; l < 32; ++l) xs[l] = Elem<F>::d(st[q + l]);
#pragma unroll
                    for (int l = 0; l < 32; ++l) {
                        n.add(xs[l]);
                        plain = __dadd_rn(plain, xs[l]);
                    }
                }
                for (; q < cnt; ++q) {
                    const double x = Elem<F>::d(st[q]);
                    n.add(x);
                    plain = __dadd_rn(plain, x);
                }
            }
        }
    }
    if (lane == 0) {
        if (anybad) atomicExch(nonfinite, 1);
        // n / plain (above) are the reference's sequential loops over the row
        // (FP32 / FP64 weights; the 16-bit pass is bside_rows16_kernel):
        // Neumaier for the mean (stats.cpp:12-24), the plain FP64 sum for
        // A-ABFT's computed y (threshold_aabft.cpp:42-46) — bit-exact for
        // every input
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
        rowsum_abs[k] = fabs(plain);
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

// ----------------------------------------- B side, 16-bit formats (HBM pass)
// One warp per B row; the row streams through a per-warp 8 KiB shared-memory
// stage (32 blocks of 128 elements) with coalesced 16-byte loads, written
// with a 16-byte-chunk XOR swizzle (chunk c of block b at c ^ (b & 15)) so
// that lane l then walks its own block l (the reference's sequential order
// inside a 128-element block) without bank conflicts. Per element: FP32
// B r1 / B r2 block partials (no FMA), an FP64 partial of the row sum (plain
// adds: exact under the guard below), packed max / min / min-nonzero
// trackers. The row sum is exact in any order when
// n max|x| < 2^(53 + lsb(min nonzero |x|)) (tail.cuh guard_exact), and then
// equals both the reference's Neumaier sum (row_stats) and its plain
// sequential sum (aabft_computed_y); rows failing the guard are redone
// sequentially by lane 0. The last CTA to finish computes the summary
// (BStatsSummary::from's sequential FP64 sums and max_k |sum_j B|).
constexpr int kB16Warps = 8;
constexpr int kB16StageGranules = 32 * 16;  // 32 blocks x 16 granules of 8 elements

template <int F>
__device__ __forceinline__ float b16_f(uint32_t bits) {
    return bits16_to_float<F>(uint16_t(bits));
}

// BStatsSummary::from's sequential FP64 sums (threshold_vabft.cpp:15-26) and
// max_k |sum_j B| (threshold_aabft.cpp:38-48), by the whole CTA: chunks of
// the inputs are staged into shared memory with coalesced loads, then thread
// 0 runs the four independent serial chains out of shared memory.
__device__ void bside_summary_cta(const double* mean, const double* vb, const double* rowsum_abs, int64_t K,
                                  double* summary, double* sm, int sm_doubles) {
    const int chunk = sm_doubles / 3;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int64_t c0 = 0; c0 < K; c0 += chunk) {
        const int cnt = int(K - c0 < chunk ? K - c0 : chunk);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            sm[i] = __ldcg(mean + c0 + i);
            sm[chunk + i] = __ldcg(vb + c0 + i);
            sm[2 * chunk + i] = __ldcg(rowsum_abs + c0 + i);
        }
        __syncthreads();
        // one chain per warp (lane 0 of warps 0..3): the chains run
        // concurrently at FP64 add latency (~8 cycles on B200) instead of
        // sharing one thread's issue slots
        if ((threadIdx.x & 31) == 0) {
            switch (threadIdx.x >> 5) {
                case 0:
#pragma unroll 8
                    for (int i = 0; i < cnt; ++i) a0 = __dadd_rn(a0, fabs(sm[i]));
                    break;
                case 1:
#pragma unroll 8
                    for (int i = 0; i < cnt; ++i) a1 = __dadd_rn(a1, __dmul_rn(sm[i], sm[i]));
                    break;
                case 2:
#pragma unroll 8
                    for (int i = 0; i < cnt; ++i) a2 = __dadd_rn(a2, sm[chunk + i]);
                    break;
                case 3:
#pragma unroll 8
                    for (int i = 0; i < cnt; ++i) a3 = fmax(a3, sm[2 * chunk + i]);
                    break;
                default: break;
            }
        }
    }
    if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < 4) {
        const int c = threadIdx.x >> 5;
        summary[c] = c == 0 ? a0 : c == 1 ? a1 : c == 2 ? a2 : a3;
    }
}

__global__ void __launch_bounds__(32 * kB16Warps) bside_summary_cta_kernel(const double* mean, const double* vb,
                                                                           const double* rowsum_abs, int64_t K,
                                                                           double* summary) {
    extern __shared__ uint4 sum_stage[];
    bside_summary_cta(mean, vb, rowsum_abs, K, summary, reinterpret_cast<double*>(sum_stage),
                      kB16Warps * kB16StageGranules * 2);
}

template <int F>
__global__ void __launch_bounds__(32 * kB16Warps) bside_rows16_kernel(const uint16_t* __restrict__ B, int64_t K,
                                                                      int64_t N, int quantize_br, BsideBuffers buf,
                                                                      unsigned int* done) {
    extern __shared__ uint4 b16_stage[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = int64_t(blockIdx.x) * kB16Warps + w;
    if (k < K) {
        uint4* st = b16_stage + w * kB16StageGranules;
        const uint4* row = reinterpret_cast<const uint4*>(B + k * N);
        const int64_t ng = N / 8, nblk = (N + 127) / 128;
        // four independent FP64 partials per lane (the sum is order-free under
        // the guard; one chain would serialize on FP64 add latency)
        double sp[4] = {0.0, 0.0, 0.0, 0.0};
        float t1 = 0.0f, t2 = 0.0f;
        uint32_t vmax = F == VABFT_BF16 ? 0xFF80FF80u : 0xFC00FC00u;
        uint32_t vmin = F == VABFT_BF16 ? 0x7F807F80u : 0x7C007C00u;
        uint32_t vmnz = 0x7FFF7FFFu, vmag = 0u;
        for (int64_t b0 = 0; b0 < nblk; b0 += 32) {
            const int64_t g0 = b0 * 16;
            const int gcnt = int(ng - g0 < kB16StageGranules ? ng - g0 : kB16StageGranules);
            __syncwarp();
            for (int q = lane; q < gcnt; q += 32) {
                const int blk = q >> 4, c = q & 15;
                st[blk * 16 + (c ^ (blk & 15))] = __ldcs(row + g0 + q);  // streamed: read once
            }
            __syncwarp();
            float p1 = 0.0f, p2 = 0.0f;
            const int64_t blk = b0 + lane;
            if (blk < nblk) {
                const int nc = int(ng - blk * 16 < 16 ? ng - blk * 16 : 16);
                for (int c = 0; c < nc; ++c) {
                    const uint4 v = st[lane * 16 + (c ^ (lane & 15))];
                    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
                    const float jb = float(blk * 128 + c * 8 + 1);  // weight of element 0 (exact: N <= 2^24)
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        uint32_t d;
                        if constexpr (F == VABFT_BF16) {
                            asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(ws[h]));
                            vmax = d;
                            asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(ws[h]));
                            vmin = d;
                        } else {
                            asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(ws[h]));
                            vmax = d;
                            asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(ws[h]));
                            vmin = d;
                        }
                        const uint32_t mag = ws[h] & 0x7FFF7FFFu;
                        asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmag), "r"(mag));
                        vmag = d;
                        asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmnz),
                            "r"(((mag | 0x80008000u) - 0x00010001u) & 0x7FFF7FFFu));
                        vmnz = d;
                        const float xa = b16_f<F>(ws[h] & 0xFFFFu), xb = b16_f<F>(ws[h] >> 16);
                        sp[h] = __dadd_rn(sp[h], __dadd_rn(double(xa), double(xb)));  // exact under the guard
                        p1 = __fadd_rn(p1, xa);
                        p2 = __fadd_rn(p2, __fmul_rn(__fadd_rn(jb, float(2 * h)), xa));
                        p1 = __fadd_rn(p1, xb);
                        p2 = __fadd_rn(p2, __fmul_rn(__fadd_rn(jb, float(2 * h + 1)), xb));
                    }
                }
            }
            const int cnt = int(nblk - b0 < 32 ? nblk - b0 : 32);
            for (int l = 0; l < cnt; ++l) {  // block partials in block order
                t1 = __fadd_rn(t1, __shfl_sync(0xffffffffu, p1, l));
                t2 = __fadd_rn(t2, __shfl_sync(0xffffffffu, p2, l));
            }
        }
        // combine lanes: the FP64 partials (exact under the guard), trackers
        double s = __dadd_rn(__dadd_rn(sp[0], sp[1]), __dadd_rn(sp[2], sp[3]));
        vmag = max(vmag & 0xFFFFu, vmag >> 16);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, m));
            uint32_t o = __shfl_xor_sync(0xffffffffu, vmax, m), d;
            if constexpr (F == VABFT_BF16) asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(o));
            else asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(o));
            vmax = d;
            o = __shfl_xor_sync(0xffffffffu, vmin, m);
            if constexpr (F == VABFT_BF16) asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(o));
            else asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(o));
            vmin = d;
            vmag = max(vmag, __shfl_xor_sync(0xffffffffu, vmag, m));
            o = __shfl_xor_sync(0xffffffffu, vmnz, m);
            asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmnz), "r"(o));
            vmnz = d;
        }
        if (lane == 0) {
            const bool finite = vmag < (F == VABFT_BF16 ? 0x7F80u : 0x7C00u);
            if (!finite) atomicExch(buf.nonfinite, 1);
            const double mx = double(fmaxf(b16_f<F>(vmax & 0xFFFFu), b16_f<F>(vmax >> 16)));
            const double mn = double(fminf(b16_f<F>(vmin & 0xFFFFu), b16_f<F>(vmin >> 16)));
            const uint32_t mz = min(vmnz & 0xFFFFu, vmnz >> 16);
            Neu n;
            double plain;
            if (finite && guard_exact<F>(float(fmax(fabs(mx), fabs(mn))), mz, N)) {
                n.s = s;
                plain = s;
            } else {  // the reference's sequential loops over the row
                const uint16_t* r = B + k * N;
                plain = 0.0;
                for (int64_t j = 0; j < N; ++j) {
                    const double x = double(b16_f<F>(r[j]));
                    n.add(x);
                    plain = __dadd_rn(plain, x);
                }
            }
            double m, v;
            stats_finish(n, mx, mn, N, &m, &v);
            buf.mean[k] = m;
            buf.vb[k] = v;
            if (quantize_br) {
                t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
                t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
            }
            buf.br1[k] = t1;
            buf.br2[k] = t2;
            buf.rowsum_abs[k] = fabs(plain);
        }
    }
    if (done == nullptr) return;
    // last CTA: the summary (self-resetting counter)
    __syncthreads();
    __shared__ unsigned int last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (last) {  // CTA-uniform
        __threadfence();
        bside_summary_cta(buf.mean, buf.vb, buf.rowsum_abs, K, buf.summary, reinterpret_cast<double*>(b16_stage),
                          kB16Warps * kB16StageGranules * 2);
        if (threadIdx.x == 0) *done = 0u;
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
    if ((fmt == VABFT_BF16 || fmt == VABFT_FP16) && N % 8 == 0 && N <= (int64_t(1) << 24)) {
        const unsigned grid16 = unsigned((K + kB16Warps - 1) / kB16Warps);
        const size_t smem = size_t(kB16Warps) * kB16StageGranules * sizeof(uint4);  // 64 KiB
        auto run = [&](auto kern) {
            ensure_smem_attr(reinterpret_cast<const void*>(kern), int(smem));
            static const bool split = std::getenv("VABFT_BSIDE_SPLIT") != nullptr;  // developer: time the parts
            kern<<<grid16, 32 * kB16Warps, smem, s>>>(static_cast<const uint16_t*>(B), K, N, quantize_br, buf,
                                                       split ? nullptr : buf.done);
            if (split) buf.done = nullptr;
        };
        if (fmt == VABFT_BF16) run(bside_rows16_kernel<VABFT_BF16>);
        else run(bside_rows16_kernel<VABFT_FP16>);
        check_cuda(cudaGetLastError(), "bside16 launch");
        if (buf.done == nullptr) {
            ensure_smem_attr(reinterpret_cast<const void*>(bside_summary_cta_kernel), int(smem));
            bside_summary_cta_kernel<<<1, 32 * kB16Warps, smem, s>>>(buf.mean, buf.vb, buf.rowsum_abs, K,
                                                                     buf.summary);
            check_cuda(cudaGetLastError(), "bside summary launch");
        }
        return;
    }
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
