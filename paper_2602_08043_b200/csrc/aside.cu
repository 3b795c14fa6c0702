// K1 (A side, per GEMM) — the HBM-streaming statistics pass of the fused
// V-ABFT GEMM for 16-bit A:
//   row_stats(A row)          proj/src/stats.cpp:9-32
//   threshold_row -> T_i      proj/src/threshold_vabft.cpp:28-42, 54-61
//   A (B r1), A (B r2)        proj/src/checksum.cpp:103-146 (FP32, blocked:128)
//   max|A| (A-ABFT y)         proj/src/threshold_aabft.cpp:38-48
//
// Mapping: a CTA owns 32 consecutive rows (lane = row) and its W warps split
// the 128-element blocks of K round-robin. Each lane streams its own row in
// 128-byte batches (8 x 16 B loads in flight per lane), the B r values are
// warp-uniform broadcast loads, and the per-block checksum partials go to
// shared memory so warp 0 can combine them in block order (NativeBlocked(128)
// exactly as reduce_terms does, precision.cpp:360-371).
//
// Row sum: plain FP64 adds in any order are EXACT whenever
// n * max|x| < 2^(53 + lsb(min nonzero |x|)); then the result equals the
// reference's sequential Neumaier sum bit for bit. The guard is evaluated per
// row from packed 16-bit max/min/min-nonzero trackers; rows that fail it are
// recomputed by the owning lane with the reference's sequential Neumaier
// pass, so the mean (and T_i) is bit-exact in every case.
#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "stats.hpp"

namespace vabft_dev {

namespace {

constexpr int kRowsPerCta = 32;
constexpr int kMaxWarps = 16;

template <int F>
__device__ __forceinline__ uint32_t pmax2(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (F == VABFT_BF16)
        asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else
        asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
template <int F>
__device__ __forceinline__ uint32_t pmin2(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (F == VABFT_BF16)
        asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else
        asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t pminu2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
// per 16-bit half: magnitude - 1, with zero mapped to 0x7FFF (above every
// finite magnitude), so an unsigned min tracks the smallest NONZERO |x|.
__device__ __forceinline__ uint32_t mag_minus_one(uint32_t w) {
    return (((w & 0x7FFF7FFFu) | 0x80008000u) - 0x00010001u) & 0x7FFF7FFFu;
}

template <int F>
__device__ __forceinline__ bool guard_exact(float max_abs, uint32_t mnz_pat, int64_t n) {
    if (mnz_pat >= 0x7FFFu) return true;  // every element zero
    if (!isfinite(max_abs)) return false;
    const uint32_t pat = mnz_pat + 1;  // smallest nonzero magnitude pattern
    int e, lsb;
    if constexpr (F == VABFT_BF16) {
        const int ef = int((pat >> 7) & 0xFF);
        e = (ef == 0 ? 1 : ef) - 127;
        lsb = e - 7;
    } else {
        const int ef = int((pat >> 10) & 0x1F);
        e = (ef == 0 ? 1 : ef) - 15;
        lsb = e - 10;
    }
    const int top = ilogbf(max_abs) + 1 + (64 - __clzll(static_cast<unsigned long long>(n)));
    return top <= 53 + lsb;
}

template <int F>
__global__ void __launch_bounds__(kRowsPerCta * kMaxWarps, 1)
    aside_kernel(const uint16_t* __restrict__ A, int64_t M, int64_t K, int64_t N,
                 const float* __restrict__ br1, const float* __restrict__ br2,
                 const double* __restrict__ bsum, int quantize_cr, double e_max, double c_sigma,
                 double* T, double* cr1, double* cr2, double* max_abs_a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nblk = (K + 127) / 128;
    float* sp = reinterpret_cast<float*>(smem);                               // [2][nblk][32]
    double* ssum = reinterpret_cast<double*>(smem + 8 * nblk * 32);           // [W][32]
    uint32_t* smax = reinterpret_cast<uint32_t*>(ssum + W * 32);              // [W][32]
    uint32_t* smin = smax + W * 32;
    uint32_t* smnz = smin + W * 32;

    const int64_t row = int64_t(blockIdx.x) * kRowsPerCta + lane;
    const bool live = row < M;
    const uint16_t* arow = A + (live ? row : M - 1) * K;

    double s0 = 0.0, s1 = 0.0;
    // running packed trackers (two 16-bit halves each)
    uint32_t vmax = F == VABFT_BF16 ? 0xFF80FF80u : 0xFC00FC00u;  // -inf, -inf
    uint32_t vmin = F == VABFT_BF16 ? 0x7F807F80u : 0x7C007C00u;  // +inf, +inf
    uint32_t vmnz = 0x7FFF7FFFu;
    for (int64_t b = warp; b < nblk; b += W) {
        const int64_t k0 = b * 128;
        const int kn = int((K - k0) < 128 ? (K - k0) : 128);  // multiple of 8
        float p1 = 0.0f, p2 = 0.0f;
        for (int c = 0; c < kn; c += 64) {
            uint4 w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (c + 8 * q < kn) w[q] = __ldg(reinterpret_cast<const uint4*>(arow + k0 + c + 8 * q));
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (c + 8 * q >= kn) break;
                const float4* g1 = reinterpret_cast<const float4*>(br1 + k0 + c + 8 * q);
                const float4* g2 = reinterpret_cast<const float4*>(br2 + k0 + c + 8 * q);
                const float4 u0 = __ldg(g1), u1 = __ldg(g1 + 1), v0 = __ldg(g2), v1 = __ldg(g2 + 1);
                const float b1[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                const float b2[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                const uint32_t ws[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    vmax = pmax2<F>(vmax, ws[h]);
                    vmin = pmin2<F>(vmin, ws[h]);
                    vmnz = pminu2(vmnz, mag_minus_one(ws[h]));
                    const float xa = Elem<F>::f(uint16_t(ws[h] & 0xFFFFu));
                    const float xb = Elem<F>::f(uint16_t(ws[h] >> 16));
                    s0 = __dadd_rn(s0, double(xa));
                    s1 = __dadd_rn(s1, double(xb));
                    p1 = __fadd_rn(p1, __fmul_rn(b1[2 * h], xa));
                    p2 = __fadd_rn(p2, __fmul_rn(b2[2 * h], xa));
                    p1 = __fadd_rn(p1, __fmul_rn(b1[2 * h + 1], xb));
                    p2 = __fadd_rn(p2, __fmul_rn(b2[2 * h + 1], xb));
                }
            }
        }
        sp[(0 * nblk + b) * 32 + lane] = p1;
        sp[(1 * nblk + b) * 32 + lane] = p2;
    }
    ssum[warp * 32 + lane] = __dadd_rn(s0, s1);
    smax[warp * 32 + lane] = vmax;
    smin[warp * 32 + lane] = vmin;
    smnz[warp * 32 + lane] = vmnz;
    __syncthreads();
    if (warp != 0 || !live) return;

    // block partials combined in block order (blocked:128)
    float t1 = 0.0f, t2 = 0.0f;
    for (int64_t b = 0; b < nblk; ++b) {
        t1 = __fadd_rn(t1, sp[(0 * nblk + b) * 32 + lane]);
        t2 = __fadd_rn(t2, sp[(1 * nblk + b) * 32 + lane]);
    }
    double sum = 0.0;
    uint32_t gmax = smax[lane], gmin = smin[lane], gmnz = smnz[lane];
    for (int q = 0; q < W; ++q) {
        sum = __dadd_rn(sum, ssum[q * 32 + lane]);
        gmax = pmax2<F>(gmax, smax[q * 32 + lane]);
        gmin = pmin2<F>(gmin, smin[q * 32 + lane]);
        gmnz = pminu2(gmnz, smnz[q * 32 + lane]);
    }
    const float mx = fmaxf(Elem<F>::f(uint16_t(gmax & 0xFFFFu)), Elem<F>::f(uint16_t(gmax >> 16)));
    const float mn = fminf(Elem<F>::f(uint16_t(gmin & 0xFFFFu)), Elem<F>::f(uint16_t(gmin >> 16)));
    const uint32_t mnz = min(gmnz & 0xFFFFu, gmnz >> 16);
    const float amax = fmaxf(fabsf(mx), fabsf(mn));
    if (!guard_exact<F>(amax, mnz, K)) {
        // the reference's sequential Neumaier pass (stats.cpp:12-24)
        Neu s;
        for (int64_t q = 0; q < K; ++q) s.add(double(Elem<F>::f(arow[q])));
        sum = __dadd_rn(s.s, s.c);
    }
    Neu fin;
    fin.s = sum;
    double mean, vb;
    stats_finish(fin, double(mx), double(mn), K, &mean, &vb);
    T[row] = vabft_threshold_total(mean, vb, bsum[0], bsum[1], bsum[2], N, e_max, c_sigma);
    if (quantize_cr) {
        t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
        t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
    }
    cr1[row] = double(t1);
    cr2[row] = double(t2);
    atomic_max_nonneg(max_abs_a, double(amax));
}

}  // namespace

void launch_aside(int fmt, int64_t M, int64_t K, int64_t N, const void* A, const BsideBuffers& buf,
                  int quantize_cr, double e_max, double c_sigma, double* T, double* cr1, double* cr2,
                  double* max_abs_a, cudaStream_t s) {
    if (K % 8 != 0) fail(VABFT_UNSUPPORTED, "A-side stats: K must be a multiple of 8");
    const int64_t nblk = (K + 127) / 128;
    const int W = int(nblk < kMaxWarps ? nblk : kMaxWarps);
    const size_t smem = size_t(8 * nblk * 32) + size_t(W) * 32 * (8 + 4 * 3);
    const dim3 grid(unsigned((M + kRowsPerCta - 1) / kRowsPerCta)), block(32 * W);
    const uint16_t* a = static_cast<const uint16_t*>(A);
    if (fmt == VABFT_BF16) {
        ensure_smem_attr(reinterpret_cast<const void*>(aside_kernel<VABFT_BF16>), 96 * 1024);
        aside_kernel<VABFT_BF16><<<grid, block, smem, s>>>(a, M, K, N, buf.br1, buf.br2, buf.summary, quantize_cr, e_max, c_sigma, T, cr1, cr2, max_abs_a);
    } else if (fmt == VABFT_FP16) {
        ensure_smem_attr(reinterpret_cast<const void*>(aside_kernel<VABFT_FP16>), 96 * 1024);
        aside_kernel<VABFT_FP16><<<grid, block, smem, s>>>(a, M, K, N, buf.br1, buf.br2, buf.summary, quantize_cr, e_max, c_sigma, T, cr1, cr2, max_abs_a);
    } else {
        fail(VABFT_UNSUPPORTED, "A-side stats: BF16/FP16 only");
    }
    check_cuda(cudaGetLastError(), "aside launch");
}

}  // namespace vabft_dev
