// Per-weight B-side state in one HBM pass (K1, B side):
//   precompute_b_stats + BStatsSummary::from   proj/src/threshold_vabft.cpp:8-26
//     (row_stats per B row, stats.cpp:9-32)
//   encode's B r1 / B r2 in the fused path's NativeBlocked(128) order
//                                              proj/src/checksum.cpp:103-115
//   max_k |sum_j B[k][j]| for A-ABFT computed y  proj/src/threshold_aabft.cpp:38-48
//
// One persistent kernel. A task is (group of 32 B rows, 128-column block):
// the warp streams the 32 x 128 tile through its shared-memory slice with
// coalesced loads (the next sub-tile's loads in flight while this one is
// processed) and then lane = row walks its block in column order, producing
// per (block, row): the blocked:128 checksum partials sum_j x and
// sum_j fl(fl(j + 1) x) in the working type (reference order inside the
// block, no FMA), an exactness-preserving partial of the row sum, max / min
// and the order-free trackers of the exactness guard (16-bit formats: those
// order-free statistics go straight into per-row atomic accumulators). The
// warp completing a row group's last block combines the group (lane = row):
// block partials in block order (the blocked:128 combination), the exact row sum -> the
// reference's Neumaier mean (guarded; rows outside the guard rerun the
// reference's loop), var_bound, and publishes the group. One summary warp
// (CTA 0, warp 0) folds the published groups, in row order, into
// BStatsSummary's three sequential FP64 sums and max_k |sum_j B| while the
// rest of the pass is still streaming: the sequential chain (K dependent
// FP64 adds, ~8 cycles each) is the kernel's latency floor, everything else
// overlaps it.
//
// Exact row sums:
//  * BF16 / FP16: plain FP64 sums of the elements; every partial sum is
//    exact when n max|x| < 2^(53 + lsb(min nonzero |x|)) (guard_exact), and
//    then equals both the reference's Neumaier result (row_stats) and its
//    plain sequential sum (aabft_computed_y).
//  * FP32 / FP64: an error-free TwoSum cascade (s, c) per block, merged per
//    row; fl(s + c) equals the reference's fl(sum + comp) unless the exact sum
//    lies within 8 (K u)^2 sum|x| of a rounding midpoint (exact_sum_safe,
//    wide.cu); such rows rerun the reference's loop. The plain sequential
//    FP64 row sum A-ABFT's computed y needs is built on first use
//    (launch_bside_rowsum).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "ptx.cuh"
#include "stats.hpp"
#include "tail.cuh"

namespace vabft_dev {

namespace {

constexpr int kBsWarps = 8;
constexpr int kBsThreads = 32 * kBsWarps;

template <int F>
struct BsT {
    static constexpr bool k16 = F == VABFT_BF16 || F == VABFT_FP16;
    using W = typename std::conditional<F == VABFT_FP64, double, float>::type;  // working type of B r
    using V = typename std::conditional<F == VABFT_FP64, double, float>::type;  // element value type
    // sub-tile: 32 rows x kCols columns, staged as 32-bit (16-bit pairs,
    // FP32) or 64-bit words, row stride padded by one word
    static constexpr int kCols = k16 ? 64 : 32;
    using Word = typename std::conditional<F == VABFT_FP64, double, uint32_t>::type;
    static constexpr int kWords = 32;   // words per staged row
    static constexpr int kStride = 36;  // padded stride: 16-byte aligned rows, conflict-free 16-byte LDS
};

// Per-(block, row) partial arrays, group-major: element (block b, row k) at
// ((k / 32) * nb + b) * 32 + k % 32, so a row group's partials of one array
// are one contiguous span (the combining warp reads them coalesced).
template <int F>
struct BsPart {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    W *p1, *p2;
    double *s, *c;  // exact-sum partials (c: TwoSum tail, wide formats)
    V *sabs, *mx, *mn;
    uint32_t* flags;  // 16-bit: min nonzero magnitude pattern - 1 (0x7FFF: none);
                      // wide: 1 if the block holds a non-finite element
    // 16-bit: per-row accumulators of the order-free statistics, folded by
    // every block task with atomics (the exact row sum under the guard is
    // order-free; max / min / min-nonzero as order-preserving keys), reset
    // by the group combine — so a combine reads only the ordered checksum
    // partials p1 / p2 of its blocks
    double* rsum;
    uint32_t *rmax, *rmin, *rmnz;
};

__host__ __device__ inline size_t bs_index(int64_t b, int64_t k, int64_t nb) {
    return size_t(((k >> 5) * nb + b) * 32 + (k & 31));
}

template <int F>
__host__ __device__ inline BsPart<F> bs_view(void* base, int64_t nb, int64_t kp) {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    const size_t n = size_t(nb) * size_t(kp);
    char* p = static_cast<char*>(base);
    BsPart<F> v;
    v.s = reinterpret_cast<double*>(p); p += 8 * n;
    v.c = reinterpret_cast<double*>(p); p += 8 * n;
    v.p1 = reinterpret_cast<W*>(p); p += sizeof(W) * n;
    v.p2 = reinterpret_cast<W*>(p); p += sizeof(W) * n;
    v.sabs = reinterpret_cast<V*>(p); p += sizeof(V) * n;
    v.mx = reinterpret_cast<V*>(p); p += sizeof(V) * n;
    v.mn = reinterpret_cast<V*>(p); p += sizeof(V) * n;
    v.flags = reinterpret_cast<uint32_t*>(p); p += 4 * n;
    v.rsum = reinterpret_cast<double*>(p); p += 8 * size_t(kp);
    v.rmax = reinterpret_cast<uint32_t*>(p); p += 4 * size_t(kp);
    v.rmin = reinterpret_cast<uint32_t*>(p); p += 4 * size_t(kp);
    v.rmnz = reinterpret_cast<uint32_t*>(p);
    return v;
}

template <int F>
size_t bs_bytes(int64_t nb, int64_t kp) {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    return size_t(nb) * size_t(kp) * (16 + 2 * sizeof(W) + 3 * sizeof(V) + 4) + size_t(kp) * 20 + 256;
}

template <int F>
struct BsJob {
    const typename Elem<F>::T* B;
    int64_t K, N, Kp;
    int64_t ldb;  // row stride of B (elements)
    int nb, ngroups, quantize_br;
    BsideBuffers buf;
    BsPart<F> part;
    unsigned* grp_cnt;   // [ngroups] block arrivals (self-resetting)
    unsigned* grp_flag;  // [ngroups] == this launch's epoch once the group is combined
    unsigned* grp_epoch;  // [2] epoch of the last complete launch, chains-done counter (device state, so a
                          // CUDA-graph replay of the launch is a new epoch too)
    float *split_hi, *split_lo;  // FP32: the transposed TF32 split written by the pass (or null)
    int debug;  // developer ablation (VABFT_BSIDE_DEBUG): 1 no summary chains, 2 also no group combine
    int trace;  // developer timeline (VABFT_BSIDE_TRACE): %globaltimer stamps into g_bs_trace
};

// developer timeline (VABFT_BSIDE_TRACE=1): [0] first CTA start, [1] last
// streaming warp done, [2..4] chain 0..2 done, [5] chain 0 first batch
// start, [6] last group combine done, [7] chain 0's duration in SM cycles
__device__ unsigned long long g_bs_trace[8];
__device__ __forceinline__ unsigned long long bs_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float bs_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double bs_add(double a, double b) { return __dadd_rn(a, b); }

// Load one sub-tile (32 rows x kCols columns from column c) of the row group
// starting at row pointer `base` (row stride N elements) into registers: lane l
// holds word l of every row. Rows at or past `rows` read as zero.
template <int F>
__device__ __forceinline__ void bs_load(const typename Elem<F>::T* __restrict__ base, int64_t N, int64_t ld, int rows,
                                        int64_t c, typename BsT<F>::Word (&v)[32]) {
    using Word = typename BsT<F>::Word;
    const int lane = threadIdx.x & 31;
    if constexpr (BsT<F>::k16) {
        const int64_t col = c + 2 * lane;
        const bool in = col < N;
        if ((ld & 1) == 0 && (N & 1) == 0) {  // rows 4-byte aligned: one 32-bit word per lane and row
            const unsigned int* p = reinterpret_cast<const unsigned int*>(base + col);
            const int64_t st = ld >> 1;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) v[rr] = (rr < rows && in) ? __ldcs(p + rr * st) : 0u;
        } else {  // odd N
            const uint16_t* p = base + col;
            const bool in2 = col + 1 < N;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
                uint32_t w = 0;
                if (rr < rows && in) {
                    w = __ldcs(p + rr * ld);
                    if (in2) w |= uint32_t(__ldcs(p + rr * ld + 1)) << 16;
                }
                v[rr] = w;
            }
        }
    } else {
        const int64_t col = c + lane;
        const bool in = col < N;
        const typename Elem<F>::T* p = base + col;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            Word w = Word(0);
            if (rr < rows && in) {
                if constexpr (F == VABFT_FP32) w = __float_as_uint(__ldcs(p + rr * ld));
                else w = __ldcs(p + rr * ld);
            }
            v[rr] = w;
        }
    }
}

// 16-byte variant for 4-byte words (16-bit pairs, FP32) when the row stride
// is a multiple of 16 bytes and B is 16-byte aligned: lane l holds words
// 4 (l % 8) .. + 3 of row 4 i + l / 8 (8 lanes per 128-byte row segment);
// stored into the staged tile with 16-byte stores.
template <int F>
__device__ __forceinline__ void bs_load_v4(const typename Elem<F>::T* __restrict__ base, int64_t N, int64_t ld, int rows,
                                           int64_t c, uint4 (&v)[8]) {
    constexpr int kPerWord = BsT<F>::k16 ? 2 : 1;  // elements per 32-bit word
    const int lane = threadIdx.x & 31;
    const int64_t col = c + int64_t(4 * kPerWord) * (lane & 7);
    const int rs = lane >> 3;
    const typename Elem<F>::T* p = base + int64_t(rs) * ld + col;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        v[i] = (4 * i + rs < rows && col < N) ? __ldcs(reinterpret_cast<const uint4*>(p + int64_t(4 * i) * ld))
                                              : make_uint4(0u, 0u, 0u, 0u);
}
__device__ __forceinline__ void bs_stage_v4(uint32_t* tile, int stride, const uint4 (&v)[8]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        *reinterpret_cast<uint4*>(tile + (4 * i + (lane >> 3)) * stride + 4 * (lane & 7)) = v[i];
}

// Per-lane accumulators of one (row, block).
template <int F>
struct BsAcc {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    W p1 = W(0), p2 = W(0);
    double s = 0.0, c = 0.0;
    V sabs = V(0), mx = V(-INFINITY), mn = V(INFINITY);
    unsigned long long bad = 0;
    // 16-bit packed trackers: max (NaN-propagating), min, min nonzero magnitude - 1
    uint32_t vmax = F == VABFT_BF16 ? 0xFF80FF80u : 0xFC00FC00u;
    uint32_t vmin = F == VABFT_BF16 ? 0x7F807F80u : 0x7C007C00u;
    uint32_t vmnz = 0x7FFF7FFFu;

    __device__ __forceinline__ void track(uint32_t w) {
        uint32_t d;
        if constexpr (F == VABFT_BF16) {
            asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(w)); vmax = d;
            asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(w)); vmin = d;
        } else {
            asm("max.NaN.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(w)); vmax = d;
            asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(w)); vmin = d;
        }
        // magnitude - 1 per half, zero -> 0x7FFF: (mag + 0x7FFF) mod 2^15
        const uint32_t mz = ((w & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x7FFF7FFFu;
        asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmnz), "r"(mz)); vmnz = d;
    }
    // one 32-bit word = 2 elements (16-bit formats); wt = weight of the first
    __device__ __forceinline__ void pair(uint32_t w, float wt) {
        track(w);
        const float xa = bits16_to_float<F>(uint16_t(w & 0xFFFFu));
        const float xb = bits16_to_float<F>(uint16_t(w >> 16));
        s = __dadd_rn(s, __dadd_rn(double(xa), double(xb)));  // exact under the guard
        p1 = __fadd_rn(__fadd_rn(p1, xa), xb);
        p2 = __fadd_rn(p2, __fmul_rn(wt, xa));
        p2 = __fadd_rn(p2, __fmul_rn(__fadd_rn(wt, 1.0f), xb));
    }
    // a lone 16-bit element (odd N), duplicated into both halves for the trackers
    __device__ __forceinline__ void single(uint32_t h, float wt) {
        track(h | (h << 16));
        const float xa = bits16_to_float<F>(uint16_t(h));
        s = __dadd_rn(s, double(xa));
        p1 = __fadd_rn(p1, xa);
        p2 = __fadd_rn(p2, __fmul_rn(wt, xa));
    }
    // one element of a wide format, weight wt
    __device__ __forceinline__ void elem(V x, float wt) {
        if constexpr (F == VABFT_FP32) {
            bad = max(bad, static_cast<unsigned long long>(__float_as_uint(x) & 0x7FFFFFFFu));
            p1 = __fadd_rn(p1, x);
            p2 = __fadd_rn(p2, __fmul_rn(wt, x));
            sabs = __fadd_rn(sabs, fabsf(x));
        } else {
            bad = max(bad, static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull);
            p1 = __dadd_rn(p1, x);
            p2 = __dadd_rn(p2, __dmul_rn(double(wt), x));
            sabs = __dadd_rn(sabs, fabs(x));
        }
        double t, e;
        two_sum(s, double(x), t, e);
        s = t;
        c = __dadd_rn(c, e);
        mx = mx < x ? x : mx;  // finite rows: fmax / fmin (non-finite rows are rejected)
        mn = x < mn ? x : mn;
    }
};

// One 16-bit sub-tile row: cnt (<= 64) elements from weight w0 (= column + 1).
template <int F>
__device__ __forceinline__ void bs16_sub(BsAcc<F>& a, const uint32_t* trow, int cnt, float w0) {
    if (cnt == 64) {  // 16-byte LDS: 8 elements per load
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4 q4 = reinterpret_cast<const uint4*>(trow)[u];
            const float wu = __fadd_rn(w0, float(8 * u));
            a.pair(q4.x, wu);
            a.pair(q4.y, __fadd_rn(wu, 2.0f));
            a.pair(q4.z, __fadd_rn(wu, 4.0f));
            a.pair(q4.w, __fadd_rn(wu, 6.0f));
        }
    } else {
        const int npair = cnt >> 1;
        for (int jj = 0; jj < npair; ++jj) a.pair(trow[jj], __fadd_rn(w0, float(2 * jj)));
        if (cnt & 1) a.single(trow[npair] & 0xFFFFu, __fadd_rn(w0, float(2 * npair)));
    }
}

// One FP32 sub-tile row (lane = row, cnt columns from column cq, weights
// w0 + j): the A pass's scheme (wide.cu, ApF32) — a plain FP64 sum of the
// sub-tile, exact when 32 max|x| < 2^(53 + lsb(min nonzero |x|)) (else the
// sub-tile is redone as a TwoSum cascade from the staged row), TwoSum-merged
// into the block's (s, c) pair; one F2F + one DADD per element instead of a
// TwoSum per element. With split_hi set, the TF32 split of each element
// (hi = rna(x), lo = rna(x - hi), lo = 0 for non-finite x; tf32_gemm.cu
// split_tf32_t_kernel) is stored transposed: element (k, n) at n K + k, so
// the warp's 32 rows make one coalesced 128-byte segment per column.
template <bool kSplit>
__device__ __forceinline__ void bs_fp32_sub(BsAcc<VABFT_FP32>& a, const uint32_t* trow, int cnt, float w0,
                                            float* hp, int64_t lo_off, int64_t K, bool rowok) {
    float p1 = a.p1, p2 = a.p2, sabs = a.sabs, mx = a.mx, mn = a.mn;
    double ps = 0.0;
    uint32_t amx = 0u, mnz = 0xFFFFFFFFu;
    auto one = [&](float x, float wt) {
        const uint32_t mag = __float_as_uint(x) & 0x7FFFFFFFu;
        amx = max(amx, mag);
        mnz = min(mnz, mag - 1u);  // 0 wraps to the maximum: ignored
        ps = __dadd_rn(ps, double(x));
        p1 = __fadd_rn(p1, x);
        p2 = __fadd_rn(p2, __fmul_rn(wt, x));
        sabs = __fadd_rn(sabs, fabsf(x));
        mx = fmaxf(mx, x);  // finite rows (non-finite ones are flagged and rejected)
        mn = fminf(mn, x);
        if constexpr (kSplit) {
            uint32_t hb, lb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
            const float r = mag < 0x7F800000u ? __fsub_rn(x, __uint_as_float(hb)) : 0.0f;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(r));
            if (rowok) {
                hp[0] = __uint_as_float(hb);
                hp[lo_off] = __uint_as_float(lb);
            }
            hp += K;
        }
    };
    if (cnt == 32) {  // 16-byte LDS
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4 q4 = reinterpret_cast<const uint4*>(trow)[u];
            const float wu = __fadd_rn(w0, float(4 * u));
            one(__uint_as_float(q4.x), wu);
            one(__uint_as_float(q4.y), __fadd_rn(wu, 1.0f));
            one(__uint_as_float(q4.z), __fadd_rn(wu, 2.0f));
            one(__uint_as_float(q4.w), __fadd_rn(wu, 3.0f));
        }
    } else {
        for (int jj = 0; jj < cnt; ++jj) one(__uint_as_float(trow[jj]), __fadd_rn(w0, float(jj)));
    }
    bool exact = true;
    if (mnz != 0xFFFFFFFFu && amx < 0x7F800000u) {
        const int ez = int((mnz + 1u) >> 23);
        const int lsb = (ez == 0 ? 1 : ez) - 127 - 23;
        const int top = int(amx >> 23) - 127 + 1 + 6;  // 32 terms < 2^6 max
        exact = top <= 53 + lsb;
    }
    double c = a.c;
    if (!exact) {  // rare: the sub-tile's exact sum as a TwoSum cascade
        double hs = 0.0, hc = 0.0;
        for (int jj = 0; jj < cnt; ++jj) {
            double tt, ee;
            two_sum(hs, double(__uint_as_float(trow[jj])), tt, ee);
            hs = tt;
            hc = __dadd_rn(hc, ee);
        }
        ps = hs;
        c = __dadd_rn(c, hc);
    }
    double tt, ee;
    two_sum(a.s, ps, tt, ee);
    a.s = tt;
    a.c = __dadd_rn(c, ee);
    a.p1 = p1;
    a.p2 = p2;
    a.sabs = sabs;
    a.mx = mx;
    a.mn = mn;
    a.bad = max(a.bad, static_cast<unsigned long long>(amx));
}

// The block's per-row partials (lane = row) into the group-major arrays.
template <int F>
__device__ __forceinline__ void bs_store(const BsJob<F>& j, const BsAcc<F>& a, int64_t rg, int b) {
    using V = typename BsT<F>::V;
    const int lane = threadIdx.x & 31;
    const int64_t r0 = rg * 32;
    const int rows = int(j.K - r0 < 32 ? j.K - r0 : 32);
    if (lane < rows) {
        const size_t o = bs_index(b, r0 + lane, j.nb);
        V mx = a.mx, mn = a.mn;
        uint32_t flg;
        if constexpr (BsT<F>::k16) {
            flg = min(a.vmnz & 0xFFFFu, a.vmnz >> 16);
            // the NaN-propagating max: a NaN anywhere in the block makes mx NaN
            const float m0 = bits16_to_float<F>(uint16_t(a.vmax & 0xFFFFu));
            const float m1 = bits16_to_float<F>(uint16_t(a.vmax >> 16));
            mx = (isnan(m0) || isnan(m1)) ? __int_as_float(0x7FC00000) : fmaxf(m0, m1);
            mn = fminf(bits16_to_float<F>(uint16_t(a.vmin & 0xFFFFu)), bits16_to_float<F>(uint16_t(a.vmin >> 16)));
        } else {
            flg = F == VABFT_FP32 ? (a.bad >= 0x7F800000ull ? 1u : 0u) : (a.bad >= 0x7FF0000000000000ull ? 1u : 0u);
            j.part.c[o] = a.c;
            j.part.sabs[o] = a.sabs;
        }
        j.part.p1[o] = a.p1;
        j.part.p2[o] = a.p2;
        if constexpr (BsT<F>::k16) {
            const int64_t k = r0 + lane;
            atomicAdd(j.part.rsum + k, a.s);  // exact in any order under the guard (else the row is redone)
            atomicMax(j.part.rmax + k, fkey(mx));
            atomicMin(j.part.rmin + k, fkey(mn));
            atomicMin(j.part.rmnz + k, flg);
        } else {
            j.part.s[o] = a.s;
            j.part.mx[o] = mx;
            j.part.mn[o] = mn;
            j.part.flags[o] = flg;
        }
    }
}

// Process the row group's block b (lane = row).
template <int F, bool kVec>
__device__ __forceinline__ void bs_block(const BsJob<F>& j, typename BsT<F>::Word* tile, int64_t rg, int b) {
    using Word = typename BsT<F>::Word;
    using V = typename BsT<F>::V;
    constexpr int kCols = BsT<F>::kCols;
    constexpr int kStride = BsT<F>::kStride;
    const int lane = threadIdx.x & 31;
    const int64_t K = j.K, N = j.N;
    const int64_t r0 = rg * 32;
    const int rows = int(K - r0 < 32 ? K - r0 : 32);
    const int64_t c0 = int64_t(b) * 128;
    const int bw = int(N - c0 < 128 ? N - c0 : 128);
    const int nsub = (bw + kCols - 1) / kCols;
    const int64_t ld = j.ldb;
    const typename Elem<F>::T* base = j.B + r0 * ld;

    BsAcc<F> a;
    Word v[kVec ? 1 : 32];
    uint4 v4[kVec ? 8 : 1];
    if constexpr (kVec) bs_load_v4<F>(base, N, ld, rows, c0, v4);
    else bs_load<F>(base, N, ld, rows, c0, v);
    __syncwarp();
    if constexpr (kVec) {
        bs_stage_v4(reinterpret_cast<uint32_t*>(tile), kStride, v4);
    } else {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) tile[rr * kStride + lane] = v[rr];
    }
    __syncwarp();
    const Word* trow = tile + lane * kStride;
    for (int q = 0; q < nsub; ++q) {
        const int64_t cq = c0 + int64_t(q) * kCols;
        // the next sub-tile's loads are in flight while this one is processed
        if (q + 1 < nsub) {
            if constexpr (kVec) bs_load_v4<F>(base, N, ld, rows, cq + kCols, v4);
            else bs_load<F>(base, N, ld, rows, cq + kCols, v);
        }
        const int cnt = int(c0 + bw - cq < kCols ? c0 + bw - cq : kCols);  // warp-uniform
        const float w0 = float(cq + 1);  // weight j + 1 of the sub-tile's first element (exact: N <= 2^24)
        if constexpr (BsT<F>::k16) {
            bs16_sub<F>(a, trow, cnt, w0);
        } else if constexpr (F == VABFT_FP32) {
            if (j.split_hi) {
                bs_fp32_sub<true>(a, trow, cnt, w0, j.split_hi + cq * K + (r0 + lane), j.split_lo - j.split_hi,
                                         K, lane < rows);
            } else {
                bs_fp32_sub<false>(a, trow, cnt, w0, nullptr, 0, K, false);
            }
        } else {
            if (cnt == kCols) {  // 16-byte LDS
                {
#pragma unroll 4
                    for (int u = 0; u < kCols / 2; ++u) {
                        const double2 q2 = reinterpret_cast<const double2*>(trow)[u];
                        const float wu = __fadd_rn(w0, float(2 * u));
                        a.elem(q2.x, wu);
                        a.elem(q2.y, __fadd_rn(wu, 1.0f));
                    }
                }
            } else {
                for (int jj = 0; jj < cnt; ++jj) a.elem(trow[jj], __fadd_rn(w0, float(jj)));
            }
        }
        if (q + 1 < nsub) {
            __syncwarp();
            if constexpr (kVec) {
                bs_stage_v4(reinterpret_cast<uint32_t*>(tile), kStride, v4);
            } else {
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) tile[rr * kStride + lane] = v[rr];
            }
            __syncwarp();
        }
    }
    bs_store<F>(j, a, rg, b);
}

// Combine a finished row group (lane = row) and publish it.
template <int F>
__device__ __forceinline__ void bs_combine(const BsJob<F>& j, int64_t rg, unsigned epoch) {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    const int lane = threadIdx.x & 31;
    const int64_t k = rg * 32 + lane;
    const int nb = j.nb;
    W t1 = W(0), t2 = W(0);
    double s = 0.0, c = 0.0, sabs = 0.0;
    V mx = V(-INFINITY), mn = V(INFINITY);
    uint32_t mz = 0x7FFFu, bad = 0u;
    const size_t o0 = bs_index(0, k, nb);
    if constexpr (BsT<F>::k16) {
        // the ordered checksum partials, 16 blocks of loads in flight per
        // round; the order-free statistics from the per-row accumulators
        // (loaded alongside), reset for the next launch
        if (k < j.K) {
            s = __ldcg(j.part.rsum + k);
            mx = fkey_decode(__ldcg(j.part.rmax + k));
            mn = fkey_decode(__ldcg(j.part.rmin + k));
            mz = __ldcg(j.part.rmnz + k);
        }
        for (int b0 = 0; b0 < nb; b0 += 16) {
            W v1[16], v2[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const bool in = b0 + q < nb;
                v1[q] = in ? __ldcg(j.part.p1 + o0 + size_t(b0 + q) * 32) : W(0);
                v2[q] = in ? __ldcg(j.part.p2 + o0 + size_t(b0 + q) * 32) : W(0);
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                if (b0 + q < nb) {  // block order: the blocked:128 combination
                    t1 = bs_add(t1, v1[q]);
                    t2 = bs_add(t2, v2[q]);
                }
            }
        }
        if (k < j.K) {
            j.part.rsum[k] = 0.0;
            j.part.rmax[k] = 0u;
            j.part.rmin[k] = 0xFFFFFFFFu;
            j.part.rmnz[k] = 0xFFFFFFFFu;
        }
    }
#pragma unroll 8
    for (int b = 0; b < (BsT<F>::k16 ? 0 : nb); ++b) {  // block order: the blocked:128 combination
        const size_t o = o0 + size_t(b) * 32;
        t1 = bs_add(t1, __ldcg(j.part.p1 + o));
        t2 = bs_add(t2, __ldcg(j.part.p2 + o));
        const V bx = __ldcg(j.part.mx + o), bn = __ldcg(j.part.mn + o);
        mx = (isnan(bx) || mx < bx) ? bx : mx;
        mn = bn < mn ? bn : mn;
        const uint32_t f = __ldcg(j.part.flags + o);
        if constexpr (BsT<F>::k16) {
            s = __dadd_rn(s, __ldcg(j.part.s + o));
            mz = min(mz, f);
        } else {
            bad |= f;
            double t, e;
            two_sum(s, __ldcg(j.part.s + o), t, e);
            s = t;
            c = __dadd_rn(__dadd_rn(c, __ldcg(j.part.c + o)), e);
            sabs = __dadd_rn(sabs, double(__ldcg(j.part.sabs + o)));
        }
    }
    bool fast = false, finite = true;
    Neu n;
    double plain = 0.0;
    if (k < j.K) {
        if constexpr (BsT<F>::k16) {
            const float amax = fmaxf(fabsf(mx), fabsf(mn));
            finite = !isnan(mx) && isfinite(amax);
            fast = finite && guard_exact<F>(amax, mz, j.N);
            n.s = s;
            plain = s;
        } else {
            finite = bad == 0u;
            double hi = 0.0;
            // sabs was summed in the element type: 1 % slack keeps it an upper bound
            fast = finite && exact_sum_safe(s, c, __dmul_rn(sabs, 1.01), j.N, &hi);
            n.s = hi;
        }
        // nonzero: this launch saw NaN / Inf
        if (!finite) atomicMax(reinterpret_cast<unsigned*>(j.buf.nonfinite), epoch);
    }
    // rows outside the exactness guard: the reference's Neumaier sum by the
    // whole warp (warp_neumaier_row: parallel error-free sum + midpoint check,
    // the sequential loop only next to a rounding midpoint)
    unsigned slow = __ballot_sync(0xffffffffu, k < j.K && finite && !fast);
    while (slow) {
        const int l = __ffs(slow) - 1;
        slow &= slow - 1;
        double pl;
        const double hs = warp_neumaier_row<F>(j.B + (rg * 32 + l) * j.ldb, j.N, BsT<F>::k16 ? &pl : nullptr);
        if (lane == l) {
            n = Neu{};
            n.s = hs;
            plain = pl;
        }
    }
    if (k < j.K) {
        double m, v;
        stats_finish(n, double(mx), double(mn), j.N, &m, &v);
        j.buf.mean[k] = m;
        j.buf.vb[k] = v;
        if constexpr (BsT<F>::k16) {
            if (j.quantize_br) {
                t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
                t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
            }
            j.buf.br1[k] = t1;
            j.buf.br2[k] = t2;
            j.buf.rowsum_abs[k] = fabs(plain);
        } else {
            j.buf.br1[k] = float(t1);
            j.buf.br2[k] = float(t2);
            if (j.buf.brd1) {
                j.buf.brd1[k] = double(t1);
                j.buf.brd2[k] = double(t2);
            }
        }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile unsigned*>(j.grp_flag + rg) = epoch;
}

// Summary: BStatsSummary::from's three sequential FP64 sums over k in row
// order (threshold_vabft.cpp:15-26), one chain per warp (warps 0..2 of CTA 0,
// on different schedulers), and max_k |sum_j B| (16-bit formats; order-free,
// so warp 3 folds it lane-parallel; the wide formats' plain row sums come from
// launch_bside_rowsum). The published row groups are consumed in batches of
// 256 rows: while lane 0 runs the chain over batch i out of shared memory
// (16-byte LDS issued ahead of the adds), the warp's coalesced loads of batch
// i + 1 are in flight, landing in the other half of the warp's double buffer.
// The chains then run at about one FP64 add latency (~8 cycles) per element:
// the kernel's floor, K x 8 cycles. (Measured: a 16-value register prefetch
// left every batch waiting ~1000 cycles on L2; a data-dependent branch or an
// fmax in the chain doubled or quadrupled its cost.)
template <int F, int kWhich, int kBatch = 256>
__device__ void bs_summary(const BsJob<F>& j, double* buf2 /* 2 x kBatch doubles */, unsigned epoch) {
    constexpr int which = kWhich;  // compile-time: no branch inside the chain
    constexpr int kPer = kBatch / 32;
    const int lane = threadIdx.x & 31;
    const double* src = which == 2 ? j.buf.vb : which == 3 ? j.buf.rowsum_abs : j.buf.mean;
    const int64_t K = j.K;
    int64_t ready = j.debug >= 3 ? j.ngroups : 0;  // groups [0, ready) are published (debug >= 3: chains alone)
    auto published = [&](int64_t kend) {  // rows [0, kend) published?
        const int64_t need = (kend + 31) / 32;
        while (ready < need) {
            const int64_t g = ready + lane;
            const bool ok = g >= j.ngroups || *reinterpret_cast<volatile const unsigned*>(j.grp_flag + g) == epoch;
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            const int run = bal == 0xffffffffu ? 32 : __ffs(~bal) - 1;
            if (run == 0) return false;
            // no fence per poll (measured to cost more than the chain): the
            // producer fenced the group's values before its flag, and the
            // value loads below are L2 (.cg) loads issued after the flag was
            // seen (control dependency)
            ready += run;
        }
        return true;
    };
    auto fetch = [&](int64_t k0, double (&v)[kPer]) {
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int64_t k = k0 + e * 32 + lane;
            v[e] = k < K ? __ldcg(src + k) : 0.0;
        }
    };
    double acc = 0.0, v[kPer];
    if constexpr (which == 3) {  // max_k |sum_j B|: order-free, lane-parallel
        for (int64_t k0 = 0; k0 < K; k0 += 2 * kBatch) {  // two batches of loads in flight
            const int64_t kend = k0 + 2 * kBatch < K ? k0 + 2 * kBatch : K;
            while (!published(kend)) __nanosleep(64);
            double w[kPer];
            fetch(k0, v);
            fetch(k0 + kBatch, w);
#pragma unroll
            for (int e = 0; e < kPer; ++e) acc = fmax(acc, fmax(v[e], w[e]));
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) acc = fmax(acc, __shfl_xor_sync(0xffffffffu, acc, m));
        if (lane == 0) j.buf.summary[3] = acc;
        return;  // (warp 3 does not take part in the epoch hand-over)
    }
    // Batches land in the warp's double buffer by cp.async (LDGSTS, .cg: L2),
    // issued one batch ahead: fire-and-forget, so they stay in flight during
    // the chain. (Measured: register fetches were sunk below the lane-0 chain
    // by the compiler, every batch then waited on L2 — 12.7 cycles per
    // element instead of ~8.)
    auto fetch_async = [&](int64_t k0, double* dst) {
#pragma unroll
        for (int ch = lane; ch < kBatch / 2; ch += 32) {  // 16-byte chunks, zero-filled past K
            const int64_t k = k0 + 2 * ch;
            const int nv = K - k >= 2 ? 16 : (K - k == 1 ? 8 : 0);
            cp_async16n(smem_u32(dst + 2 * ch), nv ? src + k : src, nv);
        }
        cp_async_commit();
    };
    while (!published(kBatch < K ? kBatch : K)) __nanosleep(64);
    if (j.trace && which == 0 && lane == 0) {
        atomicMax(&g_bs_trace[5], bs_now());
        g_bs_trace[7] = static_cast<unsigned long long>(clock64());  // chain 0's start, SM cycles
    }
    fetch_async(0, buf2);
    int cur = 0;
    for (int64_t k0 = 0; k0 < K; k0 += kBatch) {
        const int64_t k1 = k0 + kBatch;
        const bool more = k1 < K;
        const int64_t kend = k1 + kBatch < K ? k1 + kBatch : K;
        cp_async_wait<0>();  // batch k0 landed (this lane's chunks) ...
        __syncwarp();        // ... and every lane's
        const bool pre = more && published(kend);
        if (pre) fetch_async(k1, buf2 + (cur ^ 1) * kBatch);  // in flight during the chain below
        if (lane == 0) {
            const double* x = buf2 + cur * kBatch;
            const int cnt = int(K - k0 < kBatch ? K - k0 : kBatch);
            if (cnt == kBatch) {
                // 32 values per round loaded into registers before the adds,
                // so no add waits on a shared-memory load
#pragma unroll 1
                for (int e0 = 0; e0 < kBatch; e0 += 32) {  // (unrolled: no faster, and the code size
                                                           // cost the streaming warps i-cache misses)
                    double2 q[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) q[i] = reinterpret_cast<const double2*>(x + e0)[i];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        if constexpr (which == 0) acc = __dadd_rn(__dadd_rn(acc, fabs(q[i].x)), fabs(q[i].y));
                        else if constexpr (which == 1)
                            acc = __dadd_rn(__dadd_rn(acc, __dmul_rn(q[i].x, q[i].x)), __dmul_rn(q[i].y, q[i].y));
                        else acc = __dadd_rn(__dadd_rn(acc, q[i].x), q[i].y);
                    }
                }
            } else {
                for (int e = 0; e < cnt; ++e) {
                    const double xe = x[e];
                    if constexpr (which == 0) acc = __dadd_rn(acc, fabs(xe));
                    else if constexpr (which == 1) acc = __dadd_rn(acc, __dmul_rn(xe, xe));
                    else acc = __dadd_rn(acc, xe);
                }
            }
        }
        __syncwarp();  // the buffer half is refilled next round
        if (more) {
            if (!pre) {
                while (!published(kend)) __nanosleep(64);
                fetch_async(k1, buf2 + (cur ^ 1) * kBatch);
            }
            cur ^= 1;
        }
    }
    if (j.trace && lane == 0) atomicMax(&g_bs_trace[2 + which], bs_now());
    if (j.trace && which == 0 && lane == 0)
        g_bs_trace[7] = static_cast<unsigned long long>(clock64()) - g_bs_trace[7];  // chain 0's SM cycles
    if (lane == 0) {
        j.buf.summary[which] = acc;
        // the last of the three chains (every flag read) closes the epoch
        __threadfence();
        if (atomicAdd(j.grp_epoch + 1, 1u) == 2u) {
            j.grp_epoch[1] = 0u;
            __threadfence();
            j.grp_epoch[0] = epoch;
        }
    }
}

template <int F>
constexpr size_t bs_smem() {
    return size_t(kBsWarps) * 32 * BsT<F>::kStride * sizeof(typename BsT<F>::Word);
}

template <int F, bool kVec>
__global__ void __launch_bounds__(kBsThreads, F == VABFT_FP64 ? 1 : 2) bside_kernel(const __grid_constant__ BsJob<F> j) {
    using Word = typename BsT<F>::Word;
    constexpr int kStride = BsT<F>::kStride;
    constexpr int kChains = BsT<F>::k16 ? 4 : 3;  // wide formats: max_k |sum_j B| on demand
    extern __shared__ __align__(16) uint8_t bs_smem_raw[];
    Word* tiles = reinterpret_cast<Word*>(bs_smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned epoch = *reinterpret_cast<volatile const unsigned*>(j.grp_epoch) + 1u;
    if (j.trace && threadIdx.x == 0) atomicMin(&g_bs_trace[0], bs_now());
    if (blockIdx.x == 0 && warp < kChains) {  // the warp's tile slice is its double buffer (>= 2 KiB)
        double* b2 = reinterpret_cast<double*>(tiles + size_t(warp) * 32 * kStride);
        if (j.debug == 0 || j.debug == 3 || j.debug == 4 + warp) {
            switch (warp) {
                case 0: bs_summary<F, 0>(j, b2, epoch); break;
                case 1: bs_summary<F, 1>(j, b2, epoch); break;
                case 2: bs_summary<F, 2>(j, b2, epoch); break;
                default: bs_summary<F, 3>(j, b2, epoch); break;
            }
        }
        return;
    }
    // zero padding of the B r vectors (the A-side readers take whole 128-k blocks)
    if (blockIdx.x == 0 && warp == kChains) {
        const int64_t kpad = (j.K + 127) / 128 * 128;
        for (int64_t k = j.K + lane; k < kpad; k += 32) {
            j.buf.br1[k] = 0.0f;
            j.buf.br2[k] = 0.0f;
        }
    }
    if (j.debug >= 3) return;  // chains alone (developer timing)
    Word* tile = tiles + size_t(warp) * 32 * kStride;
    const int64_t tw = int64_t(blockIdx.x) * kBsWarps + warp - kChains;
    const int64_t nt = int64_t(gridDim.x) * kBsWarps - kChains;
    const int nb = j.nb;
    const int64_t tasks = int64_t(j.ngroups) * nb;
    for (int64_t t = tw; t < tasks; t += nt) {
        const int64_t rg = t / nb;
        const int b = int(t - rg * nb);
        bs_block<F, kVec>(j, tile, rg, b);
        // arrival: every lane's partial stores before lane 0's release RMW;
        // the last arriver reads the partials through L2 after a fence
        __syncwarp();
        unsigned old = 0;
        if (lane == 0) old = atom_add_release_gpu(j.grp_cnt + rg, 1u);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == unsigned(nb) - 1u && j.debug < 2) {
            __threadfence();
            if (lane == 0) j.grp_cnt[rg] = 0u;  // ready for the next launch
            bs_combine<F>(j, rg, epoch);
            if (j.trace && lane == 0) atomicMax(&g_bs_trace[6], bs_now());
        }
    }
    if (j.trace && lane == 0) atomicMax(&g_bs_trace[1], bs_now());
}

// The plain sequential FP64 row sum (threshold_aabft.cpp:42-46) of every B
// row, for A-ABFT computed y on the wide formats: a warp per row stages the
// row through shared memory and lane 0 runs the chain. max_k |sum| is folded
// with an order-free atomic max.
template <int F>
__global__ void __launch_bounds__(128) bside_rowsum_kernel(const typename Elem<F>::T* __restrict__ B, int64_t K,
                                                           int64_t N, int64_t ld, double* rowsum_abs, double* summary) {
    using T = typename Elem<F>::T;
    __shared__ T stage[4][256];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = int64_t(blockIdx.x) * 4 + w;
    if (k >= K) return;
    const T* row = B + k * ld;
    double s = 0.0;
    for (int64_t j0 = 0; j0 < N; j0 += 256) {
        const int cnt = int(N - j0 < 256 ? N - j0 : 256);
        __syncwarp();
        for (int q = lane; q < cnt; q += 32) stage[w][q] = row[j0 + q];
        __syncwarp();
        if (lane == 0)
            for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, double(stage[w][q]));
    }
    if (lane == 0) {
        rowsum_abs[k] = fabs(s);
        atomic_max_nonneg(summary + 3, fabs(s));
    }
}

void bs_trace_report(int trc, int F, int64_t K, int64_t N, cudaStream_t s) {
    if (!trc) return;
    unsigned long long t[8];
    check_cuda(cudaMemcpyFromSymbolAsync(t, g_bs_trace, sizeof(t), 0, cudaMemcpyDeviceToHost, s), "trace");
    check_cuda(cudaStreamSynchronize(s), "trace");
    auto us = [&](int i) { return t[i] ? double(t[i] - t[0]) * 1e-3 : -1.0; };
    const double c0us = t[2] && t[5] ? double(t[2] - t[5]) * 1e-3 : 0.0;
    std::fprintf(stderr, "bside trace F=%d K=%lld N=%lld: pass %.2f combine %.2f chain0-start %.2f chains %.2f %.2f %.2f us"
                 " (chain 0: %llu SM cycles, %.0f MHz)\n", F, (long long)K, (long long)N, us(1), us(6), us(5), us(2), us(3),
                 us(4), t[7], c0us > 0 ? double(t[7]) / c0us : 0.0);
}

template <int F>
void launch_bs(int64_t K, int64_t N, int64_t ld, const void* B, int quantize_br, BsideBuffers& buf, cudaStream_t s) {
    BsJob<F> j;
    j.ldb = ld;
    j.B = static_cast<const typename Elem<F>::T*>(B);
    j.K = K;
    j.N = N;
    j.ngroups = int((K + 31) / 32);
    j.Kp = int64_t(j.ngroups) * 32;
    j.nb = int((N + 127) / 128);
    j.quantize_br = quantize_br;
    j.buf = buf;
    j.part = bs_view<F>(buf.work, j.nb, j.Kp);
    j.split_hi = F == VABFT_FP32 ? buf.split_hi : nullptr;
    j.split_lo = F == VABFT_FP32 ? buf.split_lo : nullptr;
    j.grp_cnt = buf.groups;
    j.grp_flag = buf.groups + j.ngroups;
    static const int dbg = [] {
        const char* e = std::getenv("VABFT_BSIDE_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    j.debug = dbg;
    static const int trc = [] {
        const char* e = std::getenv("VABFT_BSIDE_TRACE");
        return e ? std::atoi(e) : 0;
    }();
    j.trace = trc;
    if (trc) {
        const unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
        check_cuda(cudaMemcpyToSymbolAsync(g_bs_trace, init, sizeof(init), 0, cudaMemcpyHostToDevice, s), "trace");
    }
    j.grp_epoch = buf.groups + 2 * j.ngroups;
    constexpr size_t smem = bs_smem<F>();
    // 16-byte loads when rows are 16-byte multiples and B is aligned (4-byte words only)
    const bool vec = F != VABFT_FP64 && (ld * int64_t(sizeof(typename Elem<F>::T))) % 16 == 0 &&
                     (N * int64_t(sizeof(typename Elem<F>::T))) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(B) % 16 == 0;
    auto kern = vec ? bside_kernel<F, F != VABFT_FP64> : bside_kernel<F, false>;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), int(smem));
    const int per_sm = cached_occupancy(reinterpret_cast<const void*>(kern), kBsThreads, int(smem));
    const int64_t tasks = int64_t(j.ngroups) * j.nb;
    const int64_t want = (tasks + kBsWarps - 1) / kBsWarps + 1;
    static const int per_sm_env = [] {  // developer override (VABFT_BSIDE_PERSM)
        const char* e = std::getenv("VABFT_BSIDE_PERSM");
        return e ? std::atoi(e) : 0;
    }();
    const int use_per_sm = per_sm_env > 0 ? std::min(per_sm_env, std::max(per_sm, 1)) : std::max(per_sm, 1);
    const int grid = int(std::min<int64_t>(int64_t(sm_count()) * use_per_sm, want));
    kern<<<grid, kBsThreads, smem, s>>>(j);
    check_cuda(cudaGetLastError(), "bside launch");
    bs_trace_report(trc, F, K, N, s);
}

}  // namespace

size_t bside_work_bytes(int fmt, int64_t K, int64_t N) {
    const int64_t kp = (K + 31) / 32 * 32, nb = (N + 127) / 128;
    switch (fmt) {
        case VABFT_BF16: return bs_bytes<VABFT_BF16>(nb, kp);
        case VABFT_FP16: return bs_bytes<VABFT_FP16>(nb, kp);
        case VABFT_FP32: return bs_bytes<VABFT_FP32>(nb, kp);
        default: return bs_bytes<VABFT_FP64>(nb, kp);
    }
}

size_t bside_group_words(int64_t K) { return size_t(2 * ((K + 31) / 32) + 2); }

void bside_init_work(int fmt, int64_t K, int64_t N, void* work, cudaStream_t s) {
    if (fmt != VABFT_BF16 && fmt != VABFT_FP16) return;
    const int64_t kp = (K + 31) / 32 * 32, nb = (N + 127) / 128;
    const BsPart<VABFT_BF16> v = bs_view<VABFT_BF16>(work, nb, kp);  // same layout for FP16
    // per-row accumulators at their identities: sum 0 and max key 0, then min keys all ones
    check_cuda(cudaMemsetAsync(v.rsum, 0, size_t(kp) * 12, s), "memset");
    check_cuda(cudaMemsetAsync(v.rmin, 0xFF, size_t(kp) * 8, s), "memset");
}

int64_t br_storage_floats(int64_t K) { return ((K + 127) / 128) * 128; }

void launch_bside(int fmt, int64_t K, int64_t N, const void* B, int quantize_br, BsideBuffers& buf,
                  cudaStream_t s, int64_t ld) {
    if (ld == 0) ld = N;
    if (ld < N) fail(VABFT_INVALID_ARGUMENT, "launch_bside: leading dimension below N");
    if (!buf.work || !buf.groups) fail(VABFT_LOGIC_ERROR, "launch_bside: workspace missing");
    if (N > (int64_t(1) << 24)) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: weights exceed exact range");
    switch (fmt) {
        case VABFT_BF16: launch_bs<VABFT_BF16>(K, N, ld, B, quantize_br, buf, s); break;
        case VABFT_FP16: launch_bs<VABFT_FP16>(K, N, ld, B, quantize_br, buf, s); break;
        case VABFT_FP32: launch_bs<VABFT_FP32>(K, N, ld, B, 0, buf, s); break;
        case VABFT_FP64: launch_bs<VABFT_FP64>(K, N, ld, B, 0, buf, s); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
}

void launch_bside_rowsum(int fmt, int64_t K, int64_t N, const void* B, BsideBuffers& buf, cudaStream_t s,
                         int64_t ld) {
    if (ld == 0) ld = N;
    check_cuda(cudaMemsetAsync(buf.summary + 3, 0, sizeof(double), s), "memset");
    const unsigned grid = unsigned((K + 3) / 4);
    switch (fmt) {
        case VABFT_BF16: bside_rowsum_kernel<VABFT_BF16><<<grid, 128, 0, s>>>(static_cast<const uint16_t*>(B), K, N, ld, buf.rowsum_abs, buf.summary); break;
        case VABFT_FP16: bside_rowsum_kernel<VABFT_FP16><<<grid, 128, 0, s>>>(static_cast<const uint16_t*>(B), K, N, ld, buf.rowsum_abs, buf.summary); break;
        case VABFT_FP32: bside_rowsum_kernel<VABFT_FP32><<<grid, 128, 0, s>>>(static_cast<const float*>(B), K, N, ld, buf.rowsum_abs, buf.summary); break;
        case VABFT_FP64: bside_rowsum_kernel<VABFT_FP64><<<grid, 128, 0, s>>>(static_cast<const double*>(B), K, N, ld, buf.rowsum_abs, buf.summary); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
    check_cuda(cudaGetLastError(), "bside rowsum launch");
}

}  // namespace vabft_dev
