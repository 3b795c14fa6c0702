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
// and the order-free trackers of the exactness guard. The warp completing a
// row group's last block combines the group (lane = row): block partials in
// block order (the blocked:128 combination), the exact row sum -> the
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
    static constexpr int kWords = 32;  // words per staged row
};

// Per-(block, row) partial arrays, each [nb][Kp].
template <int F>
struct BsPart {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    W *p1, *p2;
    double *s, *c;  // exact-sum partials (c: TwoSum tail, wide formats)
    V *sabs, *mx, *mn;
    uint32_t* flags;  // 16-bit: (max magnitude pattern << 16) | (min nonzero magnitude pattern - 1);
                      // wide: 1 if the block holds a non-finite element
};

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
    v.flags = reinterpret_cast<uint32_t*>(p);
    return v;
}

template <int F>
size_t bs_bytes(int64_t nb, int64_t kp) {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    return size_t(nb) * size_t(kp) * (16 + 2 * sizeof(W) + 3 * sizeof(V) + 4) + 256;
}

template <int F>
struct BsJob {
    const typename Elem<F>::T* B;
    int64_t K, N, Kp;
    int nb, ngroups, quantize_br;
    BsideBuffers buf;
    BsPart<F> part;
    unsigned* grp_cnt;   // [ngroups] block arrivals (self-resetting)
    unsigned* grp_flag;  // [ngroups] == epoch once the group is combined
    unsigned epoch;
};

__device__ __forceinline__ float bs_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double bs_add(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ void two_sum_bs(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// exact_sum_safe (wide.cu): hi = fl(s + c) equals the reference's Neumaier
// fl(sum + comp) unless the exact sum is within 8 (K u)^2 sum|x| of a midpoint
__device__ __forceinline__ bool bs_exact_safe(double s, double c, double sabs, int64_t K, double* hi_out) {
    double hi, lo;
    two_sum_bs(s, c, hi, lo);
    const double ku = double(K) * 1.1102230246251565e-16;
    const double margin = 8.0 * ku * ku * sabs * 1.01;  // sabs summed in the element type: 1 % slack
    if (!(isfinite(hi) && isfinite(lo) && isfinite(margin))) return false;
    const double nb = nextafter(hi, (lo > 0.0) ? INFINITY : -INFINITY);
    if (!(fabs(lo) + margin < fabs(__dsub_rn(nb, hi)) * 0.5)) return false;
    *hi_out = hi;
    return true;
}

// Load one sub-tile (32 rows x kCols columns starting at column c) of the
// row group into registers: lane l holds word l of every row.
template <int F>
__device__ __forceinline__ void bs_load(const BsJob<F>& j, int64_t r0, int64_t c, typename BsT<F>::Word (&v)[32]) {
    using Word = typename BsT<F>::Word;
    const int lane = threadIdx.x & 31;
    if constexpr (BsT<F>::k16) {
        const int64_t col = c + 2 * lane;
        const bool even = (j.N & 1) == 0;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            const int64_t r = r0 + rr;
            uint32_t w = 0;
            if (r < j.K && col < j.N) {
                const uint16_t* p = j.B + r * j.N + col;
                if (even) {
                    w = __ldcs(reinterpret_cast<const unsigned int*>(p));
                } else {  // odd N: rows are not 4-byte aligned
                    w = __ldcs(p);
                    if (col + 1 < j.N) w |= uint32_t(__ldcs(p + 1)) << 16;
                }
            }
            v[rr] = w;
        }
    } else {
        const int64_t col = c + lane;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            const int64_t r = r0 + rr;
            Word w = Word(0);
            if (r < j.K && col < j.N) {
                if constexpr (F == VABFT_FP32) w = __float_as_uint(__ldcs(j.B + r * j.N + col));
                else w = __ldcs(j.B + r * j.N + col);
            }
            v[rr] = w;
        }
    }
}

// Process the row group's block b (lane = row).
template <int F>
__device__ __forceinline__ void bs_block(const BsJob<F>& j, typename BsT<F>::Word* tile, int64_t rg, int b) {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    using Word = typename BsT<F>::Word;
    constexpr int kCols = BsT<F>::kCols;
    constexpr int kStride = BsT<F>::kWords + 1;
    const int lane = threadIdx.x & 31;
    const int64_t r0 = rg * 32, row = r0 + lane;
    const int64_t c0 = int64_t(b) * 128;
    const int bw = int(j.N - c0 < 128 ? j.N - c0 : 128);
    const int nsub = (bw + kCols - 1) / kCols;

    W p1 = W(0), p2 = W(0);
    double s = 0.0, cc = 0.0;
    V sabs = V(0), mx = V(-INFINITY), mn = V(INFINITY);
    uint32_t flg = 0;
    // 16-bit packed trackers
    uint32_t vmax = F == VABFT_BF16 ? 0xFF80FF80u : 0xFC00FC00u;
    uint32_t vmin = F == VABFT_BF16 ? 0x7F807F80u : 0x7C007C00u;
    uint32_t vmag = 0u, vmnz = 0x7FFF7FFFu;
    unsigned long long bad = 0;

    Word cur[32], nxt[32];
    bs_load<F>(j, r0, c0, cur);
    for (int q = 0; q < nsub; ++q) {
        const int64_t cq = c0 + int64_t(q) * kCols;
        if (q + 1 < nsub) bs_load<F>(j, r0, cq + kCols, nxt);
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) tile[rr * kStride + lane] = cur[rr];
        __syncwarp();
        const int cnt = int(c0 + bw - cq < kCols ? c0 + bw - cq : kCols);  // warp-uniform
        const Word* trow = tile + lane * kStride;
        float wj = float(cq + 1);  // weight of the next element, exact (N <= 2^24)
        if constexpr (BsT<F>::k16) {
            const int npair = cnt >> 1;
#pragma unroll 4
            for (int jj = 0; jj < npair; ++jj) {
                const uint32_t w = trow[jj];
                uint32_t d;
                if constexpr (F == VABFT_BF16) {
                    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(w)); vmax = d;
                    asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(w)); vmin = d;
                } else {
                    asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(w)); vmax = d;
                    asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(w)); vmin = d;
                }
                const uint32_t mag = w & 0x7FFF7FFFu;
                asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmag), "r"(mag)); vmag = d;
                asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmnz), "r"(((mag | 0x80008000u) - 0x00010001u) & 0x7FFF7FFFu));
                vmnz = d;
                const float xa = bits16_to_float<F>(uint16_t(w & 0xFFFFu));
                const float xb = bits16_to_float<F>(uint16_t(w >> 16));
                s = __dadd_rn(s, __dadd_rn(double(xa), double(xb)));  // exact under the guard
                p1 = __fadd_rn(p1, xa);
                p2 = __fadd_rn(p2, __fmul_rn(wj, xa));
                wj = __fadd_rn(wj, 1.0f);
                p1 = __fadd_rn(p1, xb);
                p2 = __fadd_rn(p2, __fmul_rn(wj, xb));
                wj = __fadd_rn(wj, 1.0f);
            }
            if (cnt & 1) {  // odd N: the row's last element
                const uint16_t h = uint16_t(trow[npair] & 0xFFFFu);
                const uint32_t hw = uint32_t(h) | (uint32_t(h) << 16);  // duplicate: neutral for the trackers
                uint32_t d;
                if constexpr (F == VABFT_BF16) {
                    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(hw)); vmax = d;
                    asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(hw)); vmin = d;
                } else {
                    asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmax), "r"(hw)); vmax = d;
                    asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(vmin), "r"(hw)); vmin = d;
                }
                const uint32_t mag = hw & 0x7FFF7FFFu;
                asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmag), "r"(mag)); vmag = d;
                asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(vmnz), "r"(((mag | 0x80008000u) - 0x00010001u) & 0x7FFF7FFFu));
                vmnz = d;
                const float xa = bits16_to_float<F>(h);
                s = __dadd_rn(s, double(xa));
                p1 = __fadd_rn(p1, xa);
                p2 = __fadd_rn(p2, __fmul_rn(wj, xa));
            }
        } else {
#pragma unroll 4
            for (int jj = 0; jj < cnt; ++jj) {
                V x;
                if constexpr (F == VABFT_FP32) x = __uint_as_float(trow[jj]);
                else x = trow[jj];
                const double xd = double(x);
                if constexpr (F == VABFT_FP32) {
                    bad = max(bad, static_cast<unsigned long long>(__float_as_uint(x) & 0x7FFFFFFFu));
                    p1 = __fadd_rn(p1, x);
                    p2 = __fadd_rn(p2, __fmul_rn(wj, x));
                    sabs = __fadd_rn(sabs, fabsf(x));
                } else {
                    bad = max(bad, static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull);
                    p1 = __dadd_rn(p1, x);
                    p2 = __dadd_rn(p2, __dmul_rn(double(wj), x));
                    sabs = __dadd_rn(sabs, fabs(x));
                }
                wj = __fadd_rn(wj, 1.0f);
                double t, e;
                two_sum_bs(s, xd, t, e);
                s = t;
                cc = __dadd_rn(cc, e);
                mx = mx < x ? x : mx;  // finite rows: fmax / fmin (non-finite rows are rejected)
                mn = x < mn ? x : mn;
            }
        }
        if (q + 1 < nsub) {
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) cur[rr] = nxt[rr];
        }
    }
    if (row < j.K) {
        const size_t o = size_t(b) * size_t(j.Kp) + size_t(row);
        if constexpr (BsT<F>::k16) {
            const uint32_t mg = max(vmag & 0xFFFFu, vmag >> 16);
            const uint32_t mz = min(vmnz & 0xFFFFu, vmnz >> 16);
            flg = (mg << 16) | mz;
            mx = fmaxf(bits16_to_float<F>(uint16_t(vmax & 0xFFFFu)), bits16_to_float<F>(uint16_t(vmax >> 16)));
            mn = fminf(bits16_to_float<F>(uint16_t(vmin & 0xFFFFu)), bits16_to_float<F>(uint16_t(vmin >> 16)));
        } else {
            flg = F == VABFT_FP32 ? (bad >= 0x7F800000ull ? 1u : 0u) : (bad >= 0x7FF0000000000000ull ? 1u : 0u);
            j.part.c[o] = cc;
            j.part.sabs[o] = sabs;
        }
        j.part.p1[o] = p1;
        j.part.p2[o] = p2;
        j.part.s[o] = s;
        j.part.mx[o] = mx;
        j.part.mn[o] = mn;
        j.part.flags[o] = flg;
    }
}

// Combine a finished row group (lane = row) and publish it.
template <int F>
__device__ __forceinline__ void bs_combine(const BsJob<F>& j, int64_t rg) {
    using W = typename BsT<F>::W;
    using V = typename BsT<F>::V;
    const int lane = threadIdx.x & 31;
    const int64_t k = rg * 32 + lane;
    if (k < j.K) {
        W t1 = W(0), t2 = W(0);
        double s = 0.0, c = 0.0, sabs = 0.0;
        V mx = V(-INFINITY), mn = V(INFINITY);
        uint32_t mg = 0u, mz = 0xFFFFu, bad = 0u;
#pragma unroll 4
        for (int b = 0; b < j.nb; ++b) {  // block order: the blocked:128 combination
            const size_t o = size_t(b) * size_t(j.Kp) + size_t(k);
            t1 = bs_add(t1, __ldcg(j.part.p1 + o));
            t2 = bs_add(t2, __ldcg(j.part.p2 + o));
            const V bx = __ldcg(j.part.mx + o), bn = __ldcg(j.part.mn + o);
            mx = mx < bx ? bx : mx;
            mn = bn < mn ? bn : mn;
            const uint32_t f = __ldcg(j.part.flags + o);
            if constexpr (BsT<F>::k16) {
                s = __dadd_rn(s, __ldcg(j.part.s + o));
                mg = max(mg, f >> 16);
                mz = min(mz, f & 0xFFFFu);
            } else {
                bad |= f;
                double t, e;
                two_sum_bs(s, __ldcg(j.part.s + o), t, e);
                s = t;
                c = __dadd_rn(__dadd_rn(c, __ldcg(j.part.c + o)), e);
                sabs = __dadd_rn(sabs, double(__ldcg(j.part.sabs + o)));
            }
        }
        Neu n;
        double plain = 0.0;
        bool finite, fast;
        if constexpr (BsT<F>::k16) {
            finite = mg < (F == VABFT_BF16 ? 0x7F80u : 0x7C00u);
            fast = finite && guard_exact<F>(fmaxf(fabsf(mx), fabsf(mn)), mz, j.N);
            n.s = s;
            plain = s;
        } else {
            finite = bad == 0u;
            double hi = 0.0;
            fast = finite && bs_exact_safe(s, c, sabs, j.N, &hi);
            n.s = hi;
        }
        if (!finite) atomicMax(reinterpret_cast<unsigned*>(j.buf.nonfinite), j.epoch);  // nonzero: this launch saw NaN / Inf
        if (!fast) {  // the reference's sequential loops over the row (rare)
            n = Neu{};
            plain = 0.0;
            const auto* r = j.B + k * j.N;
            for (int64_t q = 0; q < j.N; ++q) {
                const double x = Elem<F>::d(r[q]);
                n.add(x);
                plain = __dadd_rn(plain, x);
            }
        }
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
            if (!fast) j.buf.rowsum_abs[k] = fabs(plain);  // by-product of the fallback; see launch_bside_rowsum
        }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile unsigned*>(j.grp_flag + rg) = j.epoch;
}

// The summary warp: BStatsSummary::from's sequential FP64 sums over k in row
// order (threshold_vabft.cpp:15-26) and max_k |sum_j B| (16-bit formats; the
// wide formats' plain row sums come from launch_bside_rowsum), consuming row
// groups as they are published.
template <int F>
__device__ void bs_summary(const BsJob<F>& j) {
    const int lane = threadIdx.x & 31;
    double a_abs = 0.0, a_sq = 0.0, a_var = 0.0, a_max = 0.0;
    int64_t ready = 0;  // groups [0, ready) are published
    // poll the next 32 groups' flags at once; true when group rg is published
    auto poll = [&](int64_t rg) {
        if (rg < ready) return true;
        const int64_t g = ready + lane;
        const bool ok = g >= j.ngroups || *reinterpret_cast<volatile const unsigned*>(j.grp_flag + g) == j.epoch;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int run = bal == 0xffffffffu ? 32 : __ffs(~bal) - 1;
        if (run > 0) {
            __threadfence();  // the group's values were fenced before its flag
            ready += run;
        }
        return rg < ready;
    };
    auto load = [&](int64_t rg, double& m, double& v, double& rs) {
        const int64_t k = rg * 32 + lane;
        const bool valid = k < j.K;
        m = valid ? __ldcg(j.buf.mean + k) : 0.0;
        v = valid ? __ldcg(j.buf.vb + k) : 0.0;
        rs = (valid && BsT<F>::k16) ? __ldcg(j.buf.rowsum_abs + k) : 0.0;
    };
    double m, v, rs;
    while (!poll(0)) __nanosleep(64);
    load(0, m, v, rs);
    for (int64_t rg = 0; rg < j.ngroups; ++rg) {
        // the next group's values are in flight while this group's chain runs
        double mn = 0.0, vn = 0.0, rsn = 0.0;
        const bool pre = rg + 1 < j.ngroups && poll(rg + 1);
        if (pre) load(rg + 1, mn, vn, rsn);
        const int cnt = int(j.K - rg * 32 < 32 ? j.K - rg * 32 : 32);
#pragma unroll 8
        for (int q = 0; q < cnt; ++q) {
            const double mq = __shfl_sync(0xffffffffu, m, q);
            a_abs = __dadd_rn(a_abs, fabs(mq));
            a_sq = __dadd_rn(a_sq, __dmul_rn(mq, mq));
            a_var = __dadd_rn(a_var, __shfl_sync(0xffffffffu, v, q));
            a_max = fmax(a_max, __shfl_sync(0xffffffffu, rs, q));
        }
        if (rg + 1 < j.ngroups && !pre) {
            while (!poll(rg + 1)) __nanosleep(64);
            load(rg + 1, mn, vn, rsn);
        }
        m = mn;
        v = vn;
        rs = rsn;
    }
    if (lane == 0) {
        j.buf.summary[0] = a_abs;
        j.buf.summary[1] = a_sq;
        j.buf.summary[2] = a_var;
        if (BsT<F>::k16) j.buf.summary[3] = a_max;
    }
}

template <int F>
constexpr size_t bs_smem() {
    return size_t(kBsWarps) * 32 * (BsT<F>::kWords + 1) * sizeof(typename BsT<F>::Word);
}

template <int F>
__global__ void __launch_bounds__(kBsThreads, F == VABFT_FP64 ? 1 : 2) bside_kernel(const __grid_constant__ BsJob<F> j) {
    using Word = typename BsT<F>::Word;
    constexpr int kStride = BsT<F>::kWords + 1;
    extern __shared__ __align__(16) uint8_t bs_smem_raw[];
    Word* tiles = reinterpret_cast<Word*>(bs_smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && warp == 0) {
        bs_summary<F>(j);
        return;
    }
    // zero padding of the B r vectors (the A-side readers take whole 128-k blocks)
    if (blockIdx.x == 0 && warp == 1) {
        const int64_t kpad = (j.K + 127) / 128 * 128;
        for (int64_t k = j.K + lane; k < kpad; k += 32) {
            j.buf.br1[k] = 0.0f;
            j.buf.br2[k] = 0.0f;
        }
    }
    Word* tile = tiles + size_t(warp) * 32 * kStride;
    const int64_t tw = int64_t(blockIdx.x) * kBsWarps + warp - 1;
    const int64_t nt = int64_t(gridDim.x) * kBsWarps - 1;
    const int64_t tasks = int64_t(j.ngroups) * j.nb;
    for (int64_t t = tw; t < tasks; t += nt) {
        const int64_t rg = t / j.nb;
        const int b = int(t - rg * j.nb);
        bs_block<F>(j, tile, rg, b);
        __threadfence();
        __syncwarp();
        unsigned old = 0;
        if (lane == 0) old = atomicAdd(j.grp_cnt + rg, 1u);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == unsigned(j.nb) - 1u) {
            __threadfence();
            if (lane == 0) j.grp_cnt[rg] = 0u;  // ready for the next launch
            bs_combine<F>(j, rg);
        }
    }
}

// The plain sequential FP64 row sum (threshold_aabft.cpp:42-46) of every B
// row, for A-ABFT computed y on the wide formats: a warp per row stages the
// row through shared memory and lane 0 runs the chain. max_k |sum| is folded
// with an order-free atomic max.
template <int F>
__global__ void __launch_bounds__(128) bside_rowsum_kernel(const typename Elem<F>::T* __restrict__ B, int64_t K,
                                                           int64_t N, double* rowsum_abs, double* summary) {
    using T = typename Elem<F>::T;
    __shared__ T stage[4][256];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = int64_t(blockIdx.x) * 4 + w;
    if (k >= K) return;
    const T* row = B + k * N;
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

template <int F>
void launch_bs(int64_t K, int64_t N, const void* B, int quantize_br, BsideBuffers& buf, cudaStream_t s) {
    BsJob<F> j;
    j.B = static_cast<const typename Elem<F>::T*>(B);
    j.K = K;
    j.N = N;
    j.ngroups = int((K + 31) / 32);
    j.Kp = int64_t(j.ngroups) * 32;
    j.nb = int((N + 127) / 128);
    j.quantize_br = quantize_br;
    j.buf = buf;
    j.part = bs_view<F>(buf.work, j.nb, j.Kp);
    j.grp_cnt = buf.groups;
    j.grp_flag = buf.groups + j.ngroups;
    j.epoch = ++buf.epoch;
    if (j.epoch == 0) j.epoch = ++buf.epoch;  // flags are zero-initialised: never publish epoch 0
    constexpr size_t smem = bs_smem<F>();
    ensure_smem_attr(reinterpret_cast<const void*>(bside_kernel<F>), int(smem));
    const int per_sm = cached_occupancy(reinterpret_cast<const void*>(bside_kernel<F>), kBsThreads, int(smem));
    const int64_t tasks = int64_t(j.ngroups) * j.nb;
    const int64_t want = (tasks + kBsWarps - 1) / kBsWarps + 1;
    const int grid = int(std::min<int64_t>(int64_t(sm_count()) * std::max(per_sm, 1), want));
    bside_kernel<F><<<grid, kBsThreads, smem, s>>>(j);
    check_cuda(cudaGetLastError(), "bside launch");
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

size_t bside_group_words(int64_t K) { return size_t(2 * ((K + 31) / 32)); }

int64_t br_storage_floats(int64_t K) { return ((K + 127) / 128) * 128; }

void launch_bside(int fmt, int64_t K, int64_t N, const void* B, int quantize_br, BsideBuffers& buf,
                  cudaStream_t s) {
    if (!buf.work || !buf.groups) fail(VABFT_LOGIC_ERROR, "launch_bside: workspace missing");
    if (N > (int64_t(1) << 24)) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: weights exceed exact range");
    switch (fmt) {
        case VABFT_BF16: launch_bs<VABFT_BF16>(K, N, B, quantize_br, buf, s); break;
        case VABFT_FP16: launch_bs<VABFT_FP16>(K, N, B, quantize_br, buf, s); break;
        case VABFT_FP32: launch_bs<VABFT_FP32>(K, N, B, 0, buf, s); break;
        case VABFT_FP64: launch_bs<VABFT_FP64>(K, N, B, 0, buf, s); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
}

void launch_bside_rowsum(int fmt, int64_t K, int64_t N, const void* B, BsideBuffers& buf, cudaStream_t s) {
    check_cuda(cudaMemsetAsync(buf.summary + 3, 0, sizeof(double), s), "memset");
    const unsigned grid = unsigned((K + 3) / 4);
    switch (fmt) {
        case VABFT_BF16: bside_rowsum_kernel<VABFT_BF16><<<grid, 128, 0, s>>>(static_cast<const uint16_t*>(B), K, N, buf.rowsum_abs, buf.summary); break;
        case VABFT_FP16: bside_rowsum_kernel<VABFT_FP16><<<grid, 128, 0, s>>>(static_cast<const uint16_t*>(B), K, N, buf.rowsum_abs, buf.summary); break;
        case VABFT_FP32: bside_rowsum_kernel<VABFT_FP32><<<grid, 128, 0, s>>>(static_cast<const float*>(B), K, N, buf.rowsum_abs, buf.summary); break;
        case VABFT_FP64: bside_rowsum_kernel<VABFT_FP64><<<grid, 128, 0, s>>>(static_cast<const double*>(B), K, N, buf.rowsum_abs, buf.summary); break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
    check_cuda(cudaGetLastError(), "bside rowsum launch");
}

}  // namespace vabft_dev
