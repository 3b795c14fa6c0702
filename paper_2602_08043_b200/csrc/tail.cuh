// Verify tail of the fused V-ABFT GEMM, as a warp-level device function so it
// runs both inside the persistent tcgen05 kernel (after a grid barrier) and as
// a standalone kernel (profiling stage mask).
//
//   A-row statistics -> V-ABFT T_i   threshold_vabft.cpp:28-61, stats.cpp:9-32
//   A (B r) checksums, C r row sums  checksum.cpp:103-187 (FP32, blocked:128)
//   D1/D2, strict compare, NaN rule, localization, correction
//                                    detect.cpp:9-55
//
// One warp owns a 32-row group (lane = row). The ordered FP32 partials are
// row-group-major (part_index), so the group's segment of each array is one
// contiguous span: lane 0 fetches them with cp.async.bulk into the warp's
// shared-memory slice (one memory round trip per chunk) and every lane then
// combines its row's partials in block order. The order-independent A-row
// statistics come from per-row atomics, which the tail resets after use.
#pragma once

#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "ptx.cuh"

namespace vabft_dev {

constexpr int kTailChunkBlocks = 96;                        // blocks per bulk round trip
constexpr uint32_t kTailWarpSmem = 2u * kTailChunkBlocks * 32 * 4;  // 24 KiB per warp

// order-preserving uint32 keys of floats (for atomicMax / atomicMin)
__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_decode(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// n * max|x| < 2^(53 + lsb(min nonzero |x|)) => plain FP64 sums of the row are
// exact in any order (so they equal the reference's sequential Neumaier
// result); mnz_pat is (smallest nonzero magnitude - 1), >= 0x7FFF if none.
template <int F>
__device__ __forceinline__ bool guard_exact(float max_abs, uint32_t mnz_pat, int64_t n) {
    if (mnz_pat >= 0x7FFFu) return true;
    if (!isfinite(max_abs)) return false;
    const uint32_t pat = mnz_pat + 1;
    int lsb;
    if constexpr (F == VABFT_BF16) {
        const int ef = int((pat >> 7) & 0xFF);
        lsb = (ef == 0 ? 1 : ef) - 127 - 7;
    } else {
        const int ef = int((pat >> 10) & 0x1F);
        lsb = (ef == 0 ? 1 : ef) - 15 - 10;
    }
    const int top = ilogbf(max_abs) + 1 + (64 - __clzll(static_cast<unsigned long long>(n)));
    return top <= 53 + lsb;
}

// The reference's Neumaier row sum fl(sum + comp) (stats.cpp:12-24) of one
// row that failed the exactness guard, by the whole warp (all lanes call, all
// get the result). The exact sum as a TwoSum cascade per lane over strided
// elements, merged in a butterfly (TwoSum is symmetric, so every lane holds
// the same merged value); fl(s + c) is the reference's result unless the
// exact sum lies within 8 (K u)^2 sum|x| of a rounding midpoint
// (exact_sum_safe). Otherwise — or when the plain sequential FP64 sum is
// wanted too (`plain`: aabft_computed_y's row sums of B) — the reference's
// loops run in row order with the elements staged in registers: lane l holds
// elements [32 l, 32 l + 32) of each 1024-element chunk and the running
// state passes from lane to lane. Cost: ~1 us at K = 4096 (parallel), ~10 us
// (sequential, about one FP64 add latency per element).
template <int F>
__device__ __noinline__ double warp_neumaier_row(const typename Elem<F>::T* row, int64_t K, double* plain) {
    const int lane = threadIdx.x & 31;
    if (plain == nullptr) {
        double s = 0.0, c = 0.0, sabs = 0.0;
        for (int64_t q = lane; q < K; q += 32) {
            const double x = Elem<F>::d(row[q]);
            double t, e;
            two_sum(s, x, t, e);
            s = t;
            c = __dadd_rn(c, e);
            sabs = __dadd_rn(sabs, fabs(x));
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            const double so = __shfl_xor_sync(0xffffffffu, s, m), co = __shfl_xor_sync(0xffffffffu, c, m);
            double t, e;
            two_sum(s, so, t, e);
            s = t;
            c = __dadd_rn(__dadd_rn(c, co), e);
            sabs = __dadd_rn(sabs, __shfl_xor_sync(0xffffffffu, sabs, m));
        }
        double hi;
        if (exact_sum_safe(s, c, sabs, K, &hi)) return hi;
    }
    Neu n;
    double pl = 0.0;
    for (int64_t j0 = 0; j0 < K; j0 += 1024) {
        double x[32];
        const int64_t b = j0 + int64_t(lane) * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = b + e < K ? Elem<F>::d(row[b + e]) : 0.0;
        for (int l = 0; l < 32; ++l) {
            if (lane == l) {
                const int cnt = int(K - b < 32 ? (K - b > 0 ? K - b : 0) : 32);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    if (e < cnt) {
                        n.add(x[e]);
                        pl = __dadd_rn(pl, x[e]);
                    }
                }
            }
            n.s = __shfl_sync(0xffffffffu, n.s, l);
            n.c = __shfl_sync(0xffffffffu, n.c, l);
            pl = __shfl_sync(0xffffffffu, pl, l);
        }
    }
    if (plain) *plain = pl;
    return __dadd_rn(n.s, n.c);
}

// Sequentially accumulate arrays x1/x2 (blocks [0, nb) of row group g) in
// block order, fetching chunks through the warp's smem slice.
__device__ __forceinline__ void ordered_sums(const float* x1, const float* x2, int64_t nb, int64_t g,
                                             float* sbuf, uint32_t bar, uint32_t& bar_phase,
                                             float& r1, float& r2) {
    const int lane = threadIdx.x & 31;
    const size_t base = part_index(0, g * 32, nb);
    for (int64_t b0 = 0; b0 < nb; b0 += kTailChunkBlocks) {
        const int64_t cnt = (nb - b0) < kTailChunkBlocks ? (nb - b0) : kTailChunkBlocks;
        const uint32_t bytes = uint32_t(cnt * 32 * 4);
        __syncwarp();
        if (lane == 0) {
            mbar_arrive_expect_tx(bar, 2 * bytes);
            bulk_load(smem_u32(sbuf), x1 + base + b0 * 32, bytes, bar);
            bulk_load(smem_u32(sbuf + kTailChunkBlocks * 32), x2 + base + b0 * 32, bytes, bar);
        }
        mbar_wait(bar, bar_phase);
        bar_phase ^= 1u;
        for (int64_t b = 0; b < cnt; ++b) {  // reduce_terms NativeBlocked(128), in order
            r1 = __fadd_rn(r1, sbuf[b * 32 + lane]);
            r2 = __fadd_rn(r2, sbuf[kTailChunkBlocks * 32 + b * 32 + lane]);
        }
    }
}

// The reference's Neumaier row sum of one 16-bit row (a row that failed the
// exactness guard), by the warp in INTEGER arithmetic: element x = +-M 2^q
// (M the integer significand, q the exponent of its lsb) adds M << (q - qmin)
// into a per-lane 128-bit two's-complement accumulator, qmin being the lsb
// exponent of the row's smallest nonzero magnitude (from the statistics
// trackers) — no FP64 per element. (Measured: FP64 loops inside the running
// tcgen05 GEMM took ~90 us per row; 64 such rows made a 4096^3 launch 2.7x
// slower.) The exact sum E = S 2^qmin is rounded to the nearest double, ties
// to even, by integer ops.
//   Why fl(E) is the reference's fl(sum + comp) (stats.cpp:12-24): every
// running sum s_k, element and Fast2Sum error err_k is a multiple of
// 2^qmin, and |comp| <= sum_k |err_k| <= K ulp(max |s_k|) / 2 <
// 2^(ilogb(max|x|) + 2 lg K - 53). When that is below 2^(53 + qmin) —
// ilogb(max|x|) + 2 lg K - qmin <= 104 — no addition into comp rounds, so
// comp_K = sum_k err_k = E - s_K exactly and the final fl(s_K + comp_K) =
// fl(E): including exact ties, which a margin test must give up on (a BF16
// row of O(1) and ~1e-10 entries lands on a midpoint ~1 time in 7). FP16
// rows always qualify. Wider rows that still fit 127 bits take the margin
// test (exact_sum_safe, margin from K max|x| >= sum|x|); false (the caller
// falls back to warp_neumaier_row) for the rest and for non-finite rows.
template <int F>
__device__ __noinline__ bool warp_exact_sum16(const uint16_t* row /* 16-byte aligned */, int64_t K, uint32_t mnz_pat, float amax,
                                               double* out) {
    constexpr int kBias = F == VABFT_BF16 ? 134 : 25;  // q = E - kBias for normals, 1 - kBias for subnormals
    constexpr int kMant = F == VABFT_BF16 ? 7 : 10;
    const int lane = threadIdx.x & 31;
    if (mnz_pat >= 0x7FFFu || !isfinite(amax) || amax == 0.0f) return false;
    const uint32_t pat = mnz_pat + 1;
    const int ef = int(pat >> kMant);
    const int qmin = (ef == 0 ? 1 : ef) - kBias;
    const int lg = 64 - __clzll(static_cast<unsigned long long>(K));
    const int span = ilogbf(amax) - qmin;
    if (span + lg + 2 > 126) return false;
    const bool comp_exact = span + 2 * lg <= 104;
    unsigned __int128 acc = 0;
    auto add = [&](uint32_t h) {
        const uint32_t e = (h >> kMant) & (F == VABFT_BF16 ? 0xFFu : 0x1Fu);
        const uint32_t m = (h & ((1u << kMant) - 1u)) | (e ? (1u << kMant) : 0u);
        const int sh = (e ? int(e) : 1) - kBias - qmin;  // >= 0 for every nonzero element
        unsigned __int128 v = static_cast<unsigned __int128>(m) << (sh > 0 ? sh : 0);
        if (h & 0x8000u) v = ~v + 1;
        acc += v;
    };
    // the row in 4 KiB rounds of eight independent 16-byte loads per lane (K
    // % 8 == 0 and 16-byte rows on the fused path): one L2 round trip per
    // round — a strided one-element-per-iteration loop paid one per element
    // inside the running GEMM (measured ~90 us per row)
    const uint4* r4 = reinterpret_cast<const uint4*>(row);
    const int64_t n4 = K / 8;
    for (int64_t c0 = 0; c0 < n4; c0 += 32 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t idx = c0 + u * 32 + lane;
            v[u] = idx < n4 ? __ldcg(r4 + idx) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                add(w[q] & 0xFFFFu);
                add(w[q] >> 16);
            }
        }
    }
    for (int64_t j = n4 * 8 + lane; j < K; j += 32) add(row[j]);  // K % 8 tail (other callers)
#pragma unroll
    for (int mm = 16; mm >= 1; mm >>= 1) {
        const unsigned long long lo = static_cast<unsigned long long>(acc);
        const unsigned long long hi = static_cast<unsigned long long>(acc >> 64);
        const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, mm);
        const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, hi, mm);
        acc += (static_cast<unsigned __int128>(ohi) << 64) | olo;
    }
    const bool neg = static_cast<long long>(static_cast<unsigned long long>(acc >> 64)) < 0;
    const unsigned __int128 mag = neg ? ~acc + 1 : acc;
    if (mag == 0) {
        if (!comp_exact) return false;
        *out = 0.0;  // s_K + comp_K == 0 exactly: +0 under round-to-nearest
        return true;
    }
    const unsigned long long mh = static_cast<unsigned long long>(mag >> 64);
    const unsigned long long ml = static_cast<unsigned long long>(mag);
    const int nbits = mh ? 128 - __clzll(mh) : 64 - __clzll(ml);
    const int drop = nbits > 53 ? nbits - 53 : 0;
    unsigned __int128 m53 = mag >> drop;
    if (drop > 0) {  // round to nearest, ties to even
        const unsigned __int128 rem = mag - (m53 << drop);
        const unsigned __int128 half = static_cast<unsigned __int128>(1) << (drop - 1);
        if (rem > half || (rem == half && (m53 & 1))) m53 += 1;
    }
    if (comp_exact) {
        const double h = scalbn(__ull2double_rn(static_cast<unsigned long long>(m53)), drop + qmin);
        *out = neg ? -h : h;
        return true;
    }
    const unsigned __int128 hint = m53 << drop;  // |hi| in units of 2^qmin
    // lo = E - hi (|lo| <= 2^(drop - 1): rounding it to a double is far below the margin)
    const bool lneg = mag < hint;
    const unsigned __int128 r = lneg ? hint - mag : mag - hint;
    const double rd = __ull2double_rn(static_cast<unsigned long long>(r >> 64)) * 18446744073709551616.0 +
                      __ull2double_rn(static_cast<unsigned long long>(r));
    double hi = scalbn(__ull2double_rn(static_cast<unsigned long long>(m53)), drop + qmin);
    double lo = scalbn(rd, qmin);
    if (lneg) lo = -lo;
    if (neg) {
        hi = -hi;
        lo = -lo;
    }
    return exact_sum_safe(hi, lo, __dmul_ru(double(K), double(amax)), K, out);
}

__device__ unsigned long long g_tail_dbg[4];  // developer counters: integer-path successes / fallbacks

// ---------------------------------------------------------------- pieces
// Threshold of row i from its order-independent statistics (which are reset
// to their identities for the next launch) and the A (B r) checksums from
// their FP32 blocked:128 sums t1 / t2 (quantized offline).
// Called by all lanes of the warp (valid: lane's row exists). Rows failing
// the exactness guard get the reference's Neumaier sum from
// warp_neumaier_row, the whole warp working on one such row at a time.
template <int F>
__device__ __forceinline__ void row_threshold(const TailArgs& a, int64_t i, bool valid, double sum, uint32_t kmax,
                                              uint32_t kmin, uint32_t mnz, float t1, float t2, double& tv,
                                              double& c1, double& c2, float& amax) {
    const float mx = fkey_decode(kmax);
    const float mn = fkey_decode(kmin);
    amax = fmaxf(fabsf(mx), fabsf(mn));
    const bool slow = valid && !guard_exact<F>(amax, mnz, a.K);
    unsigned rows = __ballot_sync(0xffffffffu, slow);
    if (rows && (threadIdx.x & 31) == 0 && a.counts)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_SLOW_STATS),
                  static_cast<unsigned long long>(__popc(rows)));
    while (rows) {
        const int l = __ffs(rows) - 1;
        rows &= rows - 1;
        const int64_t il = i - (threadIdx.x & 31) + l;
        const uint32_t mz_l = __shfl_sync(0xffffffffu, mnz, l);
        const float amax_l = __shfl_sync(0xffffffffu, amax, l);
        double hs;
        const bool ok16 = warp_exact_sum16<F>(a.A + il * a.lda, a.K, mz_l, amax_l, &hs);
        if (!ok16) hs = warp_neumaier_row<F>(a.A + il * a.lda, a.K, nullptr);
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_tail_dbg[ok16 ? 0 : 1], 1ull);
        if ((threadIdx.x & 31) == l) sum = hs;
    }
    if (!valid) {
        amax = 0.0f;
        return;
    }
    a.rsum[i] = 0.0;
    a.rmax[i] = 0u;
    a.rmin[i] = 0xFFFFFFFFu;
    a.rmnz[i] = 0xFFFFFFFFu;
    Neu fin;
    fin.s = sum;
    double mean, vb;
    stats_finish(fin, double(mx), double(mn), a.K, &mean, &vb);
    tv = vabft_threshold_total(mean, vb, a.bsum[0], a.bsum[1], a.bsum[2], a.N, a.e_max, a.c_sigma);
    if (a.quantize_cr) {
        t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
        t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
    }
    c1 = double(t1);
    c2 = double(t2);
}

// Verdict of row i (detect.cpp:19-55) from its row sums r1 / r2, checksums
// c1 / c2 and V-ABFT threshold tv (A-ABFT methods replace it), plus the
// warp's counters.
template <int F>
__device__ __forceinline__ void row_verdict(const TailArgs& a, int64_t i, bool valid, float r1, float r2,
                                            double c1, double c2, double tv) {
    const int lane = threadIdx.x & 31;
    bool det = false, located = false, isnan_row = false, corrected = false;
    if (valid) {
        double t;
        if (a.method == 0) {
            t = tv;
        } else if (a.method == 3) {
            t = a.t_in[i * a.ldt];
        } else {
            const double y = a.method == 1 ? a.aabft_fixed_y : __dmul_rn(*a.max_abs_a, a.bsum[3]);
            t = aabft_total(a.K, a.aabft_t, y, a.aabft_conf);
        }
        if (a.T_out) a.T_out[i] = t;
        const double d1 = __dsub_rn(double(r1), c1);
        const double d2 = __dsub_rn(double(r2), c2);
        int64_t loc = -1;
        double res = 0.0;
        if (isnan(d1) || isnan(d2)) {
            det = true;
            isnan_row = true;
        } else {
            det = fabs(d1) > t;
            if (det && fabs(d1) > __dmul_rn(a.floor_scale, t)) {
                int64_t j;
                double rr;
                if (localize_dev(d1, d2, a.N, &j, &rr)) {
                    loc = j;
                    res = rr;
                    located = true;
                    // correct (detect.cpp:57-64) for a confidently located single
                    // error (residual < 0.5 - DetectOptions::residual_margin)
                    if (a.correct && a.C != nullptr && rr < 0.4) {
                        uint16_t* cij = a.C + i * a.ldc + j;
                        *cij = quantize16_bits_d<F>(__dsub_rn(double(bits16_to_float<F>(*cij)), d1));
                        corrected = true;
                    }
                }
            }
        }
        if (a.v.diff1) a.v.diff1[i] = d1;
        if (a.v.diff2) a.v.diff2[i] = d2;
        if (a.v.detected) a.v.detected[i] = det ? 1 : 0;
        if (a.v.location) a.v.location[i] = loc;
        if (a.v.residual) a.v.residual[i] = res;
        if (a.v.row_check1) a.v.row_check1[i] = c1;
        if (a.v.row_check2) a.v.row_check2[i] = c2;
    }
    if (a.counts) {
        const unsigned mv = __ballot_sync(0xffffffffu, valid);
        const unsigned md = __ballot_sync(0xffffffffu, det);
        const unsigned ml = __ballot_sync(0xffffffffu, located);
        const unsigned mn = __ballot_sync(0xffffffffu, isnan_row);
        const unsigned mc = __ballot_sync(0xffffffffu, corrected);
        if (lane == 0) {
            if (mc) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_CORRECTED), __popc(mc));
            if (mv) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_ROWS), __popc(mv));
            if (md) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_DETECTED), __popc(md));
            if (ml) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_LOCATED), __popc(ml));
            if (mn) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_NAN), __popc(mn));
        }
    }
}

// ------------------------------------------------- smem-staged (tail warps)
// phase bit 1: statistics -> T_i and A (B r); bit 2: row sums + verify.
// Phase 1 alone stages cr1/cr2/Tv for a later phase-2 pass (A-ABFT computed y
// needs the global max|A| first).
template <int F>
__device__ void verify_rowgroup(const TailArgs& a, int64_t g, int phase, float* sbuf, uint32_t bar,
                                uint32_t& bar_phase) {
    const int lane = threadIdx.x & 31;
    const int64_t i = g * 32 + lane;
    const bool valid = i < a.M;
    double c1 = 0.0, c2 = 0.0, tv = 0.0;
    if (phase & 1) {
        float t1 = 0.0f, t2 = 0.0f;
        ordered_sums(a.sp1, a.sp2, a.nblkK, g, sbuf, bar, bar_phase, t1, t2);
        float amax = 0.0f;
        row_threshold<F>(a, i, valid, valid ? __ldcg(a.rsum + i) : 0.0, valid ? __ldcg(a.rmax + i) : 0u,
                         valid ? __ldcg(a.rmin + i) : 0xFFFFFFFFu, valid ? __ldcg(a.rmnz + i) : 0xFFFFFFFFu, t1, t2, tv,
                         c1, c2, amax);
        if (valid) {
            if (phase == 1) {
                a.cr1[i] = c1;
                a.cr2[i] = c2;
                a.Tv[i] = tv;
            }
        }
        if (a.method == 2) {  // one atomic per warp for max|A| (A-ABFT computed y)
            float wmax = amax;
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, m));
            if (lane == 0) atomic_max_nonneg(a.max_abs_a, double(wmax));
        }
    }
    if (!(phase & 2)) return;
    float r1 = 0.0f, r2 = 0.0f;
    ordered_sums(a.part1, a.part2, a.nblkN, g, sbuf, bar, bar_phase, r1, r2);
    if (valid && !(phase & 1)) {
        c1 = a.cr1[i];
        c2 = a.cr2[i];
        tv = a.Tv[i];
    }
    row_verdict<F>(a, i, valid, r1, r2, c1, c2, tv);
}

// ---------------------------------------------- L2-direct (inside the GEMM)
// Streamed verification inside the GEMM, whose shared memory is all
// pipeline: everything is read straight from L2 (lane = row; each block of a
// partial array is one coalesced 128-byte line for the warp). It runs in two
// halves so that the half left after the final MMA is short:
//   stats half  (the warp completing a group's statistics, usually long
//                before its last tile): T_i and the A (B r) checksums,
//                staged in cr1 / cr2 / Tv;
//   final half  (the warp making the group's last arrival): the row sums
//                and the verdict, one round of loads for N <= 32 * 128.
constexpr int kDirectBatch = 32;

// ordered FP32 sums of two partial arrays (reduce_terms NativeBlocked(128))
__device__ __forceinline__ void ordered_sums_l2(const float* x1, const float* x2, int64_t nb, int64_t g,
                                                float& r1, float& r2) {
    const int lane = threadIdx.x & 31;
    const float* p1 = x1 + part_index(0, g * 32, nb) + lane;
    const float* p2 = x2 + part_index(0, g * 32, nb) + lane;
    for (int64_t b0 = 0; b0 < nb; b0 += kDirectBatch) {
        float v1[kDirectBatch], v2[kDirectBatch];
#pragma unroll
        for (int j = 0; j < kDirectBatch; ++j) {
            const bool ok = b0 + j < nb;
            v1[j] = ok ? __ldcg(p1 + (b0 + j) * 32) : 0.0f;
            v2[j] = ok ? __ldcg(p2 + (b0 + j) * 32) : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < kDirectBatch; ++j) {
            if (b0 + j < nb) {
                r1 = __fadd_rn(r1, v1[j]);
                r2 = __fadd_rn(r2, v2[j]);
            }
        }
    }
}

template <int F>
__device__ void stats_half_direct(const TailArgs& a, int64_t g) {
    const int lane = threadIdx.x & 31;
    const int64_t i = g * 32 + lane;
    const bool valid = i < a.M;
    double sum = 0.0;
    uint32_t kmax = 0u, kmin = 0xFFFFFFFFu, mnz = 0xFFFFFFFFu;
    if (valid) {
        sum = __ldcg(a.rsum + i);
        kmax = __ldcg(a.rmax + i);
        kmin = __ldcg(a.rmin + i);
        mnz = __ldcg(a.rmnz + i);
    }
    float t1 = 0.0f, t2 = 0.0f;
    ordered_sums_l2(a.sp1, a.sp2, a.nblkK, g, t1, t2);
    double c1, c2, tv;
    float amax;
    row_threshold<F>(a, i, valid, sum, kmax, kmin, mnz, t1, t2, tv, c1, c2, amax);
    if (valid) {
        a.cr1[i] = c1;
        a.cr2[i] = c2;
        a.Tv[i] = tv;
    }
}

template <int F>
__device__ __forceinline__ void final_half_direct(const TailArgs& a, int64_t g) {
    const int lane = threadIdx.x & 31;
    const int64_t i = g * 32 + lane;
    const bool valid = i < a.M;
    double c1 = 0.0, c2 = 0.0, tv = 0.0;
    if (valid) {
        c1 = __ldcg(a.cr1 + i);
        c2 = __ldcg(a.cr2 + i);
        tv = __ldcg(a.Tv + i);
    }
    float r1 = 0.0f, r2 = 0.0f;
    ordered_sums_l2(a.part1, a.part2, a.nblkN, g, r1, r2);
    row_verdict<F>(a, i, valid, r1, r2, c1, c2, tv);
}

// Self-resetting grid barrier for a co-resident (cooperative) grid: the last
// arriving CTA resets the count and bumps the generation, so the same state
// works across launches and CUDA-graph replays.
__device__ __forceinline__ void grid_barrier(unsigned int* count, volatile unsigned int* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int my_gen = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(const_cast<unsigned int*>(gen), 1u);
        } else {
            while (*gen == my_gen) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace vabft_dev
