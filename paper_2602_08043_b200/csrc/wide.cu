// K5 — the FP64 fused V-ABFT GEMM (SIMT DFMA) and the verify tail shared by
// the wide formats (FP32 / FP64) of vabft_fused_gemm.
//
//   dgemm_kernel      C = A B in FP64 with DFMA, k in increasing order per
//                     output (sequential FMA accumulation); the ABFT epilogue
//                     stages the 128 x 128 tile in shared memory, applies the
//                     non-finite saturation of run_gemm (precision.cpp:303-310)
//                     and the optional per-row bit flip (faults.cpp:104-168,
//                     bits 0-63 of the FP64 accumulator), and writes the
//                     per-(128-column block, row) partials of C r1 / C r2
//                     summed in column order (checksum.cpp:160-187 with a
//                     NativeBlocked(128) FP64 precision).
//   wide_tail_kernel  per row: blocked:128 combination of the partials, the
//                     V-ABFT / A-ABFT threshold (threshold_vabft.cpp:28-61,
//                     threshold_aabft.cpp:31-60), D1 / D2, strict compare, NaN
//                     rule, localization and optional correction
//                     (detect.cpp:9-64), counters.
//
// DGEMM mapping: 128 x 128 x kDBK (32) CTA tiles, 256 threads (8 warps as 4 x 2),
// an 8 x 8 register tile per thread (rows wm*32 + 8j + 2ty + {0,1}, columns
// wn*64 + 16j + 2tx + {0,1}) so that every shared-memory fragment read is a
// conflict-free 16-byte access; a 3-stage cp.async ring (A rows padded to
// kDBK + 2 doubles; 16-deep tiles with 4 stages measured ~2 % slower). Per k pair: 16 LDS.128 for 128 DFMA — the FP64 pipe (64 DFMA /
// clk / SM) is the bound, not shared memory.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "ptx.cuh"
#include "reducers.cuh"
#include "tail.cuh"

#ifndef VABFT_DBK
#define VABFT_DBK 32
#endif
#ifndef VABFT_DSTAGES
#define VABFT_DSTAGES 3
#endif

namespace vabft_dev {

namespace {

constexpr int kDBM = 128, kDBN = 128, kDBK = VABFT_DBK, kDStages = VABFT_DSTAGES, kDThreads = 256;
constexpr int kALd = kDBK + 2;          // doubles per staged A row (16-byte aligned, conflict-free)
constexpr int kAStage = kDBM * kALd;    // doubles
constexpr int kBStage = kDBK * kDBN;
constexpr int kStage = kAStage + kBStage;
constexpr int kCLd = kDBN + 1;          // epilogue staging stride: row walks are conflict-free
constexpr size_t kDSmem = sizeof(double) * size_t(kDStages) * kStage;
static_assert(sizeof(double) * kDBM * kCLd <= kDSmem, "epilogue staging reuses the operand ring");

struct DgemmParams {
    int64_t M, N, K;
    const double* A;
    const double* B;
    double* C;
    WideEpilogue epi;
};

__device__ __forceinline__ double saturate_f64(double x) {
    return isfinite(x) ? x : copysign(1.7976931348623157e308, x);
}

template <bool kAbft, bool kInject>
__global__ void __launch_bounds__(kDThreads, 1) dgemm_kernel(const __grid_constant__ DgemmParams p) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m0 = int64_t(blockIdx.y) * kDBM, n0 = int64_t(blockIdx.x) * kDBN;
    const int wm = warp & 3, wn = warp >> 2, ty = lane >> 3, tx = lane & 7;
    const int64_t ktiles = (p.K + kDBK - 1) / kDBK;
    griddep_launch_dependents();  // the A pass may start on SMs this grid's last wave leaves idle

    auto load_stage = [&](int64_t kt, int slot) {
        double* As = sm + size_t(slot) * kStage;
        double* Bs = As + kAStage;
        const int64_t k0 = kt * kDBK;
        constexpr int kAChunks = kDBK / 2;  // 16-byte chunks per staged A row
#pragma unroll
        for (int q = 0; q < kDBM * kAChunks / kDThreads; ++q) {  // A: 128 rows x kDBK / 2 chunks of 2 doubles
            const int c = tid + q * kDThreads;
            const int r = c / kAChunks, part = c % kAChunks;
            const int64_t gr = m0 + r, gk = k0 + part * 2;
            const bool ok = gr < p.M && gk < p.K;
            cp_async16(smem_u32(As + r * kALd + part * 2), ok ? p.A + gr * p.K + gk : p.A, ok);
        }
#pragma unroll
        for (int q = 0; q < kDBK * 64 / kDThreads; ++q) {  // B: kDBK rows x 64 chunks
            const int c = tid + q * kDThreads;
            const int r = c >> 6, part = c & 63;
            const int64_t gk = k0 + r, gc = n0 + part * 2;
            const bool ok = gk < p.K && gc < p.N;
            cp_async16(smem_u32(Bs + r * kDBN + part * 2), ok ? p.B + gk * p.N + gc : p.B, ok);
        }
    };

    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

#pragma unroll
    for (int s = 0; s < kDStages - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_async_commit();
    }
#pragma unroll 1
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<kDStages - 2>();
        __syncthreads();
        const int64_t nk = kt + kDStages - 1;
        if (nk < ktiles) load_stage(nk, int(nk % kDStages));
        cp_async_commit();
        const double* As = sm + size_t(kt % kDStages) * kStage;
        const double* Bs = As + kAStage;
#pragma unroll
        for (int kk = 0; kk < kDBK; kk += 2) {
            double2 a[8], b0[4], b1[4];
#pragma unroll
            for (int ri = 0; ri < 8; ++ri) {
                const int r = wm * 32 + (ri >> 1) * 8 + ty * 2 + (ri & 1);
                a[ri] = *reinterpret_cast<const double2*>(As + r * kALd + kk);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = wn * 64 + j * 16 + tx * 2;
                b0[j] = *reinterpret_cast<const double2*>(Bs + kk * kDBN + c);
                b1[j] = *reinterpret_cast<const double2*>(Bs + (kk + 1) * kDBN + c);
            }
#pragma unroll
            for (int ri = 0; ri < 8; ++ri)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[ri][2 * j] = fma(a[ri].x, b0[j].x, acc[ri][2 * j]);
                    acc[ri][2 * j + 1] = fma(a[ri].x, b0[j].y, acc[ri][2 * j + 1]);
                }
#pragma unroll
            for (int ri = 0; ri < 8; ++ri)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[ri][2 * j] = fma(a[ri].y, b1[j].x, acc[ri][2 * j]);
                    acc[ri][2 * j + 1] = fma(a[ri].y, b1[j].y, acc[ri][2 * j + 1]);
                }
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- epilogue: stage the tile, ABFT row pass, coalesced store
    double* Cs = sm;
#pragma unroll
    for (int ri = 0; ri < 8; ++ri) {
        const int r = wm * 32 + (ri >> 1) * 8 + ty * 2 + (ri & 1);
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
            const int c = wn * 64 + (ci >> 1) * 16 + tx * 2 + (ci & 1);
            Cs[r * kCLd + c] = saturate_f64(acc[ri][ci]);
        }
    }
    __syncthreads();
    if constexpr (kAbft) {
        if (tid < kDBM && m0 + tid < p.M) {
            const int64_t row = m0 + tid;
            double* cr = Cs + tid * kCLd;
            const int nc = int(p.N - n0 < kDBN ? p.N - n0 : kDBN);
            if constexpr (kInject) {
                const int64_t fc = p.epi.fault_col[row];
                if (fc >= n0 && fc < n0 + nc) {
                    const int fbit = p.epi.fault_bit[row], fdir = p.epi.fault_dir[row];
                    const double x = cr[fc - n0];
                    const uint64_t bb = uint64_t(__double_as_longlong(x));
                    const bool ok = bit_eligible(bb, fbit, fdir);
                    const double x2 = ok ? __longlong_as_double(int64_t(bb ^ (uint64_t(1) << fbit))) : x;
                    if (p.epi.fault_records) {
                        vabft_fault_record rr;
                        rr.value_before = x;
                        rr.value_after = x2;
                        rr.applied = ok ? 1 : 0;
                        rr.reserved = 0;
                        p.epi.fault_records[row] = rr;
                    }
                    cr[fc - n0] = x2;
                }
            }
            double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
            for (int c = 0; c < nc; ++c) {
                const double x = cr[c];
                s1 = __dadd_rn(s1, x);
                s2 = __dadd_rn(s2, __dmul_rn(double(n0 + c + 1), x));
            }
            const size_t o = size_t(blockIdx.x) * size_t(p.epi.ld) + size_t(row);
            static_cast<double*>(p.epi.part1)[o] = s1;
            static_cast<double*>(p.epi.part2)[o] = s2;
        }
        __syncthreads();
    }
#pragma unroll 4
    for (int q = 0; q < (kDBM * kDBN / 2) / kDThreads; ++q) {
        const int idx = tid + q * kDThreads;
        const int r = idx >> 6, cp = idx & 63;
        const int64_t gr = m0 + r, gc = n0 + cp * 2;
        if (gr < p.M && gc < p.N)
            __stcs(reinterpret_cast<double2*>(p.C + gr * p.N + gc),
                   make_double2(Cs[r * kCLd + cp * 2], Cs[r * kCLd + cp * 2 + 1]));
    }
}

// A side and verification of the wide fused path: ONE streaming pass over A
// after the GEMM on the same stream (run beside the GEMM on a second stream it
// was starved of memory bandwidth and finished late — measured; a
// programmatic launch lets it take the SMs the GEMM's last wave leaves), then
// the per-row-group combine and the verdicts as a second programmatic launch
// (wide_combine_kernel).
//
// wide_apart_kernel: persistent; a warp task is (32-row group, 128-column
// block of K). The warp streams the 32 x 128 tile through its shared-memory
// slice in 32-column sub-tiles (coalesced 128 / 256-byte row segments, the
// next sub-tile's loads in flight while this one is processed) and lane = row
// walks the block in column order; the block's B r weights are staged once in
// shared memory and read as broadcasts. Per (block, row) it writes:
//  - the NativeBlocked(128) checksum partials sum_j T(br_j) T(a_j) in the
//    working type W (checksum.cpp:103-146);
//  - an error-free (s, c) pair of the row segment's sum, sum |a|, max / min
//    (stats.cpp:9-32). FP32: per 32-element sub-tile a plain FP64 sum, exact
//    when 32 max|x| < 2^(53 + lsb(min nonzero |x|)) (a sub-tile outside that
//    guard is redone with TwoSum from the staged tile), TwoSum-merged into the
//    block's pair; FP64: a TwoSum cascade per element. sum|x| (the margin of
//    exact_sum_safe) is kept in the element type and stored rounded up by a
//    relative 2^-8 (an upper bound).
// wide_combine_kernel (one warp per row group) finishes the group, lane =
// row: checksum partials in block order,
// the (s, c) pairs merged with TwoSum; hi = fl(s + c) equals the reference's
// sequential Neumaier fl(sum + comp) unless the exact sum lies within
// 8 (K u)^2 sum|x| of a rounding midpoint (exact_sum_safe) — those rows get
// the reference's sum from warp_neumaier_row (counted as slow-stats rows), so
// the mean is bit-identical in every case. Then, for thresholds without a
// global dependency, the C-row partials of the GEMM epilogue (blocked:128
// order), the threshold, D1 / D2, the strict compare, the NaN rule,
// localization and the optional correction (detect.cpp:9-64): the whole
// verify tail, in the same kernel. A-ABFT with computed y (global max|A|
// first) stages the row statistics instead and verifies in wide_tail_kernel.
// developer timeline (VABFT_APART_TRACE=1): [0] first CTA start, [1] last
// warp's streaming done, [2] last group finished, [3] first group finished,
// [4] first warp's streaming done
__device__ unsigned long long g_ap_trace[8];
__device__ __forceinline__ unsigned long long ap_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <class W>
struct APart {  // per (block, row) partial arrays, group-major (ap_index)
    W *p1, *p2;
    double *s, *c, *sabs, *mx, *mn;
};

__host__ __device__ inline size_t ap_index(int64_t b, int64_t row, int64_t nb) {
    return size_t(((row >> 5) * nb + b) * 32 + (row & 31));
}

template <class W>
__host__ __device__ inline APart<W> apart_view(void* base, int64_t nb, int64_t ld) {
    const size_t n = size_t(nb) * size_t(ld);
    double* d = static_cast<double*>(base);
    APart<W> a;
    a.p1 = reinterpret_cast<W*>(d);
    a.p2 = reinterpret_cast<W*>(d + n);
    a.s = d + 2 * n;
    a.c = d + 3 * n;
    a.sabs = d + 4 * n;
    a.mx = d + 5 * n;
    a.mn = d + 6 * n;
    return a;
}

// Everything the A pass needs beyond the verdict arguments.
template <class W>
struct ApJob {
    WideTail t;              // verdict arguments (t.apart / t.mean ... unused here)
    const W *br1, *br2;      // B r1 / B r2 in the working type (FP32: the handle's float copies)
    APart<W> part;
    unsigned* gcnt;          // [0]: the pass's task counter (zero at rest; the combine kernel resets it)
    int finish;              // 1: verdicts in this kernel; 0: stage the row statistics
    int trace;               // developer timeline (g_ap_trace)
    double *mean, *vb, *mx, *mn, *cr1, *cr2;  // staging (finish == 0)
};

constexpr int kApWarps = 8;
constexpr int kApLd = 36;  // staged row stride (elements): 16-byte aligned rows, conflict-free 16-byte LDS

// per warp: a 2-slot ring of staged 32 x 32 sub-tiles and a 2-slot ring of
// block weights [B r1 | B r2] (128 + 128 in the working type W == T)
template <int F>
constexpr size_t ap_warp_smem() {
    using T = typename Elem<F>::T;
    return 2 * (32 * kApLd * sizeof(T)) + 2 * (2 * 128 * sizeof(T));
}
template <int F>
constexpr size_t ap_smem() {
    return size_t(kApWarps) * ap_warp_smem<F>();
}

// One element of the FP32 A pass: checksum products (no FMA), the plain FP64
// sub-tile sum, sum|x|, max / min and the exactness-guard trackers.
struct ApF32 {
    float p1 = 0.0f, p2 = 0.0f, sabs = 0.0f, mx = -INFINITY, mn = INFINITY;
    double ps = 0.0;
    uint32_t amx = 0u, mnz = 0xFFFFFFFFu;
    __device__ __forceinline__ void add(float x, float w1, float w2) {
        const uint32_t mag = __float_as_uint(x) & 0x7FFFFFFFu;
        amx = max(amx, mag);
        mnz = min(mnz, mag - 1u);  // 0 wraps to the maximum: ignored
        ps = __dadd_rn(ps, double(x));
        p1 = __fadd_rn(p1, __fmul_rn(w1, x));
        p2 = __fadd_rn(p2, __fmul_rn(w2, x));
        sabs = __fadd_rn(sabs, fabsf(x));
        mx = fmaxf(mx, x);  // finite rows (non-finite ones fail exact_sum_safe and rerun)
        mn = fminf(mn, x);
    }
};

// The verdict of the lanes' rows (lane = row) from their C-row sums r1 / r2,
// checksums c1 / c2 and statistics; warp-aggregated counters.
template <int F>
__device__ __forceinline__ void wide_verdicts(const WideTail& a, int64_t i, bool valid, double r1, double r2,
                                              double mean_i, double vb_i, double c1, double c2) {
    const int lane = threadIdx.x & 31;
    bool det = false, located = false, isnan_row = false, corrected = false;
    if (valid) {
        double t;
        if (a.method == 0) {
            t = vabft_threshold_total(mean_i, vb_i, a.bsum[0], a.bsum[1], a.bsum[2], a.N, a.e_max, a.c_sigma);
        } else if (a.method == 3) {
            t = a.t_in[i * a.ldt];
        } else {
            const double y = a.method == 1 ? a.aabft_fixed_y : __dmul_rn(*a.max_abs_a, a.bsum[3]);
            t = aabft_total(a.K, a.aabft_t, y, a.aabft_conf);
        }
        if (a.T_out) a.T_out[i] = t;
        const double d1 = __dsub_rn(r1, c1);
        const double d2 = __dsub_rn(r2, c2);
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
                    // correct (detect.cpp:57-64): C[i][j] = quantize(C[i][j] - diff1)
                    if (a.correct && a.C != nullptr && rr < 0.4) {
                        if (a.fmt == VABFT_FP64) {
                            double* cij = static_cast<double*>(a.C) + i * a.N + j;
                            *cij = __dsub_rn(*cij, d1);
                        } else {
                            float* cij = static_cast<float*>(a.C) + i * a.N + j;
                            const float q = __double2float_rn(__dsub_rn(double(*cij), d1));
                            *cij = isinf(q) ? copysignf(3.40282346638528859812e+38f, q) : q;
                        }
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
        const unsigned nv = __popc(__ballot_sync(0xffffffffu, valid));
        const unsigned nd = __popc(__ballot_sync(0xffffffffu, det));
        const unsigned nl = __popc(__ballot_sync(0xffffffffu, located));
        const unsigned nn = __popc(__ballot_sync(0xffffffffu, isnan_row));
        const unsigned nc = __popc(__ballot_sync(0xffffffffu, corrected));
        if (lane == 0) {
            unsigned long long* cnt = reinterpret_cast<unsigned long long*>(a.counts);
            if (nv) atomicAdd(cnt + VABFT_COUNT_ROWS, nv);
            if (nd) atomicAdd(cnt + VABFT_COUNT_DETECTED, nd);
            if (nl) atomicAdd(cnt + VABFT_COUNT_LOCATED, nl);
            if (nn) atomicAdd(cnt + VABFT_COUNT_NAN, nn);
            if (nc) atomicAdd(cnt + VABFT_COUNT_CORRECTED, nc);
        }
    }
}

// C r1 / C r2 of the lanes' rows: the epilogue's per-128-column partials
// ([nb][ld], lane = row: coalesced) added in block order (blocked:128).
template <class W>
__device__ __forceinline__ void wide_row_sums(const WideTail& a, int64_t i, double& r1, double& r2) {
    const W* p1 = static_cast<const W*>(a.part1) + i;
    const W* p2 = static_cast<const W*>(a.part2) + i;
    W s1 = W(0), s2 = W(0);
#pragma unroll 8
    for (int64_t b = 0; b < a.nblk; ++b) {
        s1 = radd(s1, __ldcg(p1 + b * a.ld));
        s2 = radd(s2, __ldcg(p2 + b * a.ld));
    }
    r1 = double(s1);
    r2 = double(s2);
}

// Sources of a row group's partials for ap_finish_group (lane = row i):
// straight from L2 (ApGlobal), or staged in shared memory by bulk copies
// (ApStaged: every array of the group lands in one round trip).
template <class W>
struct ApGlobal {
    const APart<W>& part;
    const WideTail& a;
    size_t o0;  // ap_index(0, i, nb)
    int64_t i;
    __device__ W p1(int64_t b) const { return __ldcg(part.p1 + o0 + size_t(b) * 32); }
    __device__ W p2(int64_t b) const { return __ldcg(part.p2 + o0 + size_t(b) * 32); }
    __device__ double s(int64_t b) const { return __ldcg(part.s + o0 + size_t(b) * 32); }
    __device__ double c(int64_t b) const { return __ldcg(part.c + o0 + size_t(b) * 32); }
    __device__ double sabs(int64_t b) const { return __ldcg(part.sabs + o0 + size_t(b) * 32); }
    __device__ double mx(int64_t b) const { return __ldcg(part.mx + o0 + size_t(b) * 32); }
    __device__ double mn(int64_t b) const { return __ldcg(part.mn + o0 + size_t(b) * 32); }
    __device__ W cp1(int64_t b) const { return __ldcg(static_cast<const W*>(a.part1) + i + b * a.ld); }
    __device__ W cp2(int64_t b) const { return __ldcg(static_cast<const W*>(a.part2) + i + b * a.ld); }
};
template <class W>
struct ApStaged {
    const W *sp1, *sp2, *scp1, *scp2;
    const double *ss, *sc, *ssabs, *smx, *smn;
    int lane;
    __device__ W p1(int64_t b) const { return sp1[b * 32 + lane]; }
    __device__ W p2(int64_t b) const { return sp2[b * 32 + lane]; }
    __device__ double s(int64_t b) const { return ss[b * 32 + lane]; }
    __device__ double c(int64_t b) const { return sc[b * 32 + lane]; }
    __device__ double sabs(int64_t b) const { return ssabs[b * 32 + lane]; }
    __device__ double mx(int64_t b) const { return smx[b * 32 + lane]; }
    __device__ double mn(int64_t b) const { return smn[b * 32 + lane]; }
    __device__ W cp1(int64_t b) const { return scp1[b * 32 + lane]; }
    __device__ W cp2(int64_t b) const { return scp2[b * 32 + lane]; }
};

// Finish a row group (lane = row): A statistics and checksums, then either
// the verdicts (finish) or the staged statistics.
template <int F, class W, class Src>
__device__ __forceinline__ void ap_finish_group(const ApJob<W>& j, int64_t rg, const Src& src) {
    using T = typename Elem<F>::T;
    const WideTail& a = j.t;
    const int lane = threadIdx.x & 31;
    const int64_t i = rg * 32 + lane;
    const bool valid = i < a.M;
    const int64_t nb = (a.K + 127) / 128;
    W t1 = W(0), t2 = W(0);
    double s = 0.0, c = 0.0, sabs = 0.0, mx = -INFINITY, mn = INFINITY;
    if (valid) {
#pragma unroll 8
        for (int64_t b = 0; b < nb; ++b) {
            t1 = radd(t1, src.p1(b));
            t2 = radd(t2, src.p2(b));
            double tt, err;
            two_sum(s, src.s(b), tt, err);
            s = tt;
            c = __dadd_rn(__dadd_rn(c, src.c(b)), err);
            sabs = __dadd_rn(sabs, src.sabs(b));
            const double bx = src.mx(b), bn = src.mn(b);
            mx = mx < bx ? bx : mx;
            mn = bn < mn ? bn : mn;
        }
    }
    Neu ns;
    const bool slow = valid && !exact_sum_safe(s, c, sabs, a.K, &ns.s);
    unsigned rows = __ballot_sync(0xffffffffu, slow);
    if (rows && lane == 0 && a.counts)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_SLOW_STATS),
                  static_cast<unsigned long long>(__popc(rows)));
    while (rows) {  // rare: rows next to a rounding midpoint (or non-finite)
        const int l = __ffs(rows) - 1;
        rows &= rows - 1;
        const double hs = warp_neumaier_row<F>(static_cast<const T*>(a.A) + (rg * 32 + l) * a.K, a.K, nullptr);
        if (lane == l) {
            ns = Neu{};
            ns.s = hs;
        }
    }
    double mean_i = 0.0, vb_i = 0.0, c1 = 0.0, c2 = 0.0;
    if (valid) {
        stats_finish(ns, mx, mn, a.K, &mean_i, &vb_i);
        c1 = double(t1);
        c2 = double(t2);
        if (a.qfmt == VABFT_FP32) {  // offline FP32: rounded to the input format (a no-op for W = float)
            c1 = double(float(c1));
            c2 = double(float(c2));
        }
    }
    if (!j.finish) {
        if (valid) {
            j.mean[i] = mean_i;
            j.vb[i] = vb_i;
            j.mx[i] = mx;
            j.mn[i] = mn;
            j.cr1[i] = c1;
            j.cr2[i] = c2;
        }
        return;
    }
    // C r1 / C r2: the GEMM epilogue's per-128-column partials in block order (blocked:128)
    double r1 = 0.0, r2 = 0.0;
    if (valid) {
        W s1 = W(0), s2 = W(0);
#pragma unroll 8
        for (int64_t b = 0; b < a.nblk; ++b) {
            s1 = radd(s1, src.cp1(b));
            s2 = radd(s2, src.cp2(b));
        }
        r1 = double(s1);
        r2 = double(s2);
    }
    wide_verdicts<F>(a, i, valid, r1, r2, mean_i, vb_i, c1, c2);
}

// Bytes of a row group's partials staged by wide_combine_kernel.
template <class W>
__host__ __device__ inline size_t ap_stage_bytes(int64_t nbK, int64_t nbN) {
    return size_t(nbK) * 32 * (2 * sizeof(W) + 5 * sizeof(double)) + size_t(nbN) * 32 * 2 * sizeof(W);
}
constexpr size_t kApStageMax = 200 * 1024;

// The per-row-group combine and verify tail of the wide A pass, one warp per
// row group, after the streaming pass (programmatic launch: scheduled as the
// pass's CTAs retire; griddepcontrol.wait for its partials). kStaged: lane 0
// bulk-copies every partial array of the group into shared memory at once —
// each array's group span is contiguous (group-major layout), the epilogue's
// C-row partials are coalesced 32-row segments loaded alongside — so the
// combine costs about one L2 round trip instead of one per eight blocks. (Measured before: inline combines by
// the last-arriving streaming warp took 5-8 us each under the streaming load
// and stalled that warp's next task; the pass ended 8 us after its last
// task.)
template <int F, class W, bool kStaged>
__global__ void __launch_bounds__(32) wide_combine_kernel(const __grid_constant__ ApJob<W> j) {
    extern __shared__ __align__(16) uint8_t cb[];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31;
    const int64_t rg = blockIdx.x;
    const WideTail& a = j.t;
    const int64_t nb = (a.K + 127) / 128;
    griddep_wait();  // the A pass (which itself waited for the GEMM) complete: partials visible
    if constexpr (kStaged) {
        const int64_t nbN = j.finish ? a.nblk : 0;
        W* sp1 = reinterpret_cast<W*>(cb);
        W* sp2 = sp1 + nb * 32;
        double* ss = reinterpret_cast<double*>(sp2 + nb * 32);
        double* sc = ss + nb * 32;
        double* ssabs = sc + nb * 32;
        double* smx = ssabs + nb * 32;
        double* smn = smx + nb * 32;
        W* scp1 = reinterpret_cast<W*>(smn + nb * 32);
        W* scp2 = scp1 + nbN * 32;
        const uint32_t b0 = smem_u32(&bar);
        if (lane == 0) {
            mbar_init(b0, 1);
            fence_mbar_init();
        }
        __syncwarp();
        if (lane == 0) {
            const uint32_t wbytes = uint32_t(nb * 32 * sizeof(W)), dbytes = uint32_t(nb * 32 * sizeof(double));
            mbar_arrive_expect_tx(b0, uint32_t(ap_stage_bytes<W>(nb, 0)));
            const size_t o = ap_index(0, rg * 32, nb);
            bulk_load(smem_u32(sp1), j.part.p1 + o, wbytes, b0);
            bulk_load(smem_u32(sp2), j.part.p2 + o, wbytes, b0);
            bulk_load(smem_u32(ss), j.part.s + o, dbytes, b0);
            bulk_load(smem_u32(sc), j.part.c + o, dbytes, b0);
            bulk_load(smem_u32(ssabs), j.part.sabs + o, dbytes, b0);
            bulk_load(smem_u32(smx), j.part.mx + o, dbytes, b0);
            bulk_load(smem_u32(smn), j.part.mn + o, dbytes, b0);
        }
        // the C-row partials (32-row segments at stride ld): coalesced loads,
        // 32 in flight per lane, parked in shared memory (each lane reads back
        // only its own row) while the bulk copies land. (Per-lane bulk copies
        // serialise: the compiler loops over the lanes with ELECT / R2UR.)
#pragma unroll 16
        for (int64_t b = 0; b < nbN; ++b) {
            const size_t o = size_t(b) * size_t(a.ld) + size_t(rg) * 32 + size_t(lane);
            scp1[b * 32 + lane] = __ldcg(static_cast<const W*>(a.part1) + o);
            scp2[b * 32 + lane] = __ldcg(static_cast<const W*>(a.part2) + o);
        }
        mbar_wait(b0, 0);
        const ApStaged<W> src{sp1, sp2, scp1, scp2, ss, sc, ssabs, smx, smn, lane};
        ap_finish_group<F, W>(j, rg, src);
    } else {
        const int64_t i = rg * 32 + lane;
        const ApGlobal<W> src{j.part, a, ap_index(0, i, nb), i};
        ap_finish_group<F, W>(j, rg, src);
    }
    if (blockIdx.x == 0 && lane == 0) *j.gcnt = 0u;  // the pass's task counter, for the next launch
    if (j.trace && lane == 0) {
        const unsigned long long t = ap_now();
        atomicMax(&g_ap_trace[2], t);
        atomicMin(&g_ap_trace[3], t);
    }
}

template <int F, class W, bool kVec>
__global__ void __launch_bounds__(32 * kApWarps, F == VABFT_FP64 ? 1 : 2)
    wide_apart_kernel(const typename Elem<F>::T* __restrict__ A, const __grid_constant__ ApJob<W> j) {
    using T = typename Elem<F>::T;
    extern __shared__ __align__(16) uint8_t ap_raw[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* mine = ap_raw + size_t(w) * ap_warp_smem<F>();
    T* tiles = reinterpret_cast<T*>(mine);                          // [2][32 * kApLd]
    W* wtsb = reinterpret_cast<W*>(mine + 2 * 32 * kApLd * sizeof(T));  // [2][256]
    const int64_t M = j.t.M, K = j.t.K;
    const int64_t nb = (K + 127) / 128, ngroups = (M + 31) / 32;
    const int64_t tasks = ngroups * nb;
    const int64_t nt = int64_t(gridDim.x) * kApWarps;
    // Every load is a cp.async into the warp's 2-slot rings, one sub-tile
    // ahead of the fold — across task boundaries too (the next task's first
    // sub-tile and block weights land while this task's last sub-tile is
    // folded) — so no register staging and no exposed load at a task start.
    // No per-task arrivals: the combine is its own launch. (Measured before:
    // long-scoreboard stalls on register staging and on each task's first
    // loads and weights, then the arrivals' release fences — which also wait
    // for the copies in flight — and the inline combines were the top costs.)
    auto issue = [&](int64_t t, int q, int slot, int wslot) {
        const int64_t rg = t / nb, b = t - rg * nb;
        const int64_t r0 = rg * 32, c = b * 128 + int64_t(q) * 32;
        const int rows = int(M - r0 < 32 ? M - r0 : 32);
        T* tile = tiles + slot * (32 * kApLd);
        if constexpr (kVec) {  // FP32, K % 4 == 0, aligned: 16-byte chunks, 8 lanes per 128-byte row segment
            const int64_t col = c + 4 * (lane & 7);
            const int rs = lane >> 3;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = 4 * i + rs;
                const bool ok = r < rows && col < K;
                cp_async16n(smem_u32(tile + r * kApLd + 4 * (lane & 7)), ok ? A + (r0 + r) * K + col : A,
                            ok ? 16 : 0);
            }
        } else {  // lane = column, one element per row
            const int64_t col = c + lane;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const bool ok = r < rows && col < K;
                cp_async_small<int(sizeof(T))>(smem_u32(tile + r * kApLd + lane), ok ? A + (r0 + r) * K + col : A, ok);
            }
        }
        if (q == 0) {  // the block's weights, 16-byte chunks (zero-filled past K)
            const int bw = int(K - b * 128 < 128 ? K - b * 128 : 128);
            constexpr int kPer = int(16 / sizeof(W));  // weights per chunk
            W* wd = wtsb + wslot * 256;
            for (int ch = lane; ch < 128 / kPer; ch += 32) {
                const int e0 = ch * kPer;
                const int nvalid = bw - e0 < 0 ? 0 : (bw - e0 > kPer ? kPer : bw - e0);
                const int64_t o = nvalid ? b * 128 + e0 : 0;  // no bytes read for an empty chunk
                cp_async16n(smem_u32(wd + e0), j.br1 + o, nvalid * int(sizeof(W)));
                cp_async16n(smem_u32(wd + 128 + e0), j.br2 + o, nvalid * int(sizeof(W)));
            }
        }
    };
    if (j.trace && threadIdx.x == 0) atomicMin(&g_ap_trace[0], ap_now());
    griddep_launch_dependents();  // the combine kernel's CTAs take the SMs this pass leaves
    int slot = 0, wslot = 0;
    // Tasks are claimed in order from a counter (j.gcnt[0], reset by the
    // combine kernel): the claim goes out two sub-tiles before a task's end
    // and its result is read at the task's last sub-tile, where the next
    // task's first loads go out. (Static dealing left 27 % of the warps idle
    // in the second round of a 4096^2 pass: 4096 tasks over 2368 warps.)
    auto claim = [&]() {
        unsigned old = 0;
        if (lane == 0) old = atomicAdd(j.gcnt, 1u);
        return old;
    };
    int64_t t = int64_t(__shfl_sync(0xffffffffu, claim(), 0));
    if (t < tasks) issue(t, 0, 0, 0);
    cp_async_commit();
    while (t < tasks) {
        unsigned pend = 0;  // the next task's claim, issued two sub-tiles before it is needed
        int64_t tn = tasks;
        const int64_t rg = t / nb, b = t - rg * nb;
        const int64_t r0 = rg * 32, c0 = b * 128;
        const int bw = int(K - c0 < 128 ? K - c0 : 128);
        const int nsub = (bw + 31) / 32;
        const W* wts = wtsb + wslot * 256;
        W p1 = W(0), p2 = W(0);
        double s = 0.0, c = 0.0;
        T sabs = T(0), mx = T(-INFINITY), mn = T(INFINITY);
        for (int q = 0; q < nsub; ++q) {
            const int64_t cq = c0 + int64_t(q) * 32;
            // (claimed late enough that the claim order follows the warps'
            // progress — a claim at the task start dealt the tasks statically)
            if (q == (nsub > 2 ? nsub - 2 : 0)) pend = claim();
            if (q + 1 < nsub) {
                issue(t, q + 1, slot ^ 1, wslot);
            } else {
                tn = int64_t(__shfl_sync(0xffffffffu, pend, 0));
                if (tn < tasks) issue(tn, 0, slot ^ 1, wslot ^ 1);
            }
            cp_async_commit();
            cp_async_wait<1>();  // this sub-tile (and the task's weights) landed
            __syncwarp();
            const T* trow = tiles + slot * (32 * kApLd) + lane * kApLd;
            const int cnt = int(c0 + bw - cq < 32 ? c0 + bw - cq : 32);  // warp-uniform
            const W* w1 = wts + q * 32;
            const W* w2 = wts + 128 + q * 32;
            if constexpr (F == VABFT_FP32) {
                ApF32 e;
                e.p1 = p1;
                e.p2 = p2;
                e.sabs = sabs;
                e.mx = mx;
                e.mn = mn;
                if (cnt == 32) {  // 16-byte LDS of 4 elements and of their weights
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float4 x4 = reinterpret_cast<const float4*>(trow)[u];
                        const float4 a4 = reinterpret_cast<const float4*>(w1)[u];
                        const float4 b4 = reinterpret_cast<const float4*>(w2)[u];
                        e.add(x4.x, a4.x, b4.x);
                        e.add(x4.y, a4.y, b4.y);
                        e.add(x4.z, a4.z, b4.z);
                        e.add(x4.w, a4.w, b4.w);
                    }
                } else {
                    for (int jj = 0; jj < cnt; ++jj) e.add(trow[jj], w1[jj], w2[jj]);
                }
                p1 = e.p1;
                p2 = e.p2;
                sabs = e.sabs;
                mx = e.mx;
                mn = e.mn;
                double ps = e.ps;
                // exactness guard of the plain sub-tile sum (see guard_exact)
                bool exact = true;
                if (e.mnz != 0xFFFFFFFFu && e.amx < 0x7F800000u) {
                    const int ez = int((e.mnz + 1u) >> 23);
                    const int lsb = (ez == 0 ? 1 : ez) - 127 - 23;
                    const int top = int(e.amx >> 23) - 127 + 1 + 6;  // 32 terms < 2^6 max
                    exact = top <= 53 + lsb;
                }
                if (!exact) {  // rare: the sub-tile's exact sum as a TwoSum cascade
                    double hs = 0.0, hc = 0.0;
                    for (int jj = 0; jj < cnt; ++jj) {
                        double tt, ee;
                        two_sum(hs, double(trow[jj]), tt, ee);
                        hs = tt;
                        hc = __dadd_rn(hc, ee);
                    }
                    ps = hs;
                    c = __dadd_rn(c, hc);
                }
                double tt, ee;
                two_sum(s, ps, tt, ee);
                s = tt;
                c = __dadd_rn(c, ee);
            } else {
#pragma unroll 4
                for (int jj = 0; jj < cnt; ++jj) {
                    const double x = trow[jj];
                    p1 = radd(p1, rmul(w1[jj], x));
                    p2 = radd(p2, rmul(w2[jj], x));
                    double tt, e;
                    two_sum(s, x, tt, e);
                    s = tt;
                    c = __dadd_rn(c, e);
                    sabs = __dadd_rn(sabs, fabs(x));
                    mx = mx < x ? x : mx;
                    mn = x < mn ? x : mn;
                }
            }
            __syncwarp();  // the slot is refilled two steps later
            slot ^= 1;
        }
        const int64_t row = r0 + lane;
        if (row < M) {
            const size_t o = ap_index(b, row, nb);
            j.part.p1[o] = p1;
            j.part.p2[o] = p2;
            j.part.s[o] = s;
            j.part.c[o] = c;
            // an upper bound of sum|x| (the element-type sum is within K u_T relatively)
            j.part.sabs[o] = __dmul_ru(double(sabs), F == VABFT_FP32 ? 1.00390625 : 1.0 + 0x1p-40);
            j.part.mx[o] = double(mx);
            j.part.mn[o] = double(mn);
        }
        wslot ^= 1;
        t = tn;
    }
    cp_async_wait<0>();
    if (j.trace && lane == 0) {
        const unsigned long long now = ap_now();
        atomicMax(&g_ap_trace[1], now);
        atomicMin(&g_ap_trace[4], now);
    }
    griddep_wait();  // never complete before the GEMM this pass may overlap
}

// Verify tail for thresholds with a global dependency (A-ABFT computed y):
// warp per 32-row group (lane = row), the row statistics staged by the A
// pass, the C-row partials in block order, the verdicts.
template <int F>
__global__ void __launch_bounds__(256) wide_tail_kernel(const WideTail a) {
    using W = std::conditional_t<F == VABFT_FP64, double, float>;
    const int64_t rg = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (rg * 32 >= a.M) return;
    const int64_t i = rg * 32 + (threadIdx.x & 31);
    const bool valid = i < a.M;
    double r1 = 0.0, r2 = 0.0, mean_i = 0.0, vb_i = 0.0, c1 = 0.0, c2 = 0.0;
    if (valid) {
        wide_row_sums<W>(a, i, r1, r2);
        mean_i = a.mean[i];
        vb_i = a.vb[i];
        c1 = a.cr1[i];
        c2 = a.cr2[i];
    }
    wide_verdicts<F>(a, i, valid, r1, r2, mean_i, vb_i, c1, c2);
}

__global__ void max_abs_rows_kernel(int64_t m, const double* mx, const double* mn, double* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double v = i < m ? fmax(fabs(mx[i]), fabs(mn[i])) : 0.0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, s));
    if ((threadIdx.x & 31) == 0 && v > 0.0) atomic_max_nonneg(out, v);
}

}  // namespace

void dgemm_launch(int64_t M, int64_t N, int64_t K, const double* A, const double* B, double* C,
                  const WideEpilogue& epi, cudaStream_t stream) {
    if (M < 1 || N < 1 || K < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
    if (K % 2 != 0 || N % 2 != 0) fail(VABFT_UNSUPPORTED, "FP64 GEMM: K and N must be even");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
        fail(VABFT_INVALID_ARGUMENT, "FP64 GEMM: operands must be 16-byte aligned");
    if ((N + kDBN - 1) / kDBN > 0x7FFFFFFF || (M + kDBM - 1) / kDBM > 65535)
        fail(VABFT_UNSUPPORTED, "FP64 GEMM: grid too large");
    DgemmParams p{M, N, K, A, B, C, epi};
    const dim3 grid(unsigned((N + kDBN - 1) / kDBN), unsigned((M + kDBM - 1) / kDBM));
    auto run = [&](void (*kern)(DgemmParams)) {
        ensure_smem_attr(reinterpret_cast<const void*>(kern), int(kDSmem));
        kern<<<grid, kDThreads, kDSmem, stream>>>(p);
    };
    if (!epi.abft) run(dgemm_kernel<false, false>);
    else if (epi.fault_col) run(dgemm_kernel<true, true>);
    else run(dgemm_kernel<true, false>);
    check_cuda(cudaGetLastError(), "dgemm launch");
}

void launch_wide_tail(const WideTail& t, cudaStream_t stream) {
    const unsigned grid = unsigned(((t.M + 31) / 32 + 7) / 8);  // 8 row groups (warps) per CTA
    if (t.fmt == VABFT_FP64) wide_tail_kernel<VABFT_FP64><<<grid, 256, 0, stream>>>(t);
    else wide_tail_kernel<VABFT_FP32><<<grid, 256, 0, stream>>>(t);
    check_cuda(cudaGetLastError(), "wide tail launch");
}

void launch_wide_aside(const WideTail& t, const void* br1, const void* br2, void* apart, unsigned* gcnt,
                       bool finish, double* mean, double* vb, double* mx, double* mn, double* cr1, double* cr2,
                       cudaStream_t stream) {
    const int64_t nb = (t.K + 127) / 128;
    auto run = [&](auto tag) {
        using T = decltype(tag);
        using W = T;
        constexpr int F = sizeof(T) == 8 ? VABFT_FP64 : VABFT_FP32;
        ApJob<W> j;
        j.t = t;
        j.br1 = static_cast<const W*>(br1);
        j.br2 = static_cast<const W*>(br2);
        j.part = apart_view<W>(apart, nb, t.ld);
        j.gcnt = gcnt;
        j.finish = finish ? 1 : 0;
        j.mean = mean;
        j.vb = vb;
        j.mx = mx;
        j.mn = mn;
        j.cr1 = cr1;
        j.cr2 = cr2;
        const bool vec = F == VABFT_FP32 && t.K % 4 == 0 && reinterpret_cast<uintptr_t>(t.A) % 16 == 0;
        auto kern = vec ? wide_apart_kernel<F, W, F == VABFT_FP32> : wide_apart_kernel<F, W, false>;
        constexpr size_t smem = ap_smem<F>();
        ensure_smem_attr(reinterpret_cast<const void*>(kern), int(smem));
        const int per_sm = cached_occupancy(reinterpret_cast<const void*>(kern), 32 * kApWarps, int(smem));
        const int64_t tasks = (t.M + 31) / 32 * nb;
        const int grid = int(std::min<int64_t>(int64_t(sm_count()) * std::max(per_sm, 1), (tasks + kApWarps - 1) / kApWarps));
        // programmatic launch: the pass reads only A and the per-weight B r
        // until a row group's verdicts (griddep_wait), so its CTAs start on
        // the SMs the GEMM's last wave leaves idle
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(32 * kApWarps);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static const int trc = [] {
            const char* e = std::getenv("VABFT_APART_TRACE");
            return e ? std::atoi(e) : 0;
        }();
        j.trace = trc;
        if (trc) {
            const unsigned long long init[8] = {~0ull, 0, 0, ~0ull, ~0ull, 0, 0, 0};
            check_cuda(cudaMemcpyToSymbolAsync(g_ap_trace, init, sizeof(init), 0, cudaMemcpyHostToDevice, stream), "trace");
        }
        check_cuda(cudaLaunchKernelEx(&cfg, kern, static_cast<const T*>(t.A), j), "wide A-side launch");
        // the combine + verify tail: one warp per row group, programmatic launch
        // after the pass; partials staged in shared memory when they fit
        const int64_t ngroups = (t.M + 31) / 32;
        const size_t sbytes = ap_stage_bytes<W>(nb, finish ? t.nblk : 0);
        const bool staged = sbytes <= kApStageMax;
        auto ck = staged ? wide_combine_kernel<F, W, true> : wide_combine_kernel<F, W, false>;
        if (staged) ensure_smem_attr(reinterpret_cast<const void*>(ck), int(sbytes));
        cudaLaunchConfig_t cc = cfg;
        cc.gridDim = dim3(unsigned(ngroups));
        cc.blockDim = dim3(32);
        cc.dynamicSmemBytes = staged ? sbytes : 0;
        check_cuda(cudaLaunchKernelEx(&cc, ck, j), "wide combine launch");
        if (trc) {
            unsigned long long tt[8];
            check_cuda(cudaMemcpyFromSymbolAsync(tt, g_ap_trace, sizeof(tt), 0, cudaMemcpyDeviceToHost, stream), "trace");
            check_cuda(cudaStreamSynchronize(stream), "trace");
            auto us = [&](int i) { return double(tt[i] - tt[0]) * 1e-3; };
            std::fprintf(stderr, "apart trace M=%lld K=%lld grid=%d: first-warp-done %.2f last-warp-done %.2f first-group %.2f last-group %.2f us\n",
                         (long long)t.M, (long long)t.K, grid, us(4), us(1), us(3), us(2));
        }
    };
    if (t.fmt == VABFT_FP64) run(double{});
    else if (t.fmt == VABFT_FP32) run(float{});
    else fail(VABFT_INVALID_ARGUMENT, "wide A side: FP32 / FP64 only");
    check_cuda(cudaGetLastError(), "wide A-side launch");
}

void launch_max_abs_rows(int64_t m, const double* mx, const double* mn, double* out, cudaStream_t stream) {
    max_abs_rows_kernel<<<unsigned((m + 255) / 256), 256, 0, stream>>>(m, mx, mn, out);
    check_cuda(cudaGetLastError(), "max|A| launch");
}

}  // namespace vabft_dev

namespace vabft_dev {

namespace {

// InputA faults of the wide path: per row i, bit fault_bit[i] of
// X[i][fault_col[i]] (inject's eligibility rule, faults.cpp:91-102), with a
// per-row record.
template <class T, class U>
__global__ void flip_rows_kernel(T* X, int64_t rows, int64_t cols, const int32_t* col, const int32_t* bit,
                                 const int32_t* dir, vabft_fault_record* rec) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int64_t k = col[i];
    if (k < 0 || k >= cols) return;
    U* p = reinterpret_cast<U*>(X + i * cols + k);
    const U b = *p;
    const bool ok = bit_eligible(uint64_t(b), bit[i], dir[i]);
    const U nb = ok ? U(b ^ (U(1) << bit[i])) : b;
    *p = nb;
    if (rec) {
        vabft_fault_record r;
        T before, after;
        memcpy(&before, &b, sizeof(T));
        memcpy(&after, &nb, sizeof(T));
        r.value_before = double(before);
        r.value_after = double(after);
        r.applied = ok ? 1 : 0;
        r.reserved = 0;
        rec[i] = r;
    }
}

}  // namespace

void launch_flip_rows(int fmt, void* X, int64_t rows, int64_t cols, const int32_t* col, const int32_t* bit,
                      const int32_t* dir, vabft_fault_record* rec, cudaStream_t s) {
    const unsigned grid = unsigned((rows + 255) / 256);
    if (fmt == VABFT_FP64)
        flip_rows_kernel<double, unsigned long long><<<grid, 256, 0, s>>>(static_cast<double*>(X), rows, cols, col,
                                                                          bit, dir, rec);
    else if (fmt == VABFT_FP32)
        flip_rows_kernel<float, unsigned int><<<grid, 256, 0, s>>>(static_cast<float*>(X), rows, cols, col, bit, dir,
                                                                   rec);
    else
        fail(VABFT_INVALID_ARGUMENT, "flip rows: FP32 / FP64 only");
    check_cuda(cudaGetLastError(), "flip rows launch");
}

}  // namespace vabft_dev
