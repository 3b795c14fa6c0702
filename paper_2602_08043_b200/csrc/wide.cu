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
// DGEMM mapping: 128 x 128 x 16 CTA tiles, 256 threads (8 warps as 4 x 2),
// an 8 x 8 register tile per thread (rows wm*32 + 8j + 2ty + {0,1}, columns
// wn*64 + 16j + 2tx + {0,1}) so that every shared-memory fragment read is a
// conflict-free 16-byte access; a 4-stage cp.async ring (A rows padded to 18
// doubles). Per k pair: 16 LDS.128 for 128 DFMA — the FP64 pipe (64 DFMA /
// clk / SM) is the bound, not shared memory.
#include <algorithm>
#include <type_traits>

#include "devcommon.cuh"
#include "internal.hpp"
#include "numerics.cuh"
#include "ptx.cuh"
#include "reducers.cuh"

namespace vabft_dev {

namespace {

constexpr int kDBM = 128, kDBN = 128, kDBK = 16, kDStages = 4, kDThreads = 256;
constexpr int kALd = kDBK + 2;          // doubles per staged A row (16-byte aligned, conflict-free)
constexpr int kAStage = kDBM * kALd;    // doubles
constexpr int kBStage = kDBK * kDBN;
constexpr int kStage = kAStage + kBStage;
constexpr int kCLd = kDBN + 1;          // epilogue staging stride: row walks are conflict-free
constexpr size_t kDSmem = sizeof(double) * size_t(kDStages) * kStage;
static_assert(sizeof(double) * kDBM * kCLd <= kDSmem, "epilogue staging reuses the operand ring");

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

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

    auto load_stage = [&](int64_t kt, int slot) {
        double* As = sm + size_t(slot) * kStage;
        double* Bs = As + kAStage;
        const int64_t k0 = kt * kDBK;
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // A: 128 rows x 8 chunks of 2 doubles
            const int c = tid + q * kDThreads;
            const int r = c >> 3, part = c & 7;
            const int64_t gr = m0 + r, gk = k0 + part * 2;
            const bool ok = gr < p.M && gk < p.K;
            cp_async16(smem_u32(As + r * kALd + part * 2), ok ? p.A + gr * p.K + gk : p.A, ok);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // B: 16 rows x 64 chunks
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

// A side of the wide fused path: ONE pass over A, then a per-row combine
// (inside the verify tail). It runs after the GEMM on the same stream: run
// beside the GEMM on a second stream it was starved of memory bandwidth and
// finished late (measured), so the serial order is the faster one.
//
// wide_apart_kernel: a warp takes 32 rows x one 128-column block (coalesced
// tile loads through shared memory; lane = row walks the block in order) and
// writes, per (block, row):
//  - the NativeBlocked(128) checksum partials sum_j T(br_j) T(a_j) in the
//    working type W (checksum.cpp:103-146);
//  - an error-free cascaded sum (TwoSum: s, c) of the row segment in FP64,
//    sum |a|, and max / min (stats.cpp:9-32).
// wide_acombine_kernel (thread per row): checksum partials in block order;
// the (s, c) pairs merged with TwoSum. With hi = fl(s + c), |s + c - S| <=
// (K u)^2 sum|x| for the exact row sum S, and the reference's sequential
// Neumaier sum + comp obeys the same bound — both round to fl(S) unless S lies
// within 8 (K u)^2 sum|x| of a rounding midpoint. That is checked per row;
// such rows (and non-finite ones) rerun the reference's loop (counted as
// slow-stats rows), so the mean is bit-identical in every case.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// hi = fl(s + c) equals the reference's fl(sum + comp) unless the exact sum
// lies within 8 (K u)^2 sum|x| of a rounding midpoint (see above).
__device__ __forceinline__ bool exact_sum_safe(double s, double c, double sabs, int64_t K, double* hi_out) {
    double hi, lo;
    two_sum(s, c, hi, lo);
    const double ku = double(K) * 1.1102230246251565e-16;  // K u, u = 2^-53
    const double margin = 8.0 * ku * ku * sabs * 1.0000001;
    if (!(isfinite(hi) && isfinite(lo) && isfinite(margin))) return false;
    const double nb = nextafter(hi, (lo > 0.0) ? INFINITY : -INFINITY);  // the midpoint on lo's side
    if (!(fabs(lo) + margin < fabs(__dsub_rn(nb, hi)) * 0.5)) return false;
    *hi_out = hi;
    return true;
}

template <class W>
struct APart {  // per (block, row) partial arrays, each [nb][ld]
    W *p1, *p2;
    double *s, *c, *sabs, *mx, *mn;
};

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

template <int F, class W>
__global__ void __launch_bounds__(128) wide_apart_kernel(const typename Elem<F>::T* __restrict__ A, int64_t M,
                                                         int64_t K, const double* __restrict__ br1,
                                                         const double* __restrict__ br2, APart<W> out, int64_t ld) {
    using T = typename Elem<F>::T;
    __shared__ T tile[4][32][33];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t(blockIdx.x) * 4 + w) * 32, b = blockIdx.y;
    if (r0 >= M) return;
    W p1 = W(0), p2 = W(0);
    double s = 0.0, c = 0.0, sabs = 0.0;
    T mx = T(-INFINITY), mn = T(INFINITY);
    for (int q = 0; q < 4; ++q) {
        const int64_t col0 = b * 128 + q * 32;
        if (col0 >= K) break;
        const int64_t col = col0 + lane;
        T v[32];  // all 32 row loads in flight before the first smem store
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            const int64_t r = r0 + rr;
            v[rr] = (r < M && col < K) ? __ldcs(A + r * K + col) : T(0);
        }
        const W w1l = col < K ? W(br1[col]) : W(0), w2l = col < K ? W(br2[col]) : W(0);
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) tile[w][rr][lane] = v[rr];
        __syncwarp();
        const int cmax = int(K - col0 < 32 ? K - col0 : 32);
        for (int jj = 0; jj < cmax; ++jj) {
            const T e = tile[w][lane][jj];
            const W x = W(e);
            p1 = radd(p1, rmul(__shfl_sync(0xffffffffu, w1l, jj), x));
            p2 = radd(p2, rmul(__shfl_sync(0xffffffffu, w2l, jj), x));
            const double xd = double(e);
            double t, err;
            two_sum(s, xd, t, err);
            s = t;
            c = __dadd_rn(c, err);
            sabs = __dadd_rn(sabs, fabs(xd));
            mx = mx < e ? e : mx;  // NaN-free rows: identical to fmax / fmin
            mn = e < mn ? e : mn;
        }
        __syncwarp();
    }
    const int64_t row = r0 + lane;
    if (row < M) {
        const size_t o = size_t(b) * size_t(ld) + size_t(row);
        out.p1[o] = p1;
        out.p2[o] = p2;
        out.s[o] = s;
        out.c[o] = c;
        out.sabs[o] = sabs;
        out.mx[o] = double(mx);
        out.mn[o] = double(mn);
    }
}

// Per-row combine of the A-side partials: stats (mean, var_bound, max, min)
// and the row checksums; see the comment above.
template <int F, class W>
__device__ __forceinline__ void acombine_row(const typename Elem<F>::T* __restrict__ A, int64_t K, const APart<W>& in,
                                             int64_t ld, int qfmt, int64_t i, int64_t* counts, double& mean,
                                             double& vb, double& mx, double& mn, double& c1, double& c2) {
    const int64_t nb = (K + 127) / 128;
    W t1 = W(0), t2 = W(0);
    double s = 0.0, c = 0.0, sabs = 0.0;
    mx = -INFINITY;
    mn = INFINITY;
#pragma unroll 4
    for (int64_t b = 0; b < nb; ++b) {
        const size_t o = size_t(b) * size_t(ld) + size_t(i);
        t1 = radd(t1, in.p1[o]);
        t2 = radd(t2, in.p2[o]);
        double t, err;
        two_sum(s, in.s[o], t, err);
        s = t;
        c = __dadd_rn(__dadd_rn(c, in.c[o]), err);
        sabs = __dadd_rn(sabs, in.sabs[o]);
        mx = mx < in.mx[o] ? in.mx[o] : mx;
        mn = in.mn[o] < mn ? in.mn[o] : mn;
    }
    Neu ns;
    if (exact_sum_safe(s, c, sabs, K, &ns.s)) {
        // ns.s = fl(sum + comp) of the reference
    } else {
        if (counts) atomicAdd(reinterpret_cast<unsigned long long*>(counts + VABFT_COUNT_SLOW_STATS), 1ull);
        const typename Elem<F>::T* arow = A + i * K;
        for (int64_t j = 0; j < K; ++j) ns.add(double(arow[j]));  // the reference's loop (stats.cpp:12-24)
    }
    stats_finish(ns, mx, mn, K, &mean, &vb);
    c1 = double(t1);
    c2 = double(t2);
    if (qfmt == VABFT_FP32) {  // offline FP32: the checksum rounded to the input format (a no-op for W = float)
        c1 = double(float(c1));
        c2 = double(float(c2));
    }
}

template <int F, class W>
__global__ void __launch_bounds__(256) wide_acombine_kernel(const typename Elem<F>::T* __restrict__ A, int64_t M,
                                                            int64_t K, APart<W> in, int64_t ld, int qfmt, double* mean,
                                                            double* vb, double* mx_out, double* mn_out, double* cr1,
                                                            double* cr2, int64_t* counts) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= M) return;
    double m, v, mx, mn, c1, c2;
    acombine_row<F, W>(A, K, in, ld, qfmt, i, counts, m, v, mx, mn, c1, c2);
    mean[i] = m;
    vb[i] = v;
    mx_out[i] = mx;
    mn_out[i] = mn;
    cr1[i] = c1;
    cr2[i] = c2;
}

template <class W>
__device__ __forceinline__ W load_part(const void* p, size_t o) {
    return static_cast<const W*>(p)[o];
}

// Verify tail, a warp per row: the C-row partials (blocked:128 order) and,
// with a.apart set (threshold methods without a global dependency), the
// A-side partials are combined across the lanes (lane = 128-column block,
// ordered sums through shuffles, TwoSum merges in a butterfly); lane 0 then
// evaluates the threshold, D1 / D2, the strict compare, NaN rule,
// localization and the optional correction. Counters are aggregated per CTA.
template <int F>
__global__ void __launch_bounds__(256) wide_tail_kernel(const WideTail a) {
    using W = std::conditional_t<F == VABFT_FP64, double, float>;
    using T = typename Elem<F>::T;
    __shared__ unsigned long long cnt[6];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 6) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (i < a.M) {
        // C r1 / C r2: block partials in order
        W r1 = W(0), r2 = W(0);
        for (int64_t g = 0; g < a.nblk; g += 32) {
            const int64_t b = g + lane;
            W q1 = W(0), q2 = W(0);
            if (b < a.nblk) {
                const size_t o = size_t(b) * size_t(a.ld) + size_t(i);
                q1 = load_part<W>(a.part1, o);
                q2 = load_part<W>(a.part2, o);
            }
            const int n = a.nblk - g < 32 ? int(a.nblk - g) : 32;
            for (int l = 0; l < n; ++l) {
                r1 = radd(r1, __shfl_sync(0xffffffffu, q1, l));
                r2 = radd(r2, __shfl_sync(0xffffffffu, q2, l));
            }
        }
        double mean_i = 0.0, vb_i = 0.0, c1 = 0.0, c2 = 0.0;
        if (a.apart) {
            const int64_t nbk = (a.K + 127) / 128;
            const APart<W> in = apart_view<W>(const_cast<void*>(a.apart), nbk, a.ld);
            W t1 = W(0), t2 = W(0);
            double s = 0.0, c = 0.0, sabs = 0.0, mx = -INFINITY, mn = INFINITY;
            for (int64_t g = 0; g < nbk; g += 32) {
                const int64_t b = g + lane;
                W q1 = W(0), q2 = W(0);
                if (b < nbk) {
                    const size_t o = size_t(b) * size_t(a.ld) + size_t(i);
                    q1 = in.p1[o];
                    q2 = in.p2[o];
                    double t, err;
                    two_sum(s, in.s[o], t, err);
                    s = t;
                    c = __dadd_rn(__dadd_rn(c, in.c[o]), err);
                    sabs = __dadd_rn(sabs, in.sabs[o]);
                    mx = mx < in.mx[o] ? in.mx[o] : mx;
                    mn = in.mn[o] < mn ? in.mn[o] : mn;
                }
                const int n = nbk - g < 32 ? int(nbk - g) : 32;
                for (int l = 0; l < n; ++l) {
                    t1 = radd(t1, __shfl_sync(0xffffffffu, q1, l));
                    t2 = radd(t2, __shfl_sync(0xffffffffu, q2, l));
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const double so = __shfl_xor_sync(0xffffffffu, s, o), co = __shfl_xor_sync(0xffffffffu, c, o);
                double t, err;
                two_sum(s, so, t, err);
                s = t;
                c = __dadd_rn(__dadd_rn(c, co), err);
                sabs = __dadd_rn(sabs, __shfl_xor_sync(0xffffffffu, sabs, o));
                const double mxo = __shfl_xor_sync(0xffffffffu, mx, o), mno = __shfl_xor_sync(0xffffffffu, mn, o);
                mx = mx < mxo ? mxo : mx;
                mn = mno < mn ? mno : mn;
            }
            Neu ns;
            const bool safe = __shfl_sync(0xffffffffu, exact_sum_safe(s, c, sabs, a.K, &ns.s) ? 1 : 0, 0) != 0;
            if (!safe) {
                // the reference's sequential loop (stats.cpp:12-24) — rows whose exact
                // sum sits on a rounding midpoint (measured ~1 in 4096 for FP64 N(0,1)
                // rows at K = 4096, ~1 in 10^5 FP32 rows). The warp stages the row
                // 256 elements at a time in its own shared-memory slice (8 coalesced
                // loads per lane in flight), then lane 0 reads 32 elements per batch
                // with 16-byte LDS ahead of the chain and runs the adds back to back.
                // (Broadcasting each element by a shuffle put a SHFL, a branch and
                // the conversion on the chain: 63 cycles per element, 131 us for
                // one K = 4096 row.)
                if (lane == 0 && a.counts) atomicAdd(&cnt[VABFT_COUNT_SLOW_STATS], 1ull);
                constexpr int kChunk = 256;
                __shared__ __align__(16) T stage[8][kChunk];
                T* st = stage[threadIdx.x >> 5];
                const T* arow = static_cast<const T*>(a.A) + i * a.K;
                ns = Neu{};
                for (int64_t j0 = 0; j0 < a.K; j0 += kChunk) {
                    const int n = a.K - j0 < kChunk ? int(a.K - j0) : kChunk;  // warp-uniform
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < kChunk / 32; ++r) {
                        const int q = r * 32 + lane;
                        if (q < n) st[q] = arow[j0 + q];
                    }
                    __syncwarp();
                    if (lane == 0) {
                        int q = 0;
                        for (; q + 32 <= n; q += 32) {
                            using V = std::conditional_t<sizeof(T) == 8, double2, float4>;
                            constexpr int kPer = 16 / sizeof(T);
                            T xs[32];
#pragma unroll
                            for (int u = 0; u < 32 / kPer; ++u) {
                                const V w = reinterpret_cast<const V*>(st + q)[u];
                                if constexpr (sizeof(T) == 8) {
                                    xs[2 * u] = w.x;
                                    xs[2 * u + 1] = w.y;
                                } else {
                                    xs[4 * u] = w.x;
                                    xs[4 * u + 1] = w.y;
                                    xs[4 * u + 2] = w.z;
                                    xs[4 * u + 3] = w.w;
                                }
                            }
#pragma unroll
                            for (int l = 0; l < 32; ++l) ns.add(double(xs[l]));
                        }
                        for (; q < n; ++q) ns.add(double(st[q]));
                    }
                }
            }
            if (lane == 0) {
                stats_finish(ns, mx, mn, a.K, &mean_i, &vb_i);
                c1 = double(t1);
                c2 = double(t2);
                if (a.qfmt == VABFT_FP32) {  // offline FP32: rounded to the input format (no-op for W = float)
                    c1 = double(float(c1));
                    c2 = double(float(c2));
                }
            }
        } else if (lane == 0) {
            mean_i = a.mean[i];
            vb_i = a.vb[i];
            c1 = a.cr1[i];
            c2 = a.cr2[i];
        }
        if (lane == 0) {
            bool det = false, located = false, isnan_row = false, corrected = false;
            double t;
            if (a.method == 0) {
                t = vabft_threshold_total(mean_i, vb_i, a.bsum[0], a.bsum[1], a.bsum[2], a.N, a.e_max, a.c_sigma);
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
            if (a.counts) {
                atomicAdd(&cnt[VABFT_COUNT_ROWS], 1ull);
                if (det) atomicAdd(&cnt[VABFT_COUNT_DETECTED], 1ull);
                if (located) atomicAdd(&cnt[VABFT_COUNT_LOCATED], 1ull);
                if (isnan_row) atomicAdd(&cnt[VABFT_COUNT_NAN], 1ull);
                if (corrected) atomicAdd(&cnt[VABFT_COUNT_CORRECTED], 1ull);
            }
        }
    }
    __syncthreads();
    if (a.counts && threadIdx.x < 6 && cnt[threadIdx.x])
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + threadIdx.x), cnt[threadIdx.x]);
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
    const unsigned grid = unsigned((t.M + 7) / 8);
    if (t.fmt == VABFT_FP64) wide_tail_kernel<VABFT_FP64><<<grid, 256, 0, stream>>>(t);
    else wide_tail_kernel<VABFT_FP32><<<grid, 256, 0, stream>>>(t);  // 8 rows (warps) per CTA
    check_cuda(cudaGetLastError(), "wide tail launch");
}

void launch_wide_aside(int fmt, int64_t M, int64_t K, const void* A, const double* br1, const double* br2, int qfmt,
                       double* mean, double* vb, double* mx, double* mn, double* cr1, double* cr2, void* apart,
                       int64_t ld, int64_t* counts, bool combine, cudaStream_t stream) {
    const int64_t nb = (K + 127) / 128;
    const dim3 grid_p(unsigned((M + 127) / 128), unsigned(nb));
    const unsigned grid_c = unsigned((M + 255) / 256);
    auto run = [&](auto tag, auto wtag) {
        using T = decltype(tag);
        using W = decltype(wtag);
        constexpr int F = sizeof(T) == 8 ? VABFT_FP64 : VABFT_FP32;
        const APart<W> part = apart_view<W>(apart, nb, ld);
        wide_apart_kernel<F, W><<<grid_p, 128, 0, stream>>>(static_cast<const T*>(A), M, K, br1, br2, part, ld);
        if (combine)
            wide_acombine_kernel<F, W><<<grid_c, 256, 0, stream>>>(static_cast<const T*>(A), M, K, part, ld, qfmt,
                                                                   mean, vb, mx, mn, cr1, cr2, counts);
    };
    if (fmt == VABFT_FP64) run(double{}, double{});
    else if (fmt == VABFT_FP32) run(float{}, float{});
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
