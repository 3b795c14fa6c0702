// Shared device helpers: typed element loads, compensated (Neumaier) sums,
// strategy-ordered reductions, the V-ABFT threshold formula and warp
// utilities. All floating-point arithmetic that must match the reference
// bit for bit uses the explicit _rn intrinsics (never contracted to FMA).
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "vabft_c.h"

namespace vabft_dev {

template <int F>
struct Elem;
template <>
struct Elem<VABFT_BF16> {
    using T = uint16_t;
    static __device__ __forceinline__ float f(T x) { return __uint_as_float(uint32_t(x) << 16); }
    static __device__ __forceinline__ double d(T x) { return double(f(x)); }
};
template <>
struct Elem<VABFT_FP16> {
    using T = uint16_t;
    static __device__ __forceinline__ float f(T x) { return __half2float(__ushort_as_half(x)); }
    static __device__ __forceinline__ double d(T x) { return double(f(x)); }
};
template <>
struct Elem<VABFT_FP32> {
    using T = float;
    static __device__ __forceinline__ float f(T x) { return x; }
    static __device__ __forceinline__ double d(T x) { return double(x); }
};
template <>
struct Elem<VABFT_FP64> {
    using T = double;
    static __device__ __forceinline__ float f(T x) { return float(x); }
    static __device__ __forceinline__ double d(T x) { return x; }
};

// --------------------------------------------------- Neumaier (stats.cpp)
struct Neu {
    double s = 0.0, c = 0.0;
    // Branch-free (selects, same operations and order as stats.cpp:16-21):
    // in an unrolled run of adds the scheduler can issue the next element's
    // s + x while this element's compensation is still in flight (the
    // sequential-fallback rows of wide_tail_kernel; DESIGN "tie rows").
    __device__ __forceinline__ void add(double x) {
        const double t = __dadd_rn(s, x);
        const bool ge = fabs(s) >= fabs(x);
        const double hi = ge ? s : x, lo = ge ? x : s;
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(hi, t), lo));
        s = t;
    }
    // Merge two compensated partials (TwoSum of the heads, sum of tails).
    __device__ __forceinline__ void merge(double os, double oc) {
        const double t = __dadd_rn(s, os);
        double e;
        if (fabs(s) >= fabs(os))
            e = __dadd_rn(__dsub_rn(s, t), os);
        else
            e = __dadd_rn(__dsub_rn(os, t), s);
        c = __dadd_rn(__dadd_rn(c, oc), e);
        s = t;
    }
};

// Error-free transformation: s + e == a + b exactly (Knuth's TwoSum).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// A row sum held as an error-free cascade (s, c): hi = fl(s + c) equals the
// reference's sequential Neumaier fl(sum + comp) (stats.cpp:12-24) unless the
// exact sum lies within 8 (K u)^2 sum|x| of a rounding midpoint — both
// results are within (K u)^2 sum|x| of the exact sum (sabs: an upper bound of
// sum|x|). False when that cannot be ruled out (the caller reruns the loop).
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

template <class T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
    return __shfl_xor_sync(0xffffffffu, v, m);
}

// Warp-wide compensated sum; every lane receives the merged (s, c).
__device__ __forceinline__ Neu warp_merge(Neu n) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const double os = shfl_xor(n.s, m), oc = shfl_xor(n.c, m);
        // Merge in a fixed lane order so all lanes agree bit for bit.
        const int lane = threadIdx.x & 31;
        Neu a, b;
        if ((lane & m) == 0) { a = n; b.s = os; b.c = oc; }
        else { a.s = os; a.c = oc; b = n; }
        a.merge(b.s, b.c);
        n = a;
    }
    return n;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = fmax(v, shfl_xor(v, m));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = fmin(v, shfl_xor(v, m));
    return v;
}

// row_stats finish (stats.cpp:26-31): mean clamped into [min, max],
// var_bound = max(0, (max-mean)(mean-min)).
__device__ __forceinline__ void stats_finish(const Neu& n, double mx, double mn, int64_t len,
                                             double* mean, double* var_bound) {
    double m = __ddiv_rn(__dadd_rn(n.s, n.c), double(len));
    if (m < mn) m = mn;
    else if (mx < m) m = mx;
    const double vb = __dmul_rn(__dsub_rn(mx, m), __dsub_rn(m, mn));
    *mean = m;
    *var_bound = vb > 0.0 ? vb : 0.0;
}

// threshold_row (threshold_vabft.cpp:28-42) in the written evaluation order.
__device__ __forceinline__ double vabft_threshold_total(double mean, double var_bound,
                                                        double s_abs_mean, double s_mean_sq,
                                                        double s_var, int64_t n, double e_max,
                                                        double c_sigma) {
    const double nn = double(n);
    const double sa = sqrt(var_bound);
    const double det = __dmul_rn(__dmul_rn(nn, fabs(mean)), s_abs_mean);
    const double inner = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(nn, mean), mean), s_var),
                                   __dmul_rn(__dmul_rn(__dmul_rn(nn, nn), var_bound), s_mean_sq));
    const double var23 = __dmul_rn(c_sigma, sqrt(inner));
    const double var4 = __dmul_rn(__dmul_rn(__dmul_rn(c_sigma, sqrt(nn)), sa), sqrt(s_var));
    return __dmul_rn(e_max, __dadd_rn(__dadd_rn(det, var23), var4));
}

// aabft_sigma (threshold_aabft.cpp:31-36) times the confidence multiplier.
__device__ __forceinline__ double aabft_total(int64_t n, int t, double y, double conf) {
    const double nn = double(n);
    const double poly = __dadd_rn(__dmul_rn(__dmul_rn(nn, __dadd_rn(nn, 1.0)), __dadd_rn(nn, 0.5)),
                                  __dmul_rn(2.0, nn));
    const double sig = __dmul_rn(__dmul_rn(sqrt(__ddiv_rn(poly, 24.0)), ldexp(1.0, -t)), y);
    return __dmul_rn(conf, sig);
}

// Non-negative doubles order like their bit patterns: atomicMax on u64.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

}  // namespace vabft_dev
