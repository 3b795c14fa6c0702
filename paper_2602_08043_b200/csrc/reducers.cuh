// Order-exact reductions in a working type T (float or double), one per
// AccumKind of the reference (proj/src/precision.cpp:344-381, 220-275):
//   SEQUENTIAL / FP32_ROUND_OUTPUT : acc += term, left to right
//   BLOCKED(bl)                    : part += term; every bl terms tot += part
//   PAIRWISE                       : balanced tree split at n/2, evaluated
//                                    left to right with an explicit stack and
//                                    a host-computed merge schedule
// Every add/multiply is an explicit round-to-nearest intrinsic, so nothing is
// contracted into an FMA.
#pragma once

#include <cstdint>

#include "vabft_c.h"

namespace vabft_dev {

__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }

// Runtime-selected reducer (kind is warp-uniform).
template <class T>
struct Reducer {
    static constexpr int kMaxDepth = 40;
    int kind;
    int64_t bl;
    const uint8_t* sched;  // merge counts after each leaf (PAIRWISE only)
    int64_t q = 0;         // leaves consumed
    T acc = T(0), part = T(0);
    T st[kMaxDepth];
    int sp = 0;

    __device__ __forceinline__ Reducer(int kind_, int64_t bl_, const uint8_t* sched_)
        : kind(kind_), bl(bl_ > 0 ? bl_ : 128), sched(sched_) {}

    __device__ __forceinline__ void push(T v, int64_t len) {
        if (kind == VABFT_ACCUM_PAIRWISE) {
            int c = sched[q];
            while (c-- > 0) v = radd(st[--sp], v);
            st[sp++] = v;
        } else if (kind == VABFT_ACCUM_BLOCKED) {
            part = radd(part, v);
            if ((q + 1) % bl == 0 || q + 1 == len) {
                acc = radd(acc, part);
                part = T(0);
            }
        } else {
            acc = radd(acc, v);
        }
        ++q;
    }
    __device__ __forceinline__ T result() const {
        if (kind == VABFT_ACCUM_PAIRWISE) return q > 0 ? st[0] : T(0);
        return acc;
    }
};

}  // namespace vabft_dev
