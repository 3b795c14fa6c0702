// Device-side restatement of the reference's scalar numerics: output
// quantization (RNE, subnormals kept, saturate to max finite), canonical
// bit encodings for fault injection, and the decision rules of verify().
//
//   quantize          proj/src/precision.cpp:129-159
//   saturation rule   proj/src/precision.cpp:303-312
//   encode/decode     proj/src/faults.cpp:25-87
//   localize/verify   proj/src/detect.cpp:9-55
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "vabft_c.h"

namespace vabft_dev {

constexpr float kBf16MaxF = 3.38953138925153547590e+38f;  // 0x1.FEp127
constexpr float kFp16MaxF = 65504.0f;

// Round an FP32 value to the 16-bit output format with the reference's
// Saturate policy; returns the raw 16-bit pattern.
template <int kFmt>
__device__ __forceinline__ uint16_t quantize16_bits(float v) {
    if constexpr (kFmt == VABFT_BF16) {
        __nv_bfloat16 h = __float2bfloat16_rn(v);
        uint16_t b = __bfloat16_as_ushort(h);
        if ((b & 0x7FFFu) == 0x7F80u) b = static_cast<uint16_t>((b & 0x8000u) | 0x7F7Fu);
        return b;
    } else {
        __half h = __float2half_rn(v);
        uint16_t b = __half_as_ushort(h);
        if ((b & 0x7FFFu) == 0x7C00u) b = static_cast<uint16_t>((b & 0x8000u) | 0x7BFFu);
        return b;
    }
}

// quantize (precision.cpp:129-159) of an FP64 value to a 16-bit format: one
// RNE rounding from double (no intermediate float), saturating.
template <int kFmt>
__device__ __forceinline__ uint16_t quantize16_bits_d(double v) {
    if constexpr (kFmt == VABFT_BF16) {
        uint16_t b = __bfloat16_as_ushort(__double2bfloat16(v));
        if ((b & 0x7FFFu) == 0x7F80u) b = static_cast<uint16_t>((b & 0x8000u) | 0x7F7Fu);
        return b;
    } else {
        uint16_t b = __half_as_ushort(__double2half(v));
        if ((b & 0x7FFFu) == 0x7C00u) b = static_cast<uint16_t>((b & 0x8000u) | 0x7BFFu);
        return b;
    }
}

template <int kFmt>
__device__ __forceinline__ float bits16_to_float(uint16_t b) {
    if constexpr (kFmt == VABFT_BF16) {
        return __uint_as_float(static_cast<uint32_t>(b) << 16);
    } else {
        return __half2float(__ushort_as_half(b));
    }
}

// Non-finite accumulator handling of run_gemm: +-max_finite(out format).
template <int kFmt>
__device__ __forceinline__ float saturate_accum(float v) {
    if (isfinite(v)) return v;
    const float mx = (kFmt == VABFT_BF16) ? kBf16MaxF : (kFmt == VABFT_FP16 ? kFp16MaxF : 3.40282346638528859812e+38f);
    return copysignf(mx, v);
}

// Bit eligibility for the flip directions (faults.cpp:91-102).
__device__ __forceinline__ bool bit_eligible(uint64_t bits, int bit, int dir) {
    const uint64_t b = (bits >> bit) & 1ull;
    if (dir == VABFT_FLIP_SET0TO1) return b == 0;
    if (dir == VABFT_FLIP_SET1TO0) return b == 1;
    return true;
}

// localize(): j = clamp(int64(nearbyint(d2/d1 - 1)), 0, n-1). The int64
// conversion follows x86-64 cvttsd2si (out-of-range -> INT64_MIN), which is
// what the reference binary does for |pos| >= 2^63.
__device__ __forceinline__ bool localize_dev(double d1, double d2, int64_t n_cols, int64_t* j,
                                             double* residual) {
    if (d1 == 0.0 || !isfinite(d1) || !isfinite(d2)) return false;
    const double pos = d2 / d1 - 1.0;
    if (!isfinite(pos)) return false;
    const double nearest = rint(pos);
    *residual = fabs(pos - nearest);
    int64_t q;
    if (nearest >= 9223372036854775808.0 || nearest < -9223372036854775808.0)
        q = INT64_MIN;
    else
        q = static_cast<int64_t>(nearest);
    if (q < 0) q = 0;
    if (q > n_cols - 1) q = n_cols - 1;
    *j = q;
    return true;
}

}  // namespace vabft_dev
