// Host-only C-ABI helpers: precision descriptors, quantize, e_max models,
// threshold formulas, localize and the canonical bit encodings. These are
// the scalar pieces of the reference API that callers use around the device
// entry points; each follows the cited reference lines exactly (the file is
// compiled with -ffp-contract=off like the reference).
#include <cmath>
#include <cstring>
#include <limits>

#include "guard.hpp"
#include "internal.hpp"

using namespace vabft_dev;

namespace {

int fmt_t(int f) { return f == VABFT_BF16 ? 8 : f == VABFT_FP16 ? 11 : f == VABFT_FP32 ? 24 : 53; }
int fmt_emin(int f) { return f == VABFT_FP16 ? -14 : f == VABFT_FP64 ? -1022 : -126; }
double fmt_max(int f) {
    switch (f) {
        case VABFT_BF16: return 0x1.FEp127;
        case VABFT_FP16: return 65504.0;
        case VABFT_FP32: return double(std::numeric_limits<float>::max());
        default: return std::numeric_limits<double>::max();
    }
}
void check_fmt(int f) {
    if (f < VABFT_BF16 || f > VABFT_FP64) fail(VABFT_INVALID_ARGUMENT, "bad format");
}

uint64_t dbits(double x) { uint64_t b; std::memcpy(&b, &x, 8); return b; }
double bitsd(uint64_t b) { double x; std::memcpy(&x, &b, 8); return x; }

// f16 canonical encoding (faults.cpp:25-62)
uint16_t f16_encode(double v) {
    if (std::isnan(v)) {
        const uint64_t b = dbits(v);
        uint16_t m = uint16_t((b >> 42) & 0x3FF);
        if (m == 0) m = 0x200;
        return uint16_t(((b >> 48) & 0x8000) | 0x7C00 | m);
    }
    const uint16_t sign = std::signbit(v) ? 0x8000 : 0;
    if (std::isinf(v)) return sign | 0x7C00;
    const double a = std::fabs(v);
    if (a == 0.0) return sign;
    const int e = std::ilogb(a);
    if (e < -14) return uint16_t(sign | uint16_t(std::llrint(std::ldexp(a, 24))));
    if (e > 15) return sign | 0x7C00;
    const uint16_t mant = uint16_t(std::llrint((std::ldexp(a, -e) - 1.0) * 1024.0));
    return uint16_t(sign | uint16_t((e + 15) << 10) | mant);
}
double f16_decode(uint16_t bits) {
    const bool neg = bits & 0x8000;
    const int e = (bits >> 10) & 0x1F;
    const uint16_t m = bits & 0x3FF;
    double v;
    if (e == 31) {
        if (m == 0) v = std::numeric_limits<double>::infinity();
        else return bitsd(0x7FF0000000000000ull | (uint64_t(neg) << 63) | (uint64_t(m) << 42));
    } else if (e == 0) {
        v = std::ldexp(double(m), -24);
    } else {
        v = std::ldexp(1.0 + double(m) / 1024.0, e - 15);
    }
    return neg ? -v : v;
}

}  // namespace

// PrecisionSpec::bf16/fp16/fp32/fp64 (precision.cpp:44-82)
extern "C" vabft_status vabft_precision_default(int32_t format, vabft_precision* out) {
    return guarded([&] {
        check_fmt(format);
        if (!out) fail(VABFT_INVALID_ARGUMENT, "null out");
        vabft_precision p{};
        p.format = format;
        p.mantissa_bits = fmt_t(format);
        p.unit_roundoff = std::ldexp(1.0, -p.mantissa_bits);
        p.overflow = 0;
        p.accumulation.block_len = 128;
        switch (format) {
            case VABFT_BF16:
                p.accumulation.kind = VABFT_ACCUM_FP32_ROUND_OUTPUT;
                p.emax_kind = 0; p.emax_offset = 8e-3;
                break;
            case VABFT_FP16:
                p.accumulation.kind = VABFT_ACCUM_FP32_ROUND_OUTPUT;
                p.emax_kind = 0; p.emax_offset = 1e-3;
                break;
            case VABFT_FP32:
                p.accumulation.kind = VABFT_ACCUM_PAIRWISE;
                p.emax_kind = 1; p.emax_scale = 5.0e-9; p.emax_offset = 1.2e-7;
                break;
            default:
                p.accumulation.kind = VABFT_ACCUM_PAIRWISE;
                p.emax_kind = 1; p.emax_scale = 1.0e-17; p.emax_offset = 2.5e-16;
                break;
        }
        *out = p;
    });
}

// quantize (precision.cpp:129-159)
extern "C" vabft_status vabft_quantize(double x, const vabft_precision* fmt, double* out) {
    return guarded([&] {
        if (!fmt || !out) fail(VABFT_INVALID_ARGUMENT, "null argument");
        check_fmt(fmt->format);
        if (!std::isfinite(x)) fail(VABFT_DOMAIN_ERROR, "quantize: non-finite input");
        const int f = fmt->format;
        if (f == VABFT_FP64 || x == 0.0) { *out = x; return; }
        const int t = fmt_t(f), emin = fmt_emin(f), drop = 53 - t;
        const uint64_t b = dbits(x);
        const int biased = int((b >> 52) & 0x7FF);
        double y;
        if (biased != 0 && biased - 1023 >= emin) {
            const uint64_t low = (uint64_t(1) << drop) - 1;
            const uint64_t lsb = (b >> drop) & 1u;
            y = bitsd((b + (low >> 1) + lsb) & ~low);
        } else {
            const double q = std::ldexp(1.0, emin - t + 1);
            y = std::nearbyint(x / q) * q;
        }
        if (std::fabs(y) > fmt_max(f)) {
            if (fmt->overflow) fail(VABFT_RANGE_ERROR, "quantize: overflow beyond max finite value");
            y = std::copysign(fmt_max(f), x);
        }
        *out = y;
    });
}

// resolve_e_max / EmaxModel::resolve (threshold_vabft.cpp:49-52, precision.cpp:39-42)
extern "C" vabft_status vabft_resolve_e_max(const vabft_precision* spec, int64_t dim, double* out) {
    return guarded([&] {
        if (!spec || !out) fail(VABFT_INVALID_ARGUMENT, "null argument");
        if (dim < 1) fail(VABFT_INVALID_ARGUMENT, "resolve_e_max: dim must be >= 1");
        *out = spec->emax_kind == 0 ? spec->emax_offset
                                    : spec->emax_scale * std::sqrt(double(dim)) + spec->emax_offset;
    });
}

// aabft_sigma (threshold_aabft.cpp:31-36)
extern "C" vabft_status vabft_aabft_sigma(int64_t n, int32_t mantissa_bits, double y, double* out) {
    return guarded([&] {
        if (!out) fail(VABFT_INVALID_ARGUMENT, "null out");
        if (n < 1) fail(VABFT_INVALID_ARGUMENT, "aabft_sigma: n must be >= 1");
        const double nn = double(n);
        const double poly = nn * (nn + 1.0) * (nn + 0.5) + 2.0 * nn;
        *out = std::sqrt(poly / 24.0) * std::ldexp(1.0, -mantissa_bits) * y;
    });
}

// threshold_row (threshold_vabft.cpp:28-42)
extern "C" vabft_status vabft_threshold_row(const double a[4], const double b[3], int64_t n,
                                            double e_max, double c_sigma, double out[4]) {
    return guarded([&] {
        if (!a || !b || !out) fail(VABFT_INVALID_ARGUMENT, "null argument");
        if (n < 1) fail(VABFT_INVALID_ARGUMENT, "threshold_row: n must be >= 1");
        const double nn = double(n), mu = a[0], sa = std::sqrt(a[3]);
        const double det = nn * std::fabs(mu) * b[0];
        const double var23 = c_sigma * std::sqrt(nn * mu * mu * b[2] + nn * nn * a[3] * b[1]);
        const double var4 = c_sigma * std::sqrt(nn) * sa * std::sqrt(b[2]);
        out[0] = det;
        out[1] = var23;
        out[2] = var4;
        out[3] = e_max * (det + var23 + var4);
    });
}

// localize (detect.cpp:9-17); out-of-range int64 conversion as x86-64 cvttsd2si.
extern "C" int32_t vabft_localize(double d1, double d2, int64_t n_cols, int64_t* j, double* residual) {
    if (d1 == 0.0 || !std::isfinite(d1) || !std::isfinite(d2)) return 0;
    const double pos = d2 / d1 - 1.0;
    if (!std::isfinite(pos)) return 0;
    const double nearest = std::nearbyint(pos);
    if (residual) *residual = std::fabs(pos - nearest);
    int64_t q = (nearest >= 0x1.0p63 || nearest < -0x1.0p63) ? INT64_MIN : int64_t(nearest);
    if (q < 0) q = 0;
    if (q > n_cols - 1) q = n_cols - 1;
    if (j) *j = q;
    return 1;
}

// encode_bits / decode_bits (faults.cpp:66-87)
extern "C" vabft_status vabft_encode_bits(double value, int32_t format, uint64_t* out) {
    return guarded([&] {
        if (!out) fail(VABFT_INVALID_ARGUMENT, "null out");
        switch (format) {
            case VABFT_BF16: { const float f = float(value); uint32_t b; std::memcpy(&b, &f, 4); *out = b >> 16; break; }
            case VABFT_FP16: *out = f16_encode(value); break;
            case VABFT_FP32: { const float f = float(value); uint32_t b; std::memcpy(&b, &f, 4); *out = b; break; }
            case VABFT_FP64: *out = dbits(value); break;
            default: fail(VABFT_INVALID_ARGUMENT, "encode_bits: bad format");
        }
    });
}

extern "C" vabft_status vabft_decode_bits(uint64_t bits, int32_t format, double* out) {
    return guarded([&] {
        if (!out) fail(VABFT_INVALID_ARGUMENT, "null out");
        switch (format) {
            case VABFT_BF16: { const uint32_t b = uint32_t(bits) << 16; float f; std::memcpy(&f, &b, 4); *out = double(f); break; }
            case VABFT_FP16: *out = f16_decode(uint16_t(bits)); break;
            case VABFT_FP32: { const uint32_t b = uint32_t(bits); float f; std::memcpy(&f, &b, 4); *out = double(f); break; }
            case VABFT_FP64: *out = bitsd(bits); break;
            default: fail(VABFT_INVALID_ARGUMENT, "decode_bits: bad format");
        }
    });
}
