// vabft_cpp.hpp — C++ drop-in for the reference API of the V-ABFT hot path
// (namespace vabft, proj/include/vabft/*.hpp of arxiv/paper_2602_08043),
// implemented on the B200 C-ABI (vabft_c.h, libvabft_b200.so).
//
// Same names, argument meaning, value semantics and exception types as the
// reference. Matrix keeps the reference's host FP64 storage; every compute
// entry point (GEMM + checksums, row sums, row statistics, thresholds,
// verification) runs on the GPU through the C-ABI — the EXACT engine, which
// reproduces the reference bit for bit — with FP64 <-> native conversion at
// the boundary. Host code here is glue only: validation, O(1)-per-row
// formulas the reference computes on scalars (threshold_row, localize,
// aabft_sigma, quantize of a single value), the Philox / ziggurat streams
// (which must match the reference draw for draw) and the host-side fault
// placement of inject(). No CPU fallback: without a usable sm_100 device the
// device entry points throw vabft::device_error.
//
// Header-only; link with -lvabft_b200 -lcudart. C++20 (std::span).
//
// Reference interfaces (file:line of proj/include/vabft/):
//   precision.hpp:10-156  Format, AccumKind, AccumStrategy, EmaxModel,
//                         PrecisionSpec, quantize, Matrix, gemm_emulated*,
//                         accumulates_in_float, reduce_in_precision, reduce
//   checksum.hpp:10-59    VerifyMode, checksum_precision_for, ChecksumVectors,
//                         EncodedProduct, encode_and_multiply, row_sums
//   stats.hpp:11-21       RowStats, row_stats
//   threshold_vabft.hpp:10-47  VabftParams, ThresholdBreakdown,
//                         precompute_b_stats, BStatsSummary, threshold_row,
//                         resolve_e_max, vabft_thresholds
//   threshold_aabft.hpp:14-36  AabftParams, aabft_sigma, AabftThresholds,
//                         aabft_threshold, aabft_computed_y
//   detect.hpp:14-46      RowVerdict, DetectOptions, localize, verify, correct
//   rng.hpp:9-49          Philox;  distribution.hpp:9-33 Distribution,
//                         random_matrix
//   faults.hpp:15-85      FaultTarget, FlipDirection, FaultSpec,
//                         InjectionRecord, encode_bits, decode_bits, inject,
//                         CampaignConfig, CampaignOutcome, ThresholdFn,
//                         injection_campaign
#ifndef VABFT_CPP_HPP_
#define VABFT_CPP_HPP_

#include <cuda_runtime_api.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vabft_c.h"

namespace vabft {

// Device / driver failure (VABFT_CUDA_ERROR): the reference has no device.
class device_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

namespace detail {

[[noreturn]] inline void raise(vabft_status st) {
    const std::string msg = vabft_last_error();
    switch (st) {
        case VABFT_INVALID_ARGUMENT:
        case VABFT_UNSUPPORTED: throw std::invalid_argument(msg);
        case VABFT_DOMAIN_ERROR: throw std::domain_error(msg);
        case VABFT_RANGE_ERROR: throw std::range_error(msg);
        case VABFT_OUT_OF_RANGE: throw std::out_of_range(msg);
        case VABFT_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw device_error(msg);
    }
}
inline void check(vabft_status st) {
    if (st != VABFT_OK) raise(st);
}
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw device_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device allocation with synchronous transfers on the legacy stream.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t bytes) : n_(bytes) {
        if (bytes) cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
    }
    DeviceBuffer(const void* host, size_t bytes) : DeviceBuffer(bytes) { upload(host, bytes); }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            if (p_) cudaFree(p_);
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
        }
        return *this;
    }
    void* get() const { return p_; }
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    void upload(const void* src, size_t bytes) {
        if (bytes) cuda_check(cudaMemcpy(p_, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    void download(void* dst, size_t bytes) const {
        if (bytes) cuda_check(cudaMemcpy(dst, p_, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }
    template <class T>
    std::vector<T> to_vector(size_t count) const {
        std::vector<T> v(count);
        download(v.data(), count * sizeof(T));
        return v;
    }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

}  // namespace detail

// ------------------------------------------------------------ precision.hpp
enum class Format : uint8_t { BF16 = 0, FP16 = 1, FP32 = 2, FP64 = 3 };

inline const char* format_name(Format f) {
    switch (f) {
        case Format::BF16: return "bf16";
        case Format::FP16: return "fp16";
        case Format::FP32: return "fp32";
        case Format::FP64: return "fp64";
    }
    return "?";
}
inline Format format_from_name(const std::string& name) {
    if (name == "bf16") return Format::BF16;
    if (name == "fp16") return Format::FP16;
    if (name == "fp32") return Format::FP32;
    if (name == "fp64") return Format::FP64;
    throw std::invalid_argument("unknown precision: " + name);
}

enum class AccumKind : uint8_t { Fp32AccumRoundOutput, NativeSequential, NativeBlocked, NativePairwise };

struct AccumStrategy {
    AccumKind kind = AccumKind::NativeSequential;
    int64_t block_len = 128;
    std::string describe() const {
        switch (kind) {
            case AccumKind::Fp32AccumRoundOutput: return "fp32-accum";
            case AccumKind::NativeSequential: return "sequential";
            case AccumKind::NativeBlocked: return "blocked:" + std::to_string(block_len);
            case AccumKind::NativePairwise: return "pairwise";
        }
        return "?";
    }
};

struct EmaxModel {
    enum class Kind : uint8_t { Constant, SqrtScaled };
    Kind kind = Kind::Constant;
    double scale = 0.0;
    double offset = 0.0;
    static EmaxModel constant(double value) { return {Kind::Constant, 0.0, value}; }
    static EmaxModel sqrt_scaled(double scale, double offset) { return {Kind::SqrtScaled, scale, offset}; }
    double resolve(int64_t dim) const {
        return kind == Kind::Constant ? offset : scale * std::sqrt(double(dim)) + offset;
    }
};

enum class OverflowPolicy : uint8_t { Saturate, Error };

struct PrecisionSpec {
    Format format = Format::FP64;
    int mantissa_bits = 53;
    double unit_roundoff = 0x1.0p-53;
    AccumStrategy accumulation{AccumKind::NativePairwise, 128};
    EmaxModel e_max_model = EmaxModel::constant(0x1.0p-52);
    OverflowPolicy overflow = OverflowPolicy::Saturate;

    static PrecisionSpec from_c(const vabft_precision& c) {
        PrecisionSpec s;
        s.format = Format(c.format);
        s.mantissa_bits = c.mantissa_bits;
        s.unit_roundoff = c.unit_roundoff;
        s.accumulation = {AccumKind(c.accumulation.kind), c.accumulation.block_len};
        s.e_max_model = {EmaxModel::Kind(c.emax_kind), c.emax_scale, c.emax_offset};
        s.overflow = OverflowPolicy(c.overflow);
        return s;
    }
    vabft_precision to_c() const {
        vabft_precision c{};
        c.format = int32_t(format);
        c.mantissa_bits = mantissa_bits;
        c.unit_roundoff = unit_roundoff;
        c.accumulation.kind = int32_t(accumulation.kind);
        c.accumulation.block_len = accumulation.block_len;
        c.emax_kind = int32_t(e_max_model.kind);
        c.overflow = int32_t(overflow);
        c.emax_scale = e_max_model.scale;
        c.emax_offset = e_max_model.offset;
        return c;
    }
    static PrecisionSpec of(Format f) {
        vabft_precision c;
        detail::check(vabft_precision_default(int32_t(f), &c));
        return from_c(c);
    }
    static PrecisionSpec bf16() { return of(Format::BF16); }
    static PrecisionSpec fp16() { return of(Format::FP16); }
    static PrecisionSpec fp32() { return of(Format::FP32); }
    static PrecisionSpec fp64() { return of(Format::FP64); }

    int min_normal_exponent() const {
        switch (format) {
            case Format::BF16: return -126;
            case Format::FP16: return -14;
            case Format::FP32: return -126;
            case Format::FP64: return -1022;
        }
        return 0;
    }
    double max_finite() const {
        switch (format) {
            case Format::BF16: return 0x1.FEp127;
            case Format::FP16: return 65504.0;
            case Format::FP32: return double(std::numeric_limits<float>::max());
            case Format::FP64: return std::numeric_limits<double>::max();
        }
        return 0.0;
    }
    double min_subnormal() const { return std::ldexp(1.0, min_normal_exponent() - mantissa_bits + 1); }
    int bit_width() const {
        return format == Format::FP64 ? 64 : format == Format::FP32 ? 32 : 16;
    }
    const char* name() const { return format_name(format); }
    PrecisionSpec with_accumulation(AccumStrategy s) const {
        PrecisionSpec r = *this;
        r.accumulation = s;
        return r;
    }
    PrecisionSpec with_e_max(EmaxModel m) const {
        PrecisionSpec r = *this;
        r.e_max_model = m;
        return r;
    }
};

inline double quantize(double x, const PrecisionSpec& fmt) {
    const vabft_precision c = fmt.to_c();
    double out;
    detail::check(vabft_quantize(x, &c, &out));
    return out;
}

class Matrix {
public:
    Matrix() = default;
    Matrix(int64_t rows, int64_t cols, PrecisionSpec fmt)
        : rows_(rows), cols_(cols), fmt_(fmt) {
        if (rows < 1 || cols < 1) throw std::invalid_argument("Matrix: dims must be >= 1");
        data_.assign(size_t(rows * cols), 0.0);
    }
    static Matrix from_values(int64_t rows, int64_t cols, std::span<const double> values, PrecisionSpec fmt,
                              bool quantize_values = true) {
        if (int64_t(values.size()) != rows * cols) throw std::invalid_argument("Matrix::from_values: size mismatch");
        Matrix m(rows, cols, fmt);
        for (size_t idx = 0; idx < values.size(); ++idx) {
            const double q = quantize(values[idx], fmt);
            if (!quantize_values && q != values[idx])
                throw std::invalid_argument("Matrix::from_values: value not representable in format");
            m.data_[idx] = q;
        }
        return m;
    }
    static Matrix identity(int64_t n, PrecisionSpec fmt) {
        Matrix m(n, n, fmt);
        for (int64_t i = 0; i < n; ++i) m.data_[size_t(i * n + i)] = 1.0;
        return m;
    }
    int64_t rows() const { return rows_; }
    int64_t cols() const { return cols_; }
    const PrecisionSpec& format() const { return fmt_; }
    double operator()(int64_t i, int64_t j) const { return data_[size_t(i * cols_ + j)]; }
    double at(int64_t i, int64_t j) const {
        if (i < 0 || i >= rows_ || j < 0 || j >= cols_) throw std::out_of_range("Matrix::at: index out of range");
        return data_[size_t(i * cols_ + j)];
    }
    void set(int64_t i, int64_t j, double v) {
        if (i < 0 || i >= rows_ || j < 0 || j >= cols_) throw std::out_of_range("Matrix::set: index out of range");
        data_[size_t(i * cols_ + j)] = quantize(v, fmt_);
    }
    std::span<const double> values() const { return data_; }
    std::span<const double> row(int64_t i) const { return {data_.data() + i * cols_, size_t(cols_)}; }
    void set_raw(int64_t i, int64_t j, double v) { data_[size_t(i * cols_ + j)] = v; }
    bool same_bits(const Matrix& o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ &&
               std::memcmp(data_.data(), o.data_.data(), data_.size() * sizeof(double)) == 0;
    }
    double* raw_data() { return data_.data(); }  // B200 extension: bulk access

private:
    int64_t rows_ = 0, cols_ = 0;
    PrecisionSpec fmt_{};
    std::vector<double> data_;
};

struct GemmResult {
    Matrix c;
    Matrix accum;
};

inline bool accumulates_in_float(const PrecisionSpec& spec) {
    return spec.accumulation.kind == AccumKind::Fp32AccumRoundOutput || spec.format == Format::FP32;
}

// ------------------------------------------------- faults.hpp (bit codecs)
inline uint64_t encode_bits(double value, Format f) {
    uint64_t out;
    detail::check(vabft_encode_bits(value, int32_t(f), &out));
    return out;
}
inline double decode_bits(uint64_t bits, Format f) {
    double out;
    detail::check(vabft_decode_bits(bits, int32_t(f), &out));
    return out;
}

namespace detail {

inline size_t native_size(Format f) { return f == Format::FP64 ? 8 : f == Format::FP32 ? 4 : 2; }

// FP64 host storage -> native device storage of format f (the canonical
// encodings of encode_bits, so injected bit patterns survive the trip).
inline std::vector<uint8_t> to_native(std::span<const double> v, Format f) {
    std::vector<uint8_t> out(v.size() * native_size(f));
    for (size_t i = 0; i < v.size(); ++i) {
        switch (f) {
            case Format::BF16:
            case Format::FP16: {
                const uint16_t b = uint16_t(f == Format::BF16 ? [&] {
                    const float x = float(v[i]);
                    uint32_t u;
                    std::memcpy(&u, &x, 4);
                    return u >> 16;
                }() : uint32_t(encode_bits(v[i], f)));
                std::memcpy(out.data() + 2 * i, &b, 2);
                break;
            }
            case Format::FP32: {
                const float x = float(v[i]);
                std::memcpy(out.data() + 4 * i, &x, 4);
                break;
            }
            case Format::FP64: std::memcpy(out.data() + 8 * i, &v[i], 8); break;
        }
    }
    return out;
}

inline std::vector<double> from_native(const std::vector<uint8_t>& b, size_t count, Format f) {
    std::vector<double> out(count);
    for (size_t i = 0; i < count; ++i) {
        switch (f) {
            case Format::BF16: {
                uint16_t h;
                std::memcpy(&h, b.data() + 2 * i, 2);
                const uint32_t u = uint32_t(h) << 16;
                float x;
                std::memcpy(&x, &u, 4);
                out[i] = double(x);
                break;
            }
            case Format::FP16: {
                uint16_t h;
                std::memcpy(&h, b.data() + 2 * i, 2);
                out[i] = decode_bits(h, Format::FP16);
                break;
            }
            case Format::FP32: {
                float x;
                std::memcpy(&x, b.data() + 4 * i, 4);
                out[i] = double(x);
                break;
            }
            case Format::FP64: std::memcpy(&out[i], b.data() + 8 * i, 8); break;
        }
    }
    return out;
}

inline DeviceBuffer upload(const Matrix& m, Format storage) {
    const std::vector<uint8_t> b = to_native(m.values(), storage);
    return DeviceBuffer(b.data(), b.size());
}
inline DeviceBuffer upload(const Matrix& m) { return upload(m, m.format().format); }

inline Matrix download(const DeviceBuffer& d, int64_t rows, int64_t cols, Format storage, const PrecisionSpec& spec) {
    const size_t n = size_t(rows * cols);
    std::vector<uint8_t> b(n * native_size(storage));
    d.download(b.data(), b.size());
    const std::vector<double> v = from_native(b, n, storage);
    Matrix m(rows, cols, spec);
    std::memcpy(m.raw_data(), v.data(), n * sizeof(double));
    return m;
}

inline DeviceBuffer upload_doubles(std::span<const double> v) { return DeviceBuffer(v.data(), v.size() * 8); }

}  // namespace detail

// gemm_emulated_with_accum (precision.cpp:320-338) on the EXACT engine.
inline GemmResult gemm_emulated_with_accum(const Matrix& a, const Matrix& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("gemm_emulated: inner dimensions disagree");
    if (a.format().format != b.format().format) throw std::invalid_argument("gemm_emulated: operand formats disagree");
    const PrecisionSpec& spec = a.format();
    const int64_t m = a.rows(), n = b.cols(), k = a.cols();
    const bool in_float = accumulates_in_float(spec);
    const PrecisionSpec accfmt = in_float ? PrecisionSpec::fp32() : PrecisionSpec::fp64();
    const vabft_precision cs = spec.to_c();
    detail::DeviceBuffer dA = detail::upload(a), dB = detail::upload(b);
    detail::DeviceBuffer dC(size_t(m * n) * detail::native_size(spec.format));
    detail::DeviceBuffer dAcc(size_t(m * n) * (in_float ? 4 : 8));
    size_t ws = 0;
    detail::check(vabft_encode_workspace_size(m, n, k, &cs, &ws));
    detail::DeviceBuffer dW(ws);
    detail::check(vabft_encode_and_multiply(&cs, VABFT_OFFLINE, VABFT_ENGINE_EXACT, m, n, k, dA.get(), dB.get(),
                                            dC.get(), dAcc.get(), nullptr, nullptr, nullptr, nullptr, dW.get(), ws,
                                            nullptr));
    detail::cuda_check(cudaDeviceSynchronize(), "gemm_emulated");
    return {detail::download(dC, m, n, spec.format, spec),
            detail::download(dAcc, m, n, in_float ? Format::FP32 : Format::FP64, accfmt)};
}
inline Matrix gemm_emulated(const Matrix& a, const Matrix& b) { return gemm_emulated_with_accum(a, b).c; }

// reduce_in_precision / reduce (precision.cpp:344-400): a strategy-ordered
// reduction of one term vector = the plain row sum of a 1 x n matrix.
inline double reduce_in_precision(std::span<const double> terms, const PrecisionSpec& spec) {
    if (terms.empty()) return 0.0;
    const vabft_precision cs = spec.to_c();
    detail::DeviceBuffer d = detail::upload_doubles(terms), r1(8), r2(8);
    detail::check(vabft_row_sums(&cs, VABFT_FP64, 1, int64_t(terms.size()), d.get(), r1.as<double>(),
                                 r2.as<double>(), nullptr));
    return r1.to_vector<double>(1)[0];
}
inline double reduce(std::span<const double> terms, AccumStrategy strat) {
    return reduce_in_precision(terms, PrecisionSpec::fp64().with_accumulation(strat));
}
inline float reduce(std::span<const float> terms, AccumStrategy strat) {
    std::vector<double> d(terms.begin(), terms.end());
    return float(reduce_in_precision(d, PrecisionSpec::fp32().with_accumulation(strat)));
}

// ------------------------------------------------------------- checksum.hpp
enum class VerifyMode : uint8_t { Offline, Online };

inline const char* verify_mode_name(VerifyMode m) { return m == VerifyMode::Offline ? "offline" : "online"; }
inline VerifyMode verify_mode_from_name(const std::string& name) {
    if (name == "offline") return VerifyMode::Offline;
    if (name == "online") return VerifyMode::Online;
    throw std::invalid_argument("unknown mode: " + name);
}

// checksum_precision_for (checksum.cpp:18-24)
inline PrecisionSpec checksum_precision_for(const PrecisionSpec& fmt, VerifyMode mode) {
    if (mode == VerifyMode::Offline) return fmt;
    const PrecisionSpec base = fmt.format == Format::FP64 ? PrecisionSpec::fp64() : PrecisionSpec::fp32();
    return base.with_accumulation(fmt.accumulation);
}

struct ChecksumVectors {
    int64_t n = 0;
    static double weight(int64_t k) { return double(k + 1); }
    static ChecksumVectors make(int64_t n, const PrecisionSpec& accum_precision) {
        if (n < 1) throw std::invalid_argument("ChecksumVectors: length must be >= 1");
        const int t = accumulates_in_float(accum_precision) ? 24 : 53;
        if (n > (int64_t(1) << t))
            throw std::invalid_argument(
                "ChecksumVectors: position weights exceed the exact-integer range of the checksum precision");
        return ChecksumVectors{n};
    }
    std::vector<double> ones() const { return std::vector<double>(size_t(n), 1.0); }
    std::vector<double> weights() const {
        std::vector<double> w(static_cast<size_t>(n));
        for (int64_t k = 0; k < n; ++k) w[size_t(k)] = weight(k);
        return w;
    }
};

struct EncodedProduct {
    Matrix c;
    std::vector<double> row_check1, row_check2, col_check1, col_check2;
    PrecisionSpec checksum_precision;
    VerifyMode mode = VerifyMode::Offline;
    Matrix c_accum;
    const Matrix& verification_source() const { return mode == VerifyMode::Online ? c_accum : c; }
};

// Engine of the reference-signature entry points (encode_and_multiply and
// what builds on it: verify of its product, calibrate, injection_campaign,
// verify_files). Exact (default): the order-exact SIMT kernels, bit-identical
// to the reference. Tensor: the B200 fast path — tcgen05 for BF16 / FP16
// (FP32 accumulator in the tensor core's order), tcgen05 kind::tf32 3xTF32 for
// FP32, SIMT DFMA for FP64 — with checksums and row sums in the accumulator's
// working type in NativeBlocked(128) order (the fused kernels' checksum
// precision), so verify() on its product compares like the fused path.
namespace b200 {
enum class Engine { Exact = VABFT_ENGINE_EXACT, Tensor = VABFT_ENGINE_TENSOR };
inline std::atomic<int>& engine_slot() {
    static std::atomic<int> e{VABFT_ENGINE_EXACT};
    return e;
}
inline void set_engine(Engine e) { engine_slot().store(int(e)); }
inline Engine engine() { return Engine(engine_slot().load()); }
}  // namespace b200

// encode_and_multiply (checksum.cpp:103-158): C, C_accum and all four
// checksum vectors from one device call (EXACT engine: bit-identical; see
// b200::set_engine for the fast path).
inline EncodedProduct encode_and_multiply(const Matrix& a, const Matrix& b, VerifyMode mode = VerifyMode::Offline) {
    if (a.cols() != b.rows()) throw std::invalid_argument("gemm_emulated: inner dimensions disagree");
    if (a.format().format != b.format().format) throw std::invalid_argument("gemm_emulated: operand formats disagree");
    const PrecisionSpec& spec = a.format();
    const int64_t m = a.rows(), n = b.cols(), k = a.cols();
    const bool in_float = accumulates_in_float(spec);
    const vabft_precision cs = spec.to_c();
    detail::DeviceBuffer dA = detail::upload(a), dB = detail::upload(b);
    detail::DeviceBuffer dC(size_t(m * n) * detail::native_size(spec.format));
    detail::DeviceBuffer dAcc(size_t(m * n) * (in_float ? 4 : 8));
    detail::DeviceBuffer rc1(size_t(m) * 8), rc2(size_t(m) * 8), cc1(size_t(n) * 8), cc2(size_t(n) * 8);
    size_t ws = 0;
    detail::check(vabft_encode_workspace_size(m, n, k, &cs, &ws));
    detail::DeviceBuffer dW(ws);
    const int eng = b200::engine_slot().load();
    detail::check(vabft_encode_and_multiply(&cs, mode == VerifyMode::Online ? VABFT_ONLINE : VABFT_OFFLINE, eng, m,
                                            n, k, dA.get(), dB.get(), dC.get(), dAcc.get(), rc1.as<double>(),
                                            rc2.as<double>(), cc1.as<double>(), cc2.as<double>(), dW.get(), ws,
                                            nullptr));
    detail::cuda_check(cudaDeviceSynchronize(), "encode_and_multiply");
    EncodedProduct out;
    out.c = detail::download(dC, m, n, spec.format, spec);
    out.c_accum = detail::download(dAcc, m, n, in_float ? Format::FP32 : Format::FP64,
                                   in_float ? PrecisionSpec::fp32() : PrecisionSpec::fp64());
    out.row_check1 = rc1.to_vector<double>(size_t(m));
    out.row_check2 = rc2.to_vector<double>(size_t(m));
    out.col_check1 = cc1.to_vector<double>(size_t(n));
    out.col_check2 = cc2.to_vector<double>(size_t(n));
    out.checksum_precision = checksum_precision_for(spec, mode);
    if (eng == VABFT_ENGINE_TENSOR)  // the fused kernels' checksum precision
        out.checksum_precision = (spec.format == Format::FP64 ? PrecisionSpec::fp64() : PrecisionSpec::fp32())
                                     .with_accumulation({AccumKind::NativeBlocked, 128});
    out.mode = mode;
    return out;
}

// row_sums (checksum.cpp:160-187)
inline std::pair<std::vector<double>, std::vector<double>> row_sums(const Matrix& c, const PrecisionSpec& sum_precision) {
    const vabft_precision cs = sum_precision.to_c();
    detail::DeviceBuffer d = detail::upload(c), r1(size_t(c.rows()) * 8), r2(size_t(c.rows()) * 8);
    detail::check(vabft_row_sums(&cs, int32_t(c.format().format), c.rows(), c.cols(), d.get(), r1.as<double>(),
                                 r2.as<double>(), nullptr));
    return {r1.to_vector<double>(size_t(c.rows())), r2.to_vector<double>(size_t(c.rows()))};
}

// ---------------------------------------------------------------- stats.hpp
struct RowStats {
    double mean = 0.0, max = 0.0, min = 0.0, var_bound = 0.0;
    int64_t n = 0;
};

namespace detail {
inline std::vector<RowStats> row_stats_device(Format f, int64_t rows, int64_t cols, const void* d) {
    DeviceBuffer mean(size_t(rows) * 8), mx(size_t(rows) * 8), mn(size_t(rows) * 8), vb(size_t(rows) * 8);
    check(vabft_row_stats(int32_t(f), rows, cols, d, mean.as<double>(), mx.as<double>(), mn.as<double>(),
                          vb.as<double>(), nullptr));
    const auto a = mean.to_vector<double>(size_t(rows)), b = mx.to_vector<double>(size_t(rows)),
               c = mn.to_vector<double>(size_t(rows)), e = vb.to_vector<double>(size_t(rows));
    std::vector<RowStats> out(static_cast<size_t>(rows));
    for (size_t i = 0; i < out.size(); ++i) out[i] = {a[i], b[i], c[i], e[i], cols};
    return out;
}
}  // namespace detail

// row_stats (stats.cpp:9-32)
inline RowStats row_stats(std::span<const double> values) {
    if (values.empty()) throw std::invalid_argument("row_stats: empty row");
    detail::DeviceBuffer d = detail::upload_doubles(values);
    return detail::row_stats_device(Format::FP64, 1, int64_t(values.size()), d.get())[0];
}

// ------------------------------------------------------ threshold_vabft.hpp
struct VabftParams {
    double e_max = 0.0;
    double c_sigma = 2.5;
};
struct ThresholdBreakdown {
    double det = 0.0, var23 = 0.0, var4 = 0.0, total = 0.0;
};

// precompute_b_stats (threshold_vabft.cpp:8-13): every row of B on the device
inline std::vector<RowStats> precompute_b_stats(const Matrix& b) {
    detail::DeviceBuffer d = detail::upload(b);
    return detail::row_stats_device(b.format().format, b.rows(), b.cols(), d.get());
}

struct BStatsSummary {
    double sum_abs_mean = 0.0, sum_mean_sq = 0.0, sum_var = 0.0;
    int64_t k_len = 0;
    // BStatsSummary::from (threshold_vabft.cpp:15-26): three sequential FP64
    // sums over K given statistics (host glue over caller data)
    static BStatsSummary from(std::span<const RowStats> b_stats) {
        if (b_stats.empty()) throw std::invalid_argument("BStatsSummary: empty stats");
        BStatsSummary s;
        s.k_len = int64_t(b_stats.size());
        for (const RowStats& r : b_stats) {
            if (r.var_bound < 0.0) throw std::logic_error("BStatsSummary: negative variance bound");
            s.sum_abs_mean += std::abs(r.mean);
            s.sum_mean_sq += r.mean * r.mean;
            s.sum_var += r.var_bound;
        }
        return s;
    }
};

// threshold_row (threshold_vabft.cpp:28-47)
inline ThresholdBreakdown threshold_row(const RowStats& a, const BStatsSummary& b, int64_t n, const VabftParams& p) {
    const double as[4] = {a.mean, a.max, a.min, a.var_bound};
    const double bs[3] = {b.sum_abs_mean, b.sum_mean_sq, b.sum_var};
    double out[4];
    detail::check(vabft_threshold_row(as, bs, n, p.e_max, p.c_sigma, out));
    return {out[0], out[1], out[2], out[3]};
}
inline ThresholdBreakdown threshold_row(const RowStats& a, std::span<const RowStats> b_stats, int64_t n,
                                        const VabftParams& p) {
    return threshold_row(a, BStatsSummary::from(b_stats), n, p);
}

// resolve_e_max (threshold_vabft.cpp:49-52)
inline double resolve_e_max(const PrecisionSpec& spec, int64_t dim) {
    const vabft_precision c = spec.to_c();
    double out;
    detail::check(vabft_resolve_e_max(&c, dim, &out));
    return out;
}

// vabft_thresholds (threshold_vabft.cpp:54-61): one device call (A and B
// statistics, B summary, T_i) when A and B agree on format and inner size;
// otherwise composed from the row statistics like the reference.
inline std::vector<double> vabft_thresholds(const Matrix& a, const Matrix& b, const VabftParams& params) {
    if (a.cols() == b.rows() && a.format().format == b.format().format) {
        detail::DeviceBuffer dA = detail::upload(a), dB = detail::upload(b), T(size_t(a.rows()) * 8);
        detail::check(vabft_vabft_thresholds(int32_t(a.format().format), a.rows(), b.cols(), a.cols(), dA.get(),
                                             dB.get(), params.e_max, params.c_sigma, T.as<double>(), nullptr,
                                             nullptr));
        return T.to_vector<double>(size_t(a.rows()));
    }
    const BStatsSummary summary = BStatsSummary::from(precompute_b_stats(b));
    detail::DeviceBuffer dA = detail::upload(a);
    const std::vector<RowStats> as = detail::row_stats_device(a.format().format, a.rows(), a.cols(), dA.get());
    std::vector<double> out(static_cast<size_t>(a.rows()));
    for (size_t i = 0; i < out.size(); ++i) out[i] = threshold_row(as[i], summary, b.cols(), params).total;
    return out;
}

// ------------------------------------------------------ threshold_aabft.hpp
struct AabftParams {
    int mantissa_bits = 53;
    std::optional<double> fixed_y = 21.0;
    double confidence_multiplier = 3.0;
    // AabftParams::for_format (threshold_aabft.cpp:8-29)
    static AabftParams for_format(Format f) {
        AabftParams p;
        switch (f) {
            case Format::FP64: p.mantissa_bits = 53; p.fixed_y = 21.0; break;
            case Format::FP32: p.mantissa_bits = 23; p.fixed_y = 21.0; break;
            case Format::BF16: p.mantissa_bits = 8; p.fixed_y.reset(); break;
            case Format::FP16: p.mantissa_bits = 11; p.fixed_y.reset(); break;
        }
        return p;
    }
    bool computed_y() const { return !fixed_y.has_value(); }
};

inline double aabft_sigma(int64_t n, int mantissa_bits, double y) {
    double out;
    detail::check(vabft_aabft_sigma(n, mantissa_bits, y, &out));
    return out;
}

struct AabftThresholds {
    std::vector<double> per_row;
    double y_used = 0.0;
    bool degenerate = false;
};

// aabft_computed_y (threshold_aabft.cpp:38-48): max|A| from A's row extrema
// and the plain sequential FP64 row sums of B, both on the device.
inline double aabft_computed_y(const Matrix& a, const Matrix& b) {
    detail::DeviceBuffer dA = detail::upload(a);
    double max_a = 0.0;
    for (const RowStats& r : detail::row_stats_device(a.format().format, a.rows(), a.cols(), dA.get()))
        max_a = std::max(max_a, std::max(std::abs(r.max), std::abs(r.min)));
    const PrecisionSpec seq = PrecisionSpec::fp64().with_accumulation({AccumKind::NativeSequential, 128});
    const std::vector<double> sums = row_sums(b, seq).first;
    double max_row_sum = 0.0;
    for (const double s : sums) max_row_sum = std::max(max_row_sum, std::abs(s));
    return max_a * max_row_sum;
}

// aabft_threshold (threshold_aabft.cpp:50-60)
inline AabftThresholds aabft_threshold(const Matrix& a, const Matrix& b, const AabftParams& params) {
    if (a.cols() != b.rows()) throw std::invalid_argument("aabft_threshold: inner dimensions disagree");
    const double y = params.fixed_y ? *params.fixed_y : aabft_computed_y(a, b);
    AabftThresholds out;
    out.y_used = y;
    out.degenerate = (y == 0.0);
    const double t = params.confidence_multiplier * aabft_sigma(a.cols(), params.mantissa_bits, y);
    out.per_row.assign(size_t(a.rows()), t);
    return out;
}

// --------------------------------------------------------------- detect.hpp
struct RowVerdict {
    int64_t row = 0;
    double diff1 = 0.0, diff2 = 0.0, threshold = 0.0;
    bool detected = false;
    std::optional<int64_t> location;
    std::optional<double> correction;
    double localization_residual = 0.0;
};

struct DetectOptions {
    double localization_floor_scale = 1e-3;
    double residual_margin = 0.1;
};

// localize (detect.cpp:9-17)
inline std::optional<std::pair<int64_t, double>> localize(double d1, double d2, int64_t n_cols) {
    int64_t j;
    double r;
    if (!vabft_localize(d1, d2, n_cols, &j, &r)) return std::nullopt;
    return std::make_pair(j, r);
}

// verify (detect.cpp:19-55): row sums of the verification source in the
// checksum precision, D1 / D2, strict compare, NaN rule, localization — on
// the device.
inline std::vector<RowVerdict> verify(const EncodedProduct& prod, std::span<const double> thresholds,
                                      const DetectOptions& opts = {}) {
    const Matrix& src = prod.verification_source();
    const int64_t m = src.rows(), n = src.cols();
    if (int64_t(thresholds.size()) != m)
        throw std::invalid_argument("verify: thresholds length must equal row count");
    const vabft_precision cs = prod.checksum_precision.to_c();
    detail::DeviceBuffer dS = detail::upload(src), rc1 = detail::upload_doubles(prod.row_check1),
                         rc2 = detail::upload_doubles(prod.row_check2), dT = detail::upload_doubles(thresholds);
    detail::DeviceBuffer d1(size_t(m) * 8), d2(size_t(m) * 8), det{static_cast<size_t>(m)}, loc(size_t(m) * 8),
        res(size_t(m) * 8);
    vabft_verdicts v{d1.as<double>(), d2.as<double>(), det.as<uint8_t>(), loc.as<int64_t>(), res.as<double>(),
                     nullptr, nullptr};
    detail::check(vabft_verify(&cs, int32_t(src.format().format), m, n, dS.get(), rc1.as<double>(), rc2.as<double>(),
                               dT.as<double>(), opts.localization_floor_scale, v, nullptr, nullptr));
    const auto D1 = d1.to_vector<double>(size_t(m)), D2 = d2.to_vector<double>(size_t(m));
    const auto DET = det.to_vector<uint8_t>(size_t(m));
    const auto LOC = loc.to_vector<int64_t>(size_t(m));
    const auto RES = res.to_vector<double>(size_t(m));
    std::vector<RowVerdict> out(static_cast<size_t>(m));
    for (size_t i = 0; i < out.size(); ++i) {
        RowVerdict& r = out[i];
        r.row = int64_t(i);
        r.diff1 = D1[i];
        r.diff2 = D2[i];
        r.threshold = thresholds[i];
        r.detected = DET[i] != 0;
        if (LOC[i] >= 0) {
            r.location = LOC[i];
            r.localization_residual = RES[i];
            r.correction = D1[i];
        }
    }
    return out;
}

// correct (detect.cpp:57-64)
inline Matrix correct(const Matrix& c, const RowVerdict& verdict) {
    if (!verdict.detected || !verdict.location || !verdict.correction)
        throw std::invalid_argument("correct: verdict has no usable location");
    Matrix out = c;
    out.set(verdict.row, *verdict.location, c(verdict.row, *verdict.location) - *verdict.correction);
    return out;
}

// ------------------------------------------------------------------ rng.hpp
// Philox4x32-10 counter-based generator (rng.cpp): counter = (block index,
// stream), key = seed; draws in the reference's exact order.
class Philox {
public:
    explicit Philox(uint64_t seed, uint64_t stream = 0) : seed_(seed), stream_(stream) {}

    static std::array<uint32_t, 4> block(const std::array<uint32_t, 4>& counter, const std::array<uint32_t, 2>& key) {
        std::array<uint32_t, 4> c = counter;
        std::array<uint32_t, 2> k = key;
        for (int r = 0; r < 10; ++r) {
            if (r) {
                k[0] += 0x9E3779B9u;
                k[1] += 0xBB67AE85u;
            }
            const uint64_t p0 = uint64_t(0xD2511F53u) * c[0];
            const uint64_t p1 = uint64_t(0xCD9E8D57u) * c[2];
            c = {uint32_t(p1 >> 32) ^ c[1] ^ k[0], uint32_t(p1), uint32_t(p0 >> 32) ^ c[3] ^ k[1], uint32_t(p0)};
        }
        return c;
    }
    uint32_t next_u32() {
        if (pos_ == 4) {
            buf_ = block({uint32_t(idx_), uint32_t(idx_ >> 32), uint32_t(stream_), uint32_t(stream_ >> 32)},
                         {uint32_t(seed_), uint32_t(seed_ >> 32)});
            ++idx_;
            pos_ = 0;
        }
        return buf_[size_t(pos_++)];
    }
    uint64_t next_u64() {
        const uint64_t lo = next_u32();
        return (uint64_t(next_u32()) << 32) | lo;
    }
    double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double a, double b) { return a + (b - a) * next_double(); }
    // standard normal, Marsaglia-Tsang ziggurat with 128 layers
    double normal() {
        const Zig& z = zig();
        constexpr double kTail = 3.442619855899;
        for (;;) {
            const int32_t hz = int32_t(next_u32());
            const int idx = hz & 127;
            if (std::abs(int64_t(hz)) < int64_t(z.kn[idx])) return hz * z.wn[idx];
            if (idx == 0) {
                for (;;) {
                    const double u1 = double((next_u64() >> 11) + 1) * 0x1.0p-53;
                    const double u2 = double((next_u64() >> 11) + 1) * 0x1.0p-53;
                    const double x = -std::log(u1) / kTail;
                    const double y = -std::log(u2);
                    if (y + y >= x * x) return hz > 0 ? kTail + x : -(kTail + x);
                }
            }
            const double x = hz * z.wn[idx];
            if (z.fn[idx] + next_double() * (z.fn[idx - 1] - z.fn[idx]) < std::exp(-0.5 * x * x)) return x;
        }
    }
    double normal(double mean, double stddev) { return mean + stddev * normal(); }
    double truncated_normal(double mean, double stddev, double lo, double hi) {
        for (;;) {
            const double v = normal(mean, stddev);
            if (v >= lo && v <= hi) return v;
        }
    }
    uint64_t next_below(uint64_t n) {
        const uint64_t limit = n * (UINT64_MAX / n);
        for (;;) {
            const uint64_t v = next_u64();
            if (v < limit) return v % n;
        }
    }
    uint64_t seed() const { return seed_; }
    uint64_t stream() const { return stream_; }

private:
    struct Zig {
        uint32_t kn[128];
        double wn[128], fn[128];
        Zig() {
            const double m1 = 2147483648.0, vn = 9.91256303526217e-3;
            double dn = 3.442619855899, tn = dn;
            const double q = vn / std::exp(-0.5 * dn * dn);
            kn[0] = uint32_t((dn / q) * m1);
            kn[1] = 0;
            wn[0] = q / m1;
            wn[127] = dn / m1;
            fn[0] = 1.0;
            fn[127] = std::exp(-0.5 * dn * dn);
            for (int i = 126; i >= 1; --i) {
                dn = std::sqrt(-2.0 * std::log(vn / dn + std::exp(-0.5 * dn * dn)));
                kn[i + 1] = uint32_t((dn / tn) * m1);
                tn = dn;
                fn[i] = std::exp(-0.5 * dn * dn);
                wn[i] = dn / m1;
            }
        }
    };
    static const Zig& zig() {
        static const Zig z;
        return z;
    }
    uint64_t seed_ = 0, stream_ = 0, idx_ = 0;
    std::array<uint32_t, 4> buf_{};
    int pos_ = 4;
};

// --------------------------------------------------------- distribution.hpp
struct Distribution {
    enum class Kind : uint8_t { Normal, Uniform, TruncNormal, AbsNormal };
    Kind kind = Kind::Uniform;
    double p0 = -1.0, p1 = 1.0, lo = -1.0, hi = 1.0;

    static Distribution normal(double mu, double sigma) { return {Kind::Normal, mu, sigma, -1.0, 1.0}; }
    static Distribution uniform(double a, double b) { return {Kind::Uniform, a, b, -1.0, 1.0}; }
    static Distribution truncated_normal(double mu, double sigma, double lo, double hi) {
        return {Kind::TruncNormal, mu, sigma, lo, hi};
    }
    static Distribution abs_normal(double mu, double sigma) { return {Kind::AbsNormal, mu, sigma, -1.0, 1.0}; }
    double sample(Philox& rng) const {
        switch (kind) {
            case Kind::Normal: return rng.normal(p0, p1);
            case Kind::Uniform: return rng.uniform(p0, p1);
            case Kind::TruncNormal: return rng.truncated_normal(p0, p1, lo, hi);
            case Kind::AbsNormal: return std::abs(rng.normal(p0, p1));
        }
        return 0.0;
    }
    std::string describe() const {
        auto num = [](double v) {
            std::ostringstream os;
            os << v;
            return os.str();
        };
        switch (kind) {
            case Kind::Normal: return "normal:" + num(p0) + "," + num(p1);
            case Kind::Uniform: return "uniform:" + num(p0) + "," + num(p1);
            case Kind::TruncNormal: return "truncnormal:" + num(p0) + "," + num(p1) + "," + num(lo) + "," + num(hi);
            case Kind::AbsNormal: return "absnormal:" + num(p0) + "," + num(p1);
        }
        return "?";
    }
    static Distribution parse(const std::string& text) {
        const size_t colon = text.find(':');
        const std::string name = text.substr(0, colon);
        std::vector<double> args;
        if (colon != std::string::npos) {
            std::stringstream ss(text.substr(colon + 1));
            std::string tok;
            while (std::getline(ss, tok, ','))
                if (!tok.empty()) args.push_back(std::stod(tok));
        }
        auto arg = [&](size_t i, double d) { return i < args.size() ? args[i] : d; };
        if (name == "normal") return normal(arg(0, 0.0), arg(1, 1.0));
        if (name == "uniform") return uniform(arg(0, -1.0), arg(1, 1.0));
        if (name == "truncnormal") return truncated_normal(arg(0, 0.0), arg(1, 1.0), arg(2, -1.0), arg(3, 1.0));
        if (name == "absnormal") return abs_normal(arg(0, 1.0), arg(1, 1.0));
        throw std::invalid_argument("unknown distribution: " + text);
    }
};

// random_matrix (distribution.cpp:95-101): row-major draws, quantized
inline Matrix random_matrix(int64_t rows, int64_t cols, const Distribution& dist, const PrecisionSpec& fmt, Philox& rng) {
    Matrix m(rows, cols, fmt);
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) m.set_raw(i, j, quantize(dist.sample(rng), fmt));
    return m;
}

// --------------------------------------------------------------- faults.hpp
enum class FaultTarget : uint8_t { OutputC, InputA, InputB };
enum class FlipDirection : uint8_t { Flip, Set0To1, Set1To0, Any };

inline const char* flip_direction_name(FlipDirection d) {
    switch (d) {
        case FlipDirection::Flip: return "flip";
        case FlipDirection::Set0To1: return "set0to1";
        case FlipDirection::Set1To0: return "set1to0";
        case FlipDirection::Any: return "any";
    }
    return "?";
}

struct FaultSpec {
    FaultTarget target = FaultTarget::OutputC;
    std::optional<std::pair<int64_t, int64_t>> position;
    int bit_index = 0;
    FlipDirection direction = FlipDirection::Flip;
};

struct InjectionRecord {
    int64_t i = -1, j = -1;
    int bit = 0;
    FlipDirection direction_taken = FlipDirection::Flip;
    double value_before = 0.0, value_after = 0.0;
    bool applied = false;
};

namespace detail {
inline bool bit_eligible(uint64_t bits, int bit, FlipDirection dir) {
    const uint64_t b = (bits >> bit) & 1u;
    return dir == FlipDirection::Set0To1 ? b == 0 : dir == FlipDirection::Set1To0 ? b == 1 : true;
}
}  // namespace detail

// inject (faults.cpp:104-168): fault placement consumes the trial's Philox
// stream exactly like the reference (direction draw for Any, up to 128
// next_below probes, then a full eligible scan).
inline std::pair<Matrix, InjectionRecord> inject(const Matrix& m, const FaultSpec& spec, Philox& rng) {
    const Format fmt = m.format().format;
    if (spec.bit_index < 0 || spec.bit_index >= m.format().bit_width())
        throw std::out_of_range("inject: bit index outside the format's width");
    FlipDirection dir = spec.direction;
    if (dir == FlipDirection::Any) dir = (rng.next_u32() & 1) ? FlipDirection::Set0To1 : FlipDirection::Set1To0;
    InjectionRecord rec;
    rec.bit = spec.bit_index;
    rec.direction_taken = dir;
    int64_t i = -1, j = -1;
    if (spec.position) {
        i = spec.position->first;
        j = spec.position->second;
        if (i < 0 || i >= m.rows() || j < 0 || j >= m.cols()) throw std::out_of_range("inject: position out of range");
        if (!detail::bit_eligible(encode_bits(m(i, j), fmt), spec.bit_index, dir)) {
            rec.i = i;
            rec.j = j;
            rec.value_before = rec.value_after = m(i, j);
            return {m, rec};
        }
    } else {
        const int64_t total = m.rows() * m.cols();
        bool found = false;
        for (int probe = 0; probe < 128 && !found; ++probe) {
            const int64_t flat = int64_t(rng.next_below(uint64_t(total)));
            if (detail::bit_eligible(encode_bits(m(flat / m.cols(), flat % m.cols()), fmt), spec.bit_index, dir)) {
                i = flat / m.cols();
                j = flat % m.cols();
                found = true;
            }
        }
        if (!found) {
            std::vector<int64_t> eligible;
            for (int64_t flat = 0; flat < total; ++flat)
                if (detail::bit_eligible(encode_bits(m(flat / m.cols(), flat % m.cols()), fmt), spec.bit_index, dir))
                    eligible.push_back(flat);
            if (eligible.empty()) return {m, rec};
            const int64_t flat = eligible[size_t(rng.next_below(eligible.size()))];
            i = flat / m.cols();
            j = flat % m.cols();
        }
    }
    const uint64_t after = encode_bits(m(i, j), fmt) ^ (uint64_t(1) << spec.bit_index);
    Matrix out = m;
    out.set_raw(i, j, decode_bits(after, fmt));
    rec.i = i;
    rec.j = j;
    rec.value_before = m(i, j);
    rec.value_after = out(i, j);
    rec.applied = true;
    return {std::move(out), rec};
}

struct CampaignConfig {
    int64_t m = 0, k = 0, n = 0;
    PrecisionSpec precision;
    Distribution dist;
    int bit_index = 0;
    int64_t trials = 1000;
    uint64_t seed = 0;
    VerifyMode mode = VerifyMode::Offline;
    FlipDirection direction = FlipDirection::Set0To1;
};

struct CampaignOutcome {
    int64_t trials = 0, applicable = 0, detected = 0, located_correctly = 0, nonfinite_after = 0;
    bool measurable() const { return applicable > 0; }
    double detection_rate() const { return applicable > 0 ? double(detected) / double(applicable) : 0.0; }
    double localization_accuracy() const { return detected > 0 ? double(located_correctly) / double(detected) : 0.0; }
};

using ThresholdFn = std::function<std::vector<double>(const Matrix&, const Matrix&)>;

// injection_campaign (faults.cpp:170-216): per trial Philox(seed, trial) ->
// A, B -> encode (device) -> thresholds_fn -> inject -> verify (device) ->
// tally of the flipped row. Same trials, same outcome counts as the
// reference. (The B200-native bulk campaign, M trials per fused launch, is
// the Python DeviceCampaign.)
inline CampaignOutcome injection_campaign(const CampaignConfig& config, const ThresholdFn& thresholds_fn) {
    if (config.trials < 1) throw std::invalid_argument("injection_campaign: trials must be >= 1");
    CampaignOutcome out;
    out.trials = config.trials;
    for (int64_t trial = 0; trial < config.trials; ++trial) {
        Philox rng(config.seed, uint64_t(trial));
        const Matrix a = random_matrix(config.m, config.k, config.dist, config.precision, rng);
        const Matrix b = random_matrix(config.k, config.n, config.dist, config.precision, rng);
        EncodedProduct prod = encode_and_multiply(a, b, config.mode);
        const std::vector<double> thresholds = thresholds_fn(a, b);
        FaultSpec spec;
        spec.bit_index = config.bit_index;
        spec.direction = config.direction;
        Matrix& target = config.mode == VerifyMode::Online ? prod.c_accum : prod.c;
        auto [corrupted, rec] = inject(target, spec, rng);
        if (!rec.applied) continue;
        target = std::move(corrupted);
        const std::vector<RowVerdict> v = verify(prod, thresholds);
        const RowVerdict& r = v[size_t(rec.i)];
        ++out.applicable;
        if (r.detected) ++out.detected;
        if (r.detected && r.location && *r.location == rec.j) ++out.located_correctly;
        if (!std::isfinite(rec.value_after)) ++out.nonfinite_after;
    }
    return out;
}

// ---------------------------------------------------------- calibration.hpp
// calibrate / fit_model (calibration.cpp:15-150): the reference's e_max
// calibration protocol, with every GEMM, checksum and row sum on the device
// EXACT engine (bit-identical to the emulator, hence the same maxima for the
// same seed). The tcgen05 fast path is calibrated by the Python
// paper_2602_08043_b200.calibration module (its accumulator differs).
struct CalibrationModel {
    EmaxModel::Kind kind = EmaxModel::Kind::Constant;
    double value = 0.0, scale = 0.0, offset = 0.0, cv = 0.0, r2 = 0.0;
};

inline CalibrationModel fit_model(std::span<const int64_t> sizes, std::span<const double> maxima) {
    if (sizes.size() != maxima.size() || sizes.empty())
        throw std::invalid_argument("fit_model: sizes and maxima must match and be nonempty");
    CalibrationModel m;
    const size_t n = maxima.size();
    double mean = 0.0;
    for (const double v : maxima) mean += v;
    mean /= double(n);
    m.value = mean;
    if (n >= 2 && mean > 0.0) {
        double ss = 0.0;
        for (const double v : maxima) ss += (v - mean) * (v - mean);
        m.cv = std::sqrt(ss / double(n - 1)) / mean;
    }
    if (n >= 2) {
        double sx = 0, sy = 0, sxx = 0, sxy = 0;
        for (size_t i = 0; i < n; ++i) {
            const double x = std::sqrt(double(sizes[i]));
            sx += x;
            sy += maxima[i];
            sxx += x * x;
            sxy += x * maxima[i];
        }
        const double denom = double(n) * sxx - sx * sx;
        if (denom != 0.0) {
            m.scale = (double(n) * sxy - sx * sy) / denom;
            m.offset = (sy - m.scale * sx) / double(n);
            double ss_res = 0, ss_tot = 0;
            for (size_t i = 0; i < n; ++i) {
                const double fit = m.scale * std::sqrt(double(sizes[i])) + m.offset;
                ss_res += (maxima[i] - fit) * (maxima[i] - fit);
                ss_tot += (maxima[i] - mean) * (maxima[i] - mean);
            }
            m.r2 = ss_tot > 0.0 ? 1.0 - ss_res / ss_tot : 1.0;
        }
    }
    const bool constant = n < 2 || m.cv < 0.15 || m.scale <= 0.0;
    m.kind = constant ? EmaxModel::Kind::Constant : EmaxModel::Kind::SqrtScaled;
    return m;
}

struct CalibrationResult {
    Format precision = Format::FP64;
    VerifyMode mode = VerifyMode::Offline;
    AccumStrategy accumulation{};
    std::vector<int64_t> sizes;
    std::vector<double> maxima;
    CalibrationModel model;
    double recommended = 0.0;
    uint64_t seed = 0;
    int64_t trials_per_size = 0;
    int64_t aborted_trials = 0;
    double unit_roundoff = 0.0;

    // e_max_for (calibration.cpp:61-74)
    double e_max_for(int64_t dim) const {
        const double floor = 2.0 * unit_roundoff;
        if (model.kind == EmaxModel::Kind::Constant) return std::max(recommended, floor);
        double lambda = 1.0;
        for (size_t i = 0; i < sizes.size(); ++i) {
            const double fit = model.scale * std::sqrt(double(sizes[i])) + model.offset;
            if (fit > 0.0) lambda = std::max(lambda, maxima[i] / fit);
        }
        return std::max(1.2 * lambda * (model.scale * std::sqrt(double(dim)) + model.offset), floor);
    }
    // recommended_model (calibration.cpp:76-86)
    EmaxModel recommended_model() const {
        if (model.kind == EmaxModel::Kind::Constant) return EmaxModel::constant(std::max(recommended, 2.0 * unit_roundoff));
        double lambda = 1.0;
        for (size_t i = 0; i < sizes.size(); ++i) {
            const double fit = model.scale * std::sqrt(double(sizes[i])) + model.offset;
            if (fit > 0.0) lambda = std::max(lambda, maxima[i] / fit);
        }
        return EmaxModel::sqrt_scaled(1.2 * lambda * model.scale, std::max(1.2 * lambda * model.offset, 0.0));
    }
};

// calibrate (calibration.cpp:88-150): per trial Philox(seed, idx) -> |N(1,1)|
// square A, B -> encode_and_multiply -> row_sums of the verification source
// -> max_i |r1 - check1| / |check1| (a non-finite ratio aborts the trial);
// per size the max over trials; fit_model; recommended = max(1.2 max, 2u).
inline CalibrationResult calibrate(const PrecisionSpec& precision, std::span<const int64_t> sizes,
                                   int64_t trials_per_size, uint64_t seed, VerifyMode mode = VerifyMode::Offline) {
    if (sizes.empty()) throw std::invalid_argument("calibrate: need at least one size");
    if (trials_per_size < 1) throw std::invalid_argument("calibrate: trials must be >= 1");
    const Distribution dist = Distribution::abs_normal(1.0, 1.0);
    const int64_t n_sizes = int64_t(sizes.size());
    CalibrationResult out;
    out.precision = precision.format;
    out.mode = mode;
    out.accumulation = precision.accumulation;
    out.sizes.assign(sizes.begin(), sizes.end());
    out.seed = seed;
    out.trials_per_size = trials_per_size;
    out.unit_roundoff = checksum_precision_for(precision, mode).unit_roundoff;
    double overall = 0.0;
    for (int64_t si = 0; si < n_sizes; ++si) {
        const int64_t s = sizes[size_t(si)];
        double mx_size = 0.0;
        for (int64_t t = 0; t < trials_per_size; ++t) {
            Philox rng(seed, uint64_t(si * trials_per_size + t));
            const Matrix a = random_matrix(s, s, dist, precision, rng);
            const Matrix b = random_matrix(s, s, dist, precision, rng);
            const EncodedProduct prod = encode_and_multiply(a, b, mode);
            const auto [r1, r2] = row_sums(prod.verification_source(), prod.checksum_precision);
            (void)r2;
            double mx = 0.0;
            bool aborted = false;
            for (int64_t i = 0; i < s; ++i) {
                const double denom = std::abs(prod.row_check1[size_t(i)]);
                const double rel = std::abs(r1[size_t(i)] - prod.row_check1[size_t(i)]) / denom;
                if (!std::isfinite(rel)) {
                    aborted = true;
                    break;
                }
                mx = std::max(mx, rel);
            }
            if (aborted) {
                ++out.aborted_trials;
                continue;
            }
            mx_size = std::max(mx_size, mx);
        }
        out.maxima.push_back(mx_size);
        overall = std::max(overall, mx_size);
    }
    out.model = fit_model(out.sizes, out.maxima);
    out.recommended = std::max(1.2 * overall, 2.0 * out.unit_roundoff);
    return out;
}

// ------------------------------------------------------------ matrix_io.hpp
// VABFTMAT binary: magic, u32 version, u8 format id, u64 rows, u64 cols,
// rows*cols little-endian FP64 (matrix_io.hpp:12-17); CSV one row per line.
// Loading quantizes finite values (Matrix::set) and keeps non-finite values
// raw (matrix_io.cpp:34-45). Host file I/O.
inline constexpr uint32_t kMatrixFileVersion = 1;

namespace detail {
inline constexpr char kMatrixMagic[8] = {'V', 'A', 'B', 'F', 'T', 'M', 'A', 'T'};
inline void fill_values(Matrix& m, const std::vector<double>& vals) {
    for (int64_t i = 0; i < m.rows(); ++i)
        for (int64_t j = 0; j < m.cols(); ++j) {
            const double v = vals[size_t(i * m.cols() + j)];
            if (std::isfinite(v)) m.set(i, j, v);
            else m.set_raw(i, j, v);
        }
}
}  // namespace detail

inline void save_matrix_binary(const Matrix& m, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open for writing: " + path);
    const uint32_t version = kMatrixFileVersion;
    const uint8_t fmt = uint8_t(m.format().format);
    const uint64_t rows = uint64_t(m.rows()), cols = uint64_t(m.cols());
    bool ok = std::fwrite(detail::kMatrixMagic, 1, 8, f) == 8 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&fmt, 1, 1, f) == 1 && std::fwrite(&rows, 8, 1, f) == 1 && std::fwrite(&cols, 8, 1, f) == 1 &&
              std::fwrite(m.values().data(), 8, m.values().size(), f) == m.values().size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write failed: " + path);
}

inline Matrix load_matrix_binary(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open: " + path);
    struct Closer {
        std::FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[8];
    if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, detail::kMatrixMagic, 8) != 0)
        throw std::runtime_error("not a VABFTMAT file: " + path);
    uint32_t version;
    uint8_t fmt;
    uint64_t rows, cols;
    if (std::fread(&version, 4, 1, f) != 1) throw std::runtime_error("truncated matrix file: " + path);
    if (version != kMatrixFileVersion) throw std::runtime_error("unsupported matrix file version in " + path);
    if (std::fread(&fmt, 1, 1, f) != 1) throw std::runtime_error("truncated matrix file: " + path);
    if (fmt > 3) throw std::runtime_error("bad format id in " + path);
    if (std::fread(&rows, 8, 1, f) != 1 || std::fread(&cols, 8, 1, f) != 1)
        throw std::runtime_error("truncated matrix file: " + path);
    if (rows < 1 || cols < 1 || rows > (uint64_t(1) << 32) || cols > (uint64_t(1) << 32))
        throw std::runtime_error("implausible dimensions in " + path);
    std::vector<double> vals(size_t(rows * cols));
    if (std::fread(vals.data(), 8, vals.size(), f) != vals.size())
        throw std::runtime_error("truncated matrix file: " + path);
    Matrix m(int64_t(rows), int64_t(cols), PrecisionSpec::of(Format(fmt)));
    detail::fill_values(m, vals);
    return m;
}

inline void save_matrix_csv(const Matrix& m, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open for writing: " + path);
    for (int64_t i = 0; i < m.rows(); ++i) {
        for (int64_t j = 0; j < m.cols(); ++j) std::fprintf(f, j ? ",%.17g" : "%.17g", m(i, j));
        std::fputc('\n', f);
    }
    std::fclose(f);
}

inline Matrix load_matrix_csv(const std::string& path, const PrecisionSpec& fmt) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw std::runtime_error("cannot open: " + path);
    std::vector<double> vals;
    int64_t rows = 0, cols = -1;
    std::string line;
    auto flush_line = [&] {
        if (line.empty()) return;
        int64_t c = 0;
        size_t pos = 0;
        while (pos <= line.size()) {
            const size_t comma = line.find(',', pos);
            const std::string tok = line.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
            if (!tok.empty()) {
                vals.push_back(std::stod(tok));
                ++c;
            }
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
        if (cols == -1) cols = c;
        else if (c != cols) throw std::runtime_error("ragged CSV row in " + path);
        ++rows;
        line.clear();
    };
    for (int ch; (ch = std::fgetc(f)) != EOF;) {
        if (ch == '\n') flush_line();
        else line.push_back(char(ch));
    }
    std::fclose(f);
    flush_line();
    if (rows == 0) throw std::runtime_error("empty CSV: " + path);
    Matrix m(rows, cols, fmt);
    detail::fill_values(m, vals);
    return m;
}

inline Matrix load_matrix_auto(const std::string& path, const std::optional<PrecisionSpec>& csv_format = std::nullopt) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open: " + path);
    char magic[8] = {};
    const size_t got = std::fread(magic, 1, 8, f);
    std::fclose(f);
    if (got == 8 && std::memcmp(magic, detail::kMatrixMagic, 8) == 0) return load_matrix_binary(path);
    return load_matrix_csv(path, csv_format.value_or(PrecisionSpec::fp64()));
}

// =========================================================== B200 extension
// The hot path on caller-owned device memory: the fused V-ABFT GEMM
// (vabft_bside_* / vabft_fused_gemm), RAII over the B-side handle and the
// workspace. Not part of the reference API.
namespace b200 {

class FusedGemm {
public:
    // B: K x N device matrix in the format's native storage (BF16 / FP16 bits
    // on tcgen05, FP32 on tcgen05 kind::tf32 with 3xTF32, FP64 on the SIMT
    // DFMA kernel), fixed weight.
    FusedGemm(Format fmt, VerifyMode mode, int64_t k, int64_t n, const void* B, double e_max, void* stream = nullptr)
        : k_(k), n_(n) {
        opts_.mode = mode == VerifyMode::Online ? VABFT_ONLINE : VABFT_OFFLINE;
        opts_.threshold_method = 0;
        opts_.e_max = e_max;
        opts_.c_sigma = 2.5;
        opts_.floor_scale = 1e-3;
        opts_.aabft_fixed_y = 21.0;
        opts_.aabft_confidence = 3.0;
        opts_.cta_mode = -1;    // the measured kernel-shape policy
        opts_.tf32_passes = 3;  // FP32: 3xTF32
        detail::check(vabft_bside_create(int32_t(fmt), opts_.mode, k, n, B, &h_, stream));
    }
    ~FusedGemm() {
        if (h_) vabft_bside_destroy(h_);
    }
    FusedGemm(const FusedGemm&) = delete;
    FusedGemm& operator=(const FusedGemm&) = delete;
    vabft_fused_opts& options() { return opts_; }
    void update_weight(const void* B, void* stream = nullptr) { detail::check(vabft_bside_update(h_, B, stream)); }
    // C = A B (M x N) with thresholds T (M, may be null), verdict arrays and
    // counters (device, accumulated); stream-ordered, no host sync.
    void operator()(int64_t m, const void* A, void* C, double* T, vabft_verdicts verdicts, int64_t* counts,
                    void* stream = nullptr) {
        size_t bytes = 0;
        detail::check(vabft_fused_workspace_size(m, n_, k_, &bytes));
        if (bytes > ws_bytes_) {
            ws_ = detail::DeviceBuffer(bytes);
            ws_bytes_ = bytes;
        }
        detail::check(vabft_fused_gemm(&opts_, h_, m, A, C, T, verdicts, counts, ws_.get(), ws_bytes_, stream));
    }

private:
    int64_t k_, n_;
    vabft_bside_t h_ = nullptr;
    vabft_fused_opts opts_{};
    detail::DeviceBuffer ws_;
    size_t ws_bytes_ = 0;
};

}  // namespace b200

}  // namespace vabft

#endif  // VABFT_CPP_HPP_
