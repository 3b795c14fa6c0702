// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" driver over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It exposes
// the hot-path API (precision/checksum/stats/threshold/detect/faults/rng/
// distribution/calibration) with plain pointers so tests/ and bench.py's
// reference arm can call the reference through ctypes. Every function is a
// thin adapter; all arithmetic happens in the reference's own code.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "vabft/calibration.hpp"
#include "vabft/matrix_io.hpp"
#include "vabft/checksum.hpp"
#include "vabft/detect.hpp"
#include "vabft/distribution.hpp"
#include "vabft/faults.hpp"
#include "vabft/parallel.hpp"
#include "vabft/precision.hpp"
#include "vabft/rng.hpp"
#include "vabft/stats.hpp"
#include "vabft/threshold_aabft.hpp"
#include "vabft/threshold_vabft.hpp"

using namespace vabft;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 domain_error, 3 range_error, 4 out_of_range, 5 logic/other
template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::range_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

PrecisionSpec spec_of(int fmt, int accum_kind, int64_t block_len) {
    PrecisionSpec s = PrecisionSpec::of(Format(fmt));
    if (accum_kind >= 0) s.accumulation = AccumStrategy{AccumKind(accum_kind), block_len};
    return s;
}

Distribution dist_of(int kind, double p0, double p1, double lo, double hi) {
    switch (kind) {
        case 0: return Distribution::normal(p0, p1);
        case 1: return Distribution::uniform(p0, p1);
        case 2: return Distribution::truncated_normal(p0, p1, lo, hi);
        default: return Distribution::abs_normal(p0, p1);
    }
}

Matrix raw_matrix(int64_t r, int64_t c, const double* v, const PrecisionSpec& s) {
    Matrix m(r, c, s);
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < c; ++j) m.set_raw(i, j, v[i * c + j]);
    return m;
}

void copy_out(const Matrix& m, double* out) {
    if (out) std::memcpy(out, m.values().data(), m.values().size() * sizeof(double));
}

ThresholdFn method_fn(int method, int fmt, double e_max, double c_sigma) {
    if (method == 0)
        return [=](const Matrix& a, const Matrix& b) {
            return vabft_thresholds(a, b, VabftParams{e_max, c_sigma});
        };
    AabftParams p = AabftParams::for_format(Format(fmt));
    if (method == 1) p.fixed_y = 21.0; else p.fixed_y.reset();
    return [=](const Matrix& a, const Matrix& b) { return aabft_threshold(a, b, p).per_row; };
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    auto r = Philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

// Draw `count` values of a stream: kind 0 u32, 1 u64, 2 double, 3 normal, 4 next_below(arg)
int ref_philox_draws(uint64_t seed, uint64_t stream, int kind, double arg, int64_t count, double* out,
                     uint64_t* out_u) {
    return guard([&] {
        Philox rng(seed, stream);
        for (int64_t i = 0; i < count; ++i) {
            switch (kind) {
                case 0: out_u[i] = rng.next_u32(); break;
                case 1: out_u[i] = rng.next_u64(); break;
                case 2: out[i] = rng.next_double(); break;
                case 3: out[i] = rng.normal(); break;
                default: out_u[i] = rng.next_below(uint64_t(arg)); break;
            }
        }
    });
}

// random_matrix draws of trial `stream`: A (m x k) then B (k x n), as the campaigns do.
int ref_trial_inputs(int64_t m, int64_t k, int64_t n, int fmt, int dist_kind, double p0, double p1,
                     double lo, double hi, uint64_t seed, uint64_t stream, double* A, double* B) {
    return guard([&] {
        Philox rng(seed, stream);
        const PrecisionSpec s = PrecisionSpec::of(Format(fmt));
        const Distribution d = dist_of(dist_kind, p0, p1, lo, hi);
        copy_out(random_matrix(m, k, d, s, rng), A);
        if (B) copy_out(random_matrix(k, n, d, s, rng), B);
    });
}

int ref_quantize(double x, int fmt, int overflow_error, double* out) {
    return guard([&] {
        PrecisionSpec s = PrecisionSpec::of(Format(fmt));
        if (overflow_error) s.overflow = OverflowPolicy::Error;
        *out = quantize(x, s);
    });
}

int ref_encode_and_multiply(int fmt, int accum_kind, int64_t block_len, int mode, int64_t m,
                            int64_t k, int64_t n, const double* A, const double* B, double* C,
                            double* C_accum, double* rc1, double* rc2, double* cc1, double* cc2) {
    return guard([&] {
        const PrecisionSpec s = spec_of(fmt, accum_kind, block_len);
        const Matrix a = raw_matrix(m, k, A, s);
        const Matrix b = raw_matrix(k, n, B, s);
        const EncodedProduct p = encode_and_multiply(a, b, VerifyMode(mode));
        copy_out(p.c, C);
        copy_out(p.c_accum, C_accum);
        if (rc1) std::memcpy(rc1, p.row_check1.data(), sizeof(double) * size_t(m));
        if (rc2) std::memcpy(rc2, p.row_check2.data(), sizeof(double) * size_t(m));
        if (cc1) std::memcpy(cc1, p.col_check1.data(), sizeof(double) * size_t(n));
        if (cc2) std::memcpy(cc2, p.col_check2.data(), sizeof(double) * size_t(n));
    });
}

// row_sums of an M x N source with the checksum precision of (fmt, mode),
// optionally overriding its accumulation strategy.
int ref_row_sums(int fmt, int mode, int accum_kind, int64_t block_len, int64_t m, int64_t n,
                 const double* src, double* r1, double* r2) {
    return guard([&] {
        PrecisionSpec cs = checksum_precision_for(PrecisionSpec::of(Format(fmt)), VerifyMode(mode));
        if (accum_kind >= 0) cs.accumulation = AccumStrategy{AccumKind(accum_kind), block_len};
        const PrecisionSpec src_spec = (mode == 1 && fmt != 3) ? PrecisionSpec::fp32()
                                                               : PrecisionSpec::of(Format(fmt));
        const Matrix c = raw_matrix(m, n, src, src_spec);
        auto [a, b] = row_sums(c, cs);
        std::memcpy(r1, a.data(), sizeof(double) * size_t(m));
        std::memcpy(r2, b.data(), sizeof(double) * size_t(m));
    });
}

int ref_row_stats(const double* v, int64_t n, double out[5]) {
    return guard([&] {
        const RowStats s = row_stats(std::span<const double>(v, size_t(n)));
        out[0] = s.mean;
        out[1] = s.max;
        out[2] = s.min;
        out[3] = s.var_bound;
        out[4] = double(s.n);
    });
}

int ref_vabft_thresholds(int fmt, int64_t m, int64_t k, int64_t n, const double* A, const double* B,
                         double e_max, double c_sigma, double* T, double* summary) {
    return guard([&] {
        const PrecisionSpec s = PrecisionSpec::of(Format(fmt));
        const Matrix a = raw_matrix(m, k, A, s);
        const Matrix b = raw_matrix(k, n, B, s);
        const std::vector<double> t = vabft_thresholds(a, b, VabftParams{e_max, c_sigma});
        std::memcpy(T, t.data(), sizeof(double) * size_t(m));
        if (summary) {
            const BStatsSummary bs = BStatsSummary::from(precompute_b_stats(b));
            summary[0] = bs.sum_abs_mean;
            summary[1] = bs.sum_mean_sq;
            summary[2] = bs.sum_var;
        }
    });
}

int ref_threshold_row(const double a_stats[4], const double b_summary[3], int64_t k_len, int64_t n,
                      double e_max, double c_sigma, double out[4]) {
    return guard([&] {
        RowStats a;
        a.mean = a_stats[0];
        a.max = a_stats[1];
        a.min = a_stats[2];
        a.var_bound = a_stats[3];
        BStatsSummary b;
        b.sum_abs_mean = b_summary[0];
        b.sum_mean_sq = b_summary[1];
        b.sum_var = b_summary[2];
        b.k_len = k_len;
        const ThresholdBreakdown t = threshold_row(a, b, n, VabftParams{e_max, c_sigma});
        out[0] = t.det;
        out[1] = t.var23;
        out[2] = t.var4;
        out[3] = t.total;
    });
}

int ref_resolve_e_max(int fmt, int64_t dim, double* out) {
    return guard([&] { *out = resolve_e_max(PrecisionSpec::of(Format(fmt)), dim); });
}

int ref_aabft_sigma(int64_t n, int t, double y, double* out) {
    return guard([&] { *out = aabft_sigma(n, t, y); });
}

// fixed_y: NaN selects computed y; mantissa_bits < 0 uses the format default.
int ref_aabft_threshold(int fmt, int64_t m, int64_t k, int64_t n, const double* A, const double* B,
                        int mantissa_bits, double fixed_y, double conf, double* T, double* y_used,
                        int* degenerate) {
    return guard([&] {
        const PrecisionSpec s = PrecisionSpec::of(Format(fmt));
        const Matrix a = raw_matrix(m, k, A, s);
        const Matrix b = raw_matrix(k, n, B, s);
        AabftParams p = AabftParams::for_format(Format(fmt));
        if (mantissa_bits >= 0) p.mantissa_bits = mantissa_bits;
        if (std::isnan(fixed_y)) p.fixed_y.reset(); else p.fixed_y = fixed_y;
        if (conf > 0) p.confidence_multiplier = conf;
        const AabftThresholds t = aabft_threshold(a, b, p);
        std::memcpy(T, t.per_row.data(), sizeof(double) * size_t(m));
        *y_used = t.y_used;
        *degenerate = t.degenerate ? 1 : 0;
    });
}

int ref_localize(double d1, double d2, int64_t n_cols, int64_t* j, double* residual) {
    const auto r = localize(d1, d2, n_cols);
    if (!r) return 0;
    *j = r->first;
    *residual = r->second;
    return 1;
}

// verify() on an explicit product: source values (c or c_accum), checksums,
// thresholds. accum_kind >= 0 overrides the checksum precision's strategy.
int ref_verify(int fmt, int mode, int accum_kind, int64_t block_len, int64_t m, int64_t n,
               const double* source, const double* rc1, const double* rc2, const double* T,
               double floor_scale, double* diff1, double* diff2, uint8_t* detected,
               int64_t* location, double* residual) {
    return guard([&] {
        EncodedProduct p;
        const PrecisionSpec in = PrecisionSpec::of(Format(fmt));
        p.mode = VerifyMode(mode);
        p.checksum_precision = checksum_precision_for(in, p.mode);
        if (accum_kind >= 0)
            p.checksum_precision.accumulation = AccumStrategy{AccumKind(accum_kind), block_len};
        const PrecisionSpec src_spec = (mode == 1 && fmt != 3) ? PrecisionSpec::fp32() : in;
        if (p.mode == VerifyMode::Online) {
            p.c_accum = raw_matrix(m, n, source, src_spec);
            p.c = Matrix(m, n, in);
        } else {
            p.c = raw_matrix(m, n, source, src_spec);
        }
        p.row_check1.assign(rc1, rc1 + m);
        p.row_check2.assign(rc2, rc2 + m);
        DetectOptions o;
        o.localization_floor_scale = floor_scale;
        const std::vector<RowVerdict> v = verify(p, std::span<const double>(T, size_t(m)), o);
        for (int64_t i = 0; i < m; ++i) {
            const RowVerdict& r = v[size_t(i)];
            if (diff1) diff1[i] = r.diff1;
            if (diff2) diff2[i] = r.diff2;
            if (detected) detected[i] = r.detected ? 1 : 0;
            if (location) location[i] = r.location ? *r.location : -1;
            if (residual) residual[i] = r.localization_residual;
        }
    });
}

int ref_correct(int fmt, int64_t m, int64_t n, const double* c, int64_t row, int64_t loc,
                double correction, double* out) {
    return guard([&] {
        const Matrix cm = raw_matrix(m, n, c, PrecisionSpec::of(Format(fmt)));
        RowVerdict v;
        v.row = row;
        v.detected = true;
        if (loc >= 0) v.location = loc;
        v.correction = correction;
        copy_out(correct(cm, v), out);
    });
}

int ref_encode_bits(double v, int fmt, uint64_t* out) {
    return guard([&] { *out = encode_bits(v, Format(fmt)); });
}
int ref_decode_bits(uint64_t b, int fmt, double* out) {
    return guard([&] { *out = decode_bits(b, Format(fmt)); });
}

// inject() on an M x N matrix. pos_i < 0 selects a random position drawn
// from Philox(seed, stream) after `skip_u32` raw draws (so callers can
// replay a campaign trial). rec: {i, j, applied, dir_taken}, vals: {before, after}.
int ref_inject(int fmt, int src_fp32, int64_t m, int64_t n, double* X, int64_t pos_i, int64_t pos_j,
               int bit, int dir, uint64_t seed, uint64_t stream, int64_t* rec, double* vals) {
    return guard([&] {
        PrecisionSpec s = PrecisionSpec::of(Format(fmt));
        if (src_fp32) s = PrecisionSpec::fp32();
        const Matrix mat = raw_matrix(m, n, X, s);
        FaultSpec f;
        if (pos_i >= 0) f.position = std::make_pair(pos_i, pos_j);
        f.bit_index = bit;
        f.direction = FlipDirection(dir);
        Philox rng(seed, stream);
        auto [out, r] = inject(mat, f, rng);
        copy_out(out, X);
        rec[0] = r.i;
        rec[1] = r.j;
        rec[2] = r.applied ? 1 : 0;
        rec[3] = int64_t(r.direction_taken);
        vals[0] = r.value_before;
        vals[1] = r.value_after;
    });
}

// One trial of injection_campaign (faults.cpp:181-203), run serially:
// out = {applied, detected, located, nonfinite, i, j}.
int ref_campaign_trial(int64_t m, int64_t k, int64_t n, int fmt, int dist_kind, double p0, double p1,
                       double lo, double hi, int bit, int dir, uint64_t seed, uint64_t trial,
                       int mode, int method, double e_max, double c_sigma, int64_t out[6]) {
    return guard([&] {
        const PrecisionSpec s = PrecisionSpec::of(Format(fmt));
        const Distribution d = dist_of(dist_kind, p0, p1, lo, hi);
        Philox rng(seed, trial);
        const Matrix a = random_matrix(m, k, d, s, rng);
        const Matrix b = random_matrix(k, n, d, s, rng);
        EncodedProduct prod = encode_and_multiply(a, b, VerifyMode(mode));
        const std::vector<double> thr = method_fn(method, fmt, e_max, c_sigma)(a, b);
        FaultSpec spec;
        spec.bit_index = bit;
        spec.direction = FlipDirection(dir);
        Matrix& target = mode == 1 ? prod.c_accum : prod.c;
        auto [corrupted, rec] = inject(target, spec, rng);
        for (int q = 0; q < 6; ++q) out[q] = 0;
        out[4] = rec.i;
        out[5] = rec.j;
        if (!rec.applied) return;
        target = std::move(corrupted);
        const std::vector<RowVerdict> v = verify(prod, thr);
        const RowVerdict& r = v[size_t(rec.i)];
        out[0] = 1;
        out[1] = r.detected ? 1 : 0;
        out[2] = (r.detected && r.location && *r.location == rec.j) ? 1 : 0;
        out[3] = std::isfinite(rec.value_after) ? 0 : 1;
    });
}

// injection_campaign (faults.cpp:170-216): out = {trials, applicable, detected, located, nonfinite}.
int ref_injection_campaign(int64_t m, int64_t k, int64_t n, int fmt, int dist_kind, double p0,
                           double p1, double lo, double hi, int bit, int dir, int64_t trials,
                           uint64_t seed, int mode, int method, double e_max, double c_sigma,
                           int64_t out[5]) {
    return guard([&] {
        CampaignConfig cc;
        cc.m = m;
        cc.k = k;
        cc.n = n;
        cc.precision = PrecisionSpec::of(Format(fmt));
        cc.dist = dist_of(dist_kind, p0, p1, lo, hi);
        cc.bit_index = bit;
        cc.trials = trials;
        cc.seed = seed;
        cc.mode = VerifyMode(mode);
        cc.direction = FlipDirection(dir);
        const CampaignOutcome o = injection_campaign(cc, method_fn(method, fmt, e_max, c_sigma));
        out[0] = o.trials;
        out[1] = o.applicable;
        out[2] = o.detected;
        out[3] = o.located_correctly;
        out[4] = o.nonfinite_after;
    });
}

// calibrate (calibration.cpp:88-150): maxima per size, model, recommended, e_max at dim.
int ref_calibrate(int fmt, int mode, const int64_t* sizes, int64_t n_sizes, int64_t trials,
                  uint64_t seed, int64_t dim, double* maxima, double out[6]) {
    return guard([&] {
        const CalibrationResult r =
            calibrate(PrecisionSpec::of(Format(fmt)), std::span<const int64_t>(sizes, size_t(n_sizes)),
                      trials, seed, VerifyMode(mode));
        for (int64_t i = 0; i < n_sizes; ++i) maxima[i] = r.maxima[size_t(i)];
        out[0] = r.model.kind == EmaxModel::Kind::Constant ? 0.0 : 1.0;
        out[1] = r.model.value;
        out[2] = r.model.scale;
        out[3] = r.model.offset;
        out[4] = r.recommended;
        out[5] = r.e_max_for(dim);
    });
}

int ref_max_threads() { return max_threads(); }

// matrix_io (matrix_io.cpp:49-137): save a raw matrix / load with the
// reference's loaders (dims first with out == nullptr, then the values).
int ref_save_matrix(int binary, int fmt, int64_t m, int64_t n, const double* v, const char* path) {
    return guard([&] {
        const Matrix mat = raw_matrix(m, n, v, PrecisionSpec::of(Format(fmt)));
        if (binary) save_matrix_binary(mat, path);
        else save_matrix_csv(mat, path);
    });
}
int ref_load_matrix(const char* path, int csv_fmt, int64_t* dims, double* out) {
    return guard([&] {
        const Matrix mat = load_matrix_auto(path, PrecisionSpec::of(Format(csv_fmt)));
        dims[0] = mat.rows();
        dims[1] = mat.cols();
        dims[2] = int64_t(mat.format().format);
        if (out) copy_out(mat, out);
    });
}

}  // extern "C"
