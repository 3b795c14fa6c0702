// _core — pybind11 binding of the C++ drop-in (include/vabft_cpp.hpp), the
// module the reference declares as vabft._core (proj/python/CMakeLists.txt:17-21,
// whose bindings.cpp is not in the reference tree). Names follow the C++ API;
// Matrix converts to / from numpy (float64, row-major). Exceptions map to
// Python as pybind11 does for the standard types (invalid_argument /
// domain_error / range_error -> ValueError, out_of_range -> IndexError,
// logic_error -> RuntimeError) plus vabft.device_error -> DeviceError.
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "vabft_cpp.hpp"

namespace py = pybind11;
using namespace vabft;

namespace {

using DArr = py::array_t<double, py::array::c_style | py::array::forcecast>;

py::array_t<double> to_numpy(const Matrix& m) {
    py::array_t<double> out({m.rows(), m.cols()});
    std::memcpy(out.mutable_data(), m.values().data(), sizeof(double) * size_t(m.rows() * m.cols()));
    return out;
}

Matrix from_numpy(const DArr& a, const PrecisionSpec& fmt, bool quantize_values) {
    if (a.ndim() != 2) throw std::invalid_argument("Matrix: expected a 2-D array");
    return Matrix::from_values(a.shape(0), a.shape(1), std::span<const double>(a.data(), size_t(a.size())), fmt,
                               quantize_values);
}

std::vector<double> vec(const DArr& a) { return std::vector<double>(a.data(), a.data() + a.size()); }

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B200 V-ABFT C++ drop-in (namespace vabft) over libvabft_b200";
    py::register_exception<device_error>(m, "DeviceError", PyExc_RuntimeError);

    py::enum_<Format>(m, "Format")
        .value("BF16", Format::BF16).value("FP16", Format::FP16).value("FP32", Format::FP32).value("FP64", Format::FP64);
    m.def("format_name", &format_name);
    m.def("format_from_name", &format_from_name);
    py::enum_<AccumKind>(m, "AccumKind")
        .value("Fp32AccumRoundOutput", AccumKind::Fp32AccumRoundOutput)
        .value("NativeSequential", AccumKind::NativeSequential)
        .value("NativeBlocked", AccumKind::NativeBlocked)
        .value("NativePairwise", AccumKind::NativePairwise);
    py::class_<AccumStrategy>(m, "AccumStrategy")
        .def(py::init([](AccumKind k, int64_t bl) { return AccumStrategy{k, bl}; }), py::arg("kind"),
             py::arg("block_len") = 128)
        .def_readwrite("kind", &AccumStrategy::kind)
        .def_readwrite("block_len", &AccumStrategy::block_len)
        .def("describe", &AccumStrategy::describe);
    py::class_<EmaxModel> em(m, "EmaxModel");
    py::enum_<EmaxModel::Kind>(em, "Kind").value("Constant", EmaxModel::Kind::Constant).value("SqrtScaled", EmaxModel::Kind::SqrtScaled);
    em.def_readwrite("kind", &EmaxModel::kind)
        .def_readwrite("scale", &EmaxModel::scale)
        .def_readwrite("offset", &EmaxModel::offset)
        .def_static("constant", &EmaxModel::constant)
        .def_static("sqrt_scaled", &EmaxModel::sqrt_scaled)
        .def("resolve", &EmaxModel::resolve);
    py::enum_<OverflowPolicy>(m, "OverflowPolicy").value("Saturate", OverflowPolicy::Saturate).value("Error", OverflowPolicy::Error);
    py::class_<PrecisionSpec>(m, "PrecisionSpec")
        .def(py::init<>())
        .def_readwrite("format", &PrecisionSpec::format)
        .def_readwrite("mantissa_bits", &PrecisionSpec::mantissa_bits)
        .def_readwrite("unit_roundoff", &PrecisionSpec::unit_roundoff)
        .def_readwrite("accumulation", &PrecisionSpec::accumulation)
        .def_readwrite("e_max_model", &PrecisionSpec::e_max_model)
        .def_readwrite("overflow", &PrecisionSpec::overflow)
        .def_static("bf16", &PrecisionSpec::bf16)
        .def_static("fp16", &PrecisionSpec::fp16)
        .def_static("fp32", &PrecisionSpec::fp32)
        .def_static("fp64", &PrecisionSpec::fp64)
        .def_static("of", &PrecisionSpec::of)
        .def("min_normal_exponent", &PrecisionSpec::min_normal_exponent)
        .def("max_finite", &PrecisionSpec::max_finite)
        .def("min_subnormal", &PrecisionSpec::min_subnormal)
        .def("bit_width", &PrecisionSpec::bit_width)
        .def("name", &PrecisionSpec::name)
        .def("with_accumulation", &PrecisionSpec::with_accumulation)
        .def("with_e_max", &PrecisionSpec::with_e_max);
    m.def("quantize", &quantize);
    m.def("accumulates_in_float", &accumulates_in_float);

    py::class_<Matrix>(m, "Matrix")
        .def(py::init<int64_t, int64_t, PrecisionSpec>())
        .def_static("from_values", [](int64_t r, int64_t c, const DArr& v, const PrecisionSpec& f, bool q) {
            return Matrix::from_values(r, c, std::span<const double>(v.data(), size_t(v.size())), f, q);
        }, py::arg("rows"), py::arg("cols"), py::arg("values"), py::arg("fmt"), py::arg("quantize_values") = true)
        .def_static("from_numpy", &from_numpy, py::arg("array"), py::arg("fmt"), py::arg("quantize_values") = true)
        .def_static("identity", &Matrix::identity)
        .def("rows", &Matrix::rows)
        .def("cols", &Matrix::cols)
        .def("format", &Matrix::format)
        .def("__call__", &Matrix::operator())
        .def("at", &Matrix::at)
        .def("set", &Matrix::set)
        .def("set_raw", &Matrix::set_raw)
        .def("same_bits", &Matrix::same_bits)
        .def("values", [](const Matrix& x) { return to_numpy(x); })
        .def("row", [](const Matrix& x, int64_t i) {
            if (i < 0 || i >= x.rows()) throw std::out_of_range("Matrix::row: index out of range");
            auto r = x.row(i);
            return std::vector<double>(r.begin(), r.end());
        });
    py::class_<GemmResult>(m, "GemmResult").def_readonly("c", &GemmResult::c).def_readonly("accum", &GemmResult::accum);
    m.def("gemm_emulated", &gemm_emulated);
    m.def("gemm_emulated_with_accum", &gemm_emulated_with_accum);
    m.def("reduce_in_precision", [](const DArr& t, const PrecisionSpec& s) { return reduce_in_precision(vec(t), s); });

    py::enum_<VerifyMode>(m, "VerifyMode").value("Offline", VerifyMode::Offline).value("Online", VerifyMode::Online);
    m.def("verify_mode_name", &verify_mode_name);
    m.def("verify_mode_from_name", &verify_mode_from_name);
    m.def("checksum_precision_for", &checksum_precision_for);
    py::class_<ChecksumVectors>(m, "ChecksumVectors")
        .def_readonly("n", &ChecksumVectors::n)
        .def_static("weight", &ChecksumVectors::weight)
        .def_static("make", &ChecksumVectors::make)
        .def("ones", &ChecksumVectors::ones)
        .def("weights", &ChecksumVectors::weights);
    py::class_<EncodedProduct>(m, "EncodedProduct")
        .def_readwrite("c", &EncodedProduct::c)
        .def_readwrite("row_check1", &EncodedProduct::row_check1)
        .def_readwrite("row_check2", &EncodedProduct::row_check2)
        .def_readwrite("col_check1", &EncodedProduct::col_check1)
        .def_readwrite("col_check2", &EncodedProduct::col_check2)
        .def_readwrite("checksum_precision", &EncodedProduct::checksum_precision)
        .def_readwrite("mode", &EncodedProduct::mode)
        .def_readwrite("c_accum", &EncodedProduct::c_accum)
        .def("verification_source", &EncodedProduct::verification_source, py::return_value_policy::reference_internal);
    m.def("encode_and_multiply", &encode_and_multiply, py::arg("a"), py::arg("b"), py::arg("mode") = VerifyMode::Offline);
    m.def("row_sums", &row_sums);

    py::class_<RowStats>(m, "RowStats")
        .def(py::init<>())
        .def_readwrite("mean", &RowStats::mean)
        .def_readwrite("max", &RowStats::max)
        .def_readwrite("min", &RowStats::min)
        .def_readwrite("var_bound", &RowStats::var_bound)
        .def_readwrite("n", &RowStats::n);
    m.def("row_stats", [](const DArr& v) { return row_stats(vec(v)); });

    py::class_<VabftParams>(m, "VabftParams")
        .def(py::init([](double e, double c) { return VabftParams{e, c}; }), py::arg("e_max") = 0.0, py::arg("c_sigma") = 2.5)
        .def_readwrite("e_max", &VabftParams::e_max)
        .def_readwrite("c_sigma", &VabftParams::c_sigma);
    py::class_<ThresholdBreakdown>(m, "ThresholdBreakdown")
        .def_readonly("det", &ThresholdBreakdown::det)
        .def_readonly("var23", &ThresholdBreakdown::var23)
        .def_readonly("var4", &ThresholdBreakdown::var4)
        .def_readonly("total", &ThresholdBreakdown::total);
    m.def("precompute_b_stats", &precompute_b_stats);
    py::class_<BStatsSummary>(m, "BStatsSummary")
        .def(py::init<>())
        .def_readwrite("sum_abs_mean", &BStatsSummary::sum_abs_mean)
        .def_readwrite("sum_mean_sq", &BStatsSummary::sum_mean_sq)
        .def_readwrite("sum_var", &BStatsSummary::sum_var)
        .def_readwrite("k_len", &BStatsSummary::k_len)
        .def_static("from_", [](const std::vector<RowStats>& s) { return BStatsSummary::from(s); });
    m.def("threshold_row", py::overload_cast<const RowStats&, const BStatsSummary&, int64_t, const VabftParams&>(&threshold_row));
    m.def("threshold_row", [](const RowStats& a, const std::vector<RowStats>& b, int64_t n, const VabftParams& p) {
        return threshold_row(a, std::span<const RowStats>(b), n, p);
    });
    m.def("resolve_e_max", &resolve_e_max);
    m.def("vabft_thresholds", &vabft_thresholds);

    py::class_<AabftParams>(m, "AabftParams")
        .def(py::init<>())
        .def_readwrite("mantissa_bits", &AabftParams::mantissa_bits)
        .def_readwrite("fixed_y", &AabftParams::fixed_y)
        .def_readwrite("confidence_multiplier", &AabftParams::confidence_multiplier)
        .def_static("for_format", &AabftParams::for_format)
        .def("computed_y", &AabftParams::computed_y);
    m.def("aabft_sigma", &aabft_sigma);
    py::class_<AabftThresholds>(m, "AabftThresholds")
        .def_readonly("per_row", &AabftThresholds::per_row)
        .def_readonly("y_used", &AabftThresholds::y_used)
        .def_readonly("degenerate", &AabftThresholds::degenerate);
    m.def("aabft_threshold", &aabft_threshold);
    m.def("aabft_computed_y", &aabft_computed_y);

    py::class_<RowVerdict>(m, "RowVerdict")
        .def(py::init<>())
        .def_readwrite("row", &RowVerdict::row)
        .def_readwrite("diff1", &RowVerdict::diff1)
        .def_readwrite("diff2", &RowVerdict::diff2)
        .def_readwrite("threshold", &RowVerdict::threshold)
        .def_readwrite("detected", &RowVerdict::detected)
        .def_readwrite("location", &RowVerdict::location)
        .def_readwrite("correction", &RowVerdict::correction)
        .def_readwrite("localization_residual", &RowVerdict::localization_residual);
    py::class_<DetectOptions>(m, "DetectOptions")
        .def(py::init<>())
        .def_readwrite("localization_floor_scale", &DetectOptions::localization_floor_scale)
        .def_readwrite("residual_margin", &DetectOptions::residual_margin);
    m.def("localize", &localize);
    m.def("verify", [](const EncodedProduct& p, const DArr& t, const DetectOptions& o) { return verify(p, vec(t), o); },
          py::arg("prod"), py::arg("thresholds"), py::arg("opts") = DetectOptions{});
    m.def("correct", &correct);

    py::class_<Philox>(m, "Philox")
        .def(py::init<uint64_t, uint64_t>(), py::arg("seed"), py::arg("stream") = 0)
        .def("next_u32", &Philox::next_u32)
        .def("next_u64", &Philox::next_u64)
        .def("next_double", &Philox::next_double)
        .def("uniform", &Philox::uniform)
        .def("normal", py::overload_cast<>(&Philox::normal))
        .def("normal", py::overload_cast<double, double>(&Philox::normal))
        .def("truncated_normal", &Philox::truncated_normal)
        .def("next_below", &Philox::next_below)
        .def_static("block", &Philox::block);
    py::class_<Distribution> dist(m, "Distribution");
    py::enum_<Distribution::Kind>(dist, "Kind")
        .value("Normal", Distribution::Kind::Normal).value("Uniform", Distribution::Kind::Uniform)
        .value("TruncNormal", Distribution::Kind::TruncNormal).value("AbsNormal", Distribution::Kind::AbsNormal);
    dist.def_readwrite("kind", &Distribution::kind)
        .def_static("normal", &Distribution::normal)
        .def_static("uniform", &Distribution::uniform)
        .def_static("truncated_normal", &Distribution::truncated_normal)
        .def_static("abs_normal", &Distribution::abs_normal)
        .def_static("parse", &Distribution::parse)
        .def("sample", &Distribution::sample)
        .def("describe", &Distribution::describe);
    m.def("random_matrix", &random_matrix);

    py::enum_<FaultTarget>(m, "FaultTarget")
        .value("OutputC", FaultTarget::OutputC).value("InputA", FaultTarget::InputA).value("InputB", FaultTarget::InputB);
    py::enum_<FlipDirection>(m, "FlipDirection")
        .value("Flip", FlipDirection::Flip).value("Set0To1", FlipDirection::Set0To1)
        .value("Set1To0", FlipDirection::Set1To0).value("Any", FlipDirection::Any);
    m.def("flip_direction_name", &flip_direction_name);
    py::class_<FaultSpec>(m, "FaultSpec")
        .def(py::init<>())
        .def_readwrite("target", &FaultSpec::target)
        .def_readwrite("position", &FaultSpec::position)
        .def_readwrite("bit_index", &FaultSpec::bit_index)
        .def_readwrite("direction", &FaultSpec::direction);
    py::class_<InjectionRecord>(m, "InjectionRecord")
        .def_readonly("i", &InjectionRecord::i)
        .def_readonly("j", &InjectionRecord::j)
        .def_readonly("bit", &InjectionRecord::bit)
        .def_readonly("direction_taken", &InjectionRecord::direction_taken)
        .def_readonly("value_before", &InjectionRecord::value_before)
        .def_readonly("value_after", &InjectionRecord::value_after)
        .def_readonly("applied", &InjectionRecord::applied);
    m.def("encode_bits", &encode_bits);
    m.def("decode_bits", &decode_bits);
    m.def("inject", &inject);
    py::class_<CampaignConfig>(m, "CampaignConfig")
        .def(py::init<>())
        .def_readwrite("m", &CampaignConfig::m)
        .def_readwrite("k", &CampaignConfig::k)
        .def_readwrite("n", &CampaignConfig::n)
        .def_readwrite("precision", &CampaignConfig::precision)
        .def_readwrite("dist", &CampaignConfig::dist)
        .def_readwrite("bit_index", &CampaignConfig::bit_index)
        .def_readwrite("trials", &CampaignConfig::trials)
        .def_readwrite("seed", &CampaignConfig::seed)
        .def_readwrite("mode", &CampaignConfig::mode)
        .def_readwrite("direction", &CampaignConfig::direction);
    py::class_<CampaignOutcome>(m, "CampaignOutcome")
        .def_readonly("trials", &CampaignOutcome::trials)
        .def_readonly("applicable", &CampaignOutcome::applicable)
        .def_readonly("detected", &CampaignOutcome::detected)
        .def_readonly("located_correctly", &CampaignOutcome::located_correctly)
        .def_readonly("nonfinite_after", &CampaignOutcome::nonfinite_after)
        .def("measurable", &CampaignOutcome::measurable)
        .def("detection_rate", &CampaignOutcome::detection_rate)
        .def("localization_accuracy", &CampaignOutcome::localization_accuracy);
    m.def("injection_campaign", &injection_campaign);

    py::enum_<b200::Engine>(m, "Engine").value("Exact", b200::Engine::Exact).value("Tensor", b200::Engine::Tensor);
    m.def("set_engine", &b200::set_engine);
    m.def("engine", &b200::engine);

    py::class_<CalibrationModel>(m, "CalibrationModel")
        .def(py::init<>())
        .def_readwrite("kind", &CalibrationModel::kind)
        .def_readwrite("value", &CalibrationModel::value)
        .def_readwrite("scale", &CalibrationModel::scale)
        .def_readwrite("offset", &CalibrationModel::offset)
        .def_readwrite("cv", &CalibrationModel::cv)
        .def_readwrite("r2", &CalibrationModel::r2);
    py::class_<CalibrationResult>(m, "CalibrationResult")
        .def_readonly("precision", &CalibrationResult::precision)
        .def_readonly("mode", &CalibrationResult::mode)
        .def_readonly("sizes", &CalibrationResult::sizes)
        .def_readonly("maxima", &CalibrationResult::maxima)
        .def_readonly("model", &CalibrationResult::model)
        .def_readonly("recommended", &CalibrationResult::recommended)
        .def_readonly("seed", &CalibrationResult::seed)
        .def_readonly("trials_per_size", &CalibrationResult::trials_per_size)
        .def_readonly("aborted_trials", &CalibrationResult::aborted_trials)
        .def_readonly("unit_roundoff", &CalibrationResult::unit_roundoff)
        .def("e_max_for", &CalibrationResult::e_max_for)
        .def("recommended_model", &CalibrationResult::recommended_model);
    m.def("fit_model", [](const std::vector<int64_t>& sizes, const std::vector<double>& maxima) {
        return fit_model(sizes, maxima);
    });
    m.def("calibrate",
          [](const PrecisionSpec& p, const std::vector<int64_t>& sizes, int64_t trials, uint64_t seed, VerifyMode mode) {
              return calibrate(p, sizes, trials, seed, mode);
          },
          py::arg("precision"), py::arg("sizes"), py::arg("trials_per_size"), py::arg("seed"),
          py::arg("mode") = VerifyMode::Offline);

    m.attr("kMatrixFileVersion") = kMatrixFileVersion;
    m.def("save_matrix_binary", &save_matrix_binary);
    m.def("load_matrix_binary", &load_matrix_binary);
    m.def("save_matrix_csv", &save_matrix_csv);
    m.def("load_matrix_csv", &load_matrix_csv);
    m.def("load_matrix_auto", &load_matrix_auto, py::arg("path"), py::arg("csv_format") = std::nullopt);

    // B200 extension: the fused path on device pointers (integers, e.g.
    // torch's data_ptr()); verdict arrays optional (0 = not written)
    py::class_<b200::FusedGemm>(m, "FusedGemm")
        .def(py::init([](Format fmt, VerifyMode mode, int64_t k, int64_t n, uintptr_t B, double e_max,
                         uintptr_t stream) {
                 return std::make_unique<b200::FusedGemm>(fmt, mode, k, n, reinterpret_cast<const void*>(B), e_max,
                                                          reinterpret_cast<void*>(stream));
             }),
             py::arg("format"), py::arg("mode"), py::arg("k"), py::arg("n"), py::arg("B"), py::arg("e_max"),
             py::arg("stream") = 0)
        .def("__call__",
             [](b200::FusedGemm& g, int64_t m, uintptr_t A, uintptr_t C, uintptr_t T, uintptr_t detected,
                uintptr_t location, uintptr_t counts, uintptr_t stream) {
                 vabft_verdicts v{};
                 v.detected = reinterpret_cast<uint8_t*>(detected);
                 v.location = reinterpret_cast<int64_t*>(location);
                 g(m, reinterpret_cast<const void*>(A), reinterpret_cast<void*>(C), reinterpret_cast<double*>(T), v,
                   reinterpret_cast<int64_t*>(counts), reinterpret_cast<void*>(stream));
             },
             py::arg("m"), py::arg("A"), py::arg("C"), py::arg("T") = 0, py::arg("detected") = 0,
             py::arg("location") = 0, py::arg("counts") = 0, py::arg("stream") = 0);
}
