// C-ABI entry points of the plain GEMMs (overhead baselines): tcgen05 for the
// 16-bit formats and FP32 (3xTF32), the SIMT DFMA kernel (wide.cu) for FP64.
#include "guard.hpp"
#include "internal.hpp"

using namespace vabft_dev;

extern "C" vabft_status vabft_gemm_plain(int32_t format, int32_t b_kmajor, int64_t m, int64_t n,
                                         int64_t k, const void* A, const void* B, void* C,
                                         void* stream) {
    return guarded([&] {
        if (!A || !B || !C) fail(VABFT_INVALID_ARGUMENT, "vabft_gemm_plain: null pointer");
        if (format == VABFT_FP64) {
            if (b_kmajor) fail(VABFT_UNSUPPORTED, "vabft_gemm_plain: FP64 needs a row-major B");
            dgemm_launch(m, n, k, static_cast<const double*>(A), static_cast<const double*>(B),
                         static_cast<double*>(C), WideEpilogue{}, as_stream(stream));
            return;
        }
        if (format == VABFT_FP32) {
            if (b_kmajor) fail(VABFT_UNSUPPORTED, "vabft_gemm_plain: FP32 needs a row-major B");
            tf32_gemm_run(m, n, k, static_cast<const float*>(A), static_cast<const float*>(B), static_cast<float*>(C),
                          WideEpilogue{}, 3, as_stream(stream));
            return;
        }
        TcEpilogue epi;
        tc_gemm_launch(format, b_kmajor != 0, m, n, k, A, B, C, epi, as_stream(stream));
    });
}

extern "C" vabft_status vabft_gemm_plain_mode(int32_t format, int32_t b_kmajor, int64_t m, int64_t n,
                                              int64_t k, const void* A, const void* B, void* C,
                                              int32_t cta_mode, void* stream) {
    return guarded([&] {
        if (!A || !B || !C) fail(VABFT_INVALID_ARGUMENT, "vabft_gemm_plain: null pointer");
        if (cta_mode < -1 || cta_mode > 1) fail(VABFT_INVALID_ARGUMENT, "vabft_gemm_plain: bad cta_mode");
        if (format == VABFT_FP64) {
            if (b_kmajor) fail(VABFT_UNSUPPORTED, "vabft_gemm_plain: FP64 needs a row-major B");
            dgemm_launch(m, n, k, static_cast<const double*>(A), static_cast<const double*>(B),
                         static_cast<double*>(C), WideEpilogue{}, as_stream(stream));
            return;
        }
        if (format == VABFT_FP32) {
            if (b_kmajor) fail(VABFT_UNSUPPORTED, "vabft_gemm_plain: FP32 needs a row-major B");
            tf32_gemm_run(m, n, k, static_cast<const float*>(A), static_cast<const float*>(B), static_cast<float*>(C),
                          WideEpilogue{}, 3, as_stream(stream));
            return;
        }
        TcEpilogue epi;
        epi.cta_mode = cta_mode;
        tc_gemm_launch(format, b_kmajor != 0, m, n, k, A, B, C, epi, as_stream(stream));
    });
}

