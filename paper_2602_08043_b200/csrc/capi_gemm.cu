// C-ABI entry points of the tcgen05 GEMM (plain, overhead baseline).
#include "guard.hpp"
#include "internal.hpp"

using namespace vabft_dev;

extern "C" vabft_status vabft_gemm_plain(int32_t format, int32_t b_kmajor, int64_t m, int64_t n,
                                         int64_t k, const void* A, const void* B, void* C,
                                         void* stream) {
    return guarded([&] {
        if (!A || !B || !C) fail(VABFT_INVALID_ARGUMENT, "vabft_gemm_plain: null pointer");
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
        TcEpilogue epi;
        epi.cta_mode = cta_mode;
        tc_gemm_launch(format, b_kmajor != 0, m, n, k, A, B, C, epi, as_stream(stream));
    });
}

