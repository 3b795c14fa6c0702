// C-ABI plumbing: thread-local last error, status mapping, device info.
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "internal.hpp"

namespace vabft_dev {

thread_local std::string g_last_error;

int sm_count() {
    static int cached = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    static int cached_dev = -1;
    if (cached < 0 || cached_dev != dev) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached = n;
        cached_dev = dev;
    }
    return cached;
}

size_t elem_size(int fmt) {
    switch (fmt) {
        case VABFT_BF16:
        case VABFT_FP16: return 2;
        case VABFT_FP32: return 4;
        case VABFT_FP64: return 8;
    }
    fail(VABFT_INVALID_ARGUMENT, "bad format");
}

void set_last_error(const std::string& s) { g_last_error = s; }

}  // namespace vabft_dev

extern "C" const char* vabft_last_error(void) { return vabft_dev::g_last_error.c_str(); }

extern "C" int32_t vabft_api_version(void) { return VABFT_C_API_VERSION; }

extern "C" vabft_status vabft_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        vabft_dev::set_last_error(std::string("cudaGetDevice: ") + cudaGetErrorString(e));
        return VABFT_CUDA_ERROR;
    }
    int sm = 0, ma = 0, mi = 0;
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev);
    if (sm_count) *sm_count = sm;
    if (cc_major) *cc_major = ma;
    if (cc_minor) *cc_minor = mi;
    return VABFT_OK;
}
