// C-ABI plumbing: thread-local last error, status mapping, device info.
#include <array>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "internal.hpp"

namespace vabft_dev {

thread_local std::string g_last_error;

namespace {
constexpr int kMaxDevices = 64;
std::atomic<int> g_sm_count[kMaxDevices];  // 0 = not yet queried
std::mutex g_attr_mu;
std::set<std::tuple<const void*, int, int>> g_attr_done;   // (kernel, device, smem bytes)
std::map<std::pair<const void*, int>, int> g_clusters;      // (kernel, device) -> co-resident clusters
}  // namespace

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    return dev;
}

// Per device (a process may drive several GPUs), lock-free after the first query.
int sm_count() {
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) {
        int n = 0;
        return cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0 ? n : 148;
    }
    int n = g_sm_count[dev].load(std::memory_order_relaxed);
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sm_count[dev].store(n, std::memory_order_relaxed);
    return n;
}

// cudaFuncSetAttribute is per (function, device): apply it once for each
// device the calling thread's launches target, thread-safely.
void ensure_smem_attr(const void* fn, int bytes) {
    const auto key = std::make_tuple(fn, current_device(), bytes);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (g_attr_done.count(key)) return;
    check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
               "cudaFuncSetAttribute(max dynamic shared memory)");
    g_attr_done.insert(key);
}

int cached_occupancy(const void* fn, int threads, int smem) {
    return cached_cluster_count(
        fn,
        [](const void* f, void* ctx) {
            const int* a = static_cast<const int*>(ctx);
            int n = 0;
            check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, a[0], size_t(a[1])),
                       "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
            return n;
        },
        const_cast<int*>(std::array<int, 2>{threads, smem}.data()));
}

int cached_cluster_count(const void* fn, int (*compute)(const void*, void*), void* ctx) {
    const auto key = std::make_pair(fn, current_device());
    {
        std::lock_guard<std::mutex> lk(g_attr_mu);
        auto it = g_clusters.find(key);
        if (it != g_clusters.end()) return it->second;
    }
    const int n = compute(fn, ctx);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    g_clusters[key] = n;
    return n;
}

CUtensorMap encode_map_2d(CUtensorMapDataType dt, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t elem_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swizzle) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }();
    if (!fn) fail(VABFT_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * elem_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(VABFT_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
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
