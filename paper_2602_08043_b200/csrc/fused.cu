// The hot path: V-ABFT fused GEMM (TENSOR engine).
//
//   vabft_bside_create   per-weight B state: precompute_b_stats +
//                        BStatsSummary::from (threshold_vabft.cpp:8-26), B r1 /
//                        B r2 (checksum.cpp:110-115), max_k |sum_j B| for A-ABFT
//                        computed y (threshold_aabft.cpp:38-48).
//   vabft_fused_gemm     1. aside_kernel: A row stats -> V-ABFT T_i
//                           (threshold_vabft.cpp:54-61), A (B r1/2), max|A|
//                        2. tc_gemm (tcgen05): C plus per-128-column row
//                           partials of the FP32 accumulator (online) or of
//                           the quantized output (offline), optional in-
//                           epilogue fault injection (faults.cpp:104-168)
//                        3. verify tail: blocked:128 row sums, D1/D2, strict
//                           compare, NaN rule, localization (detect.cpp:9-55),
//                           warp-aggregated counters.
// No host synchronization anywhere on this path.
#include <cstring>

#include "devcommon.cuh"
#include "guard.hpp"
#include "internal.hpp"
#include "numerics.cuh"
#include "stats.hpp"

struct vabft_bside {
    int fmt;
    int mode;
    int b_kmajor;
    int64_t k, n;
    const void* B;  // not owned
    vabft_dev::BsideBuffers buf;
    void* storage;  // one cudaMalloc holding every buffer
};

namespace vabft_dev {

namespace {

__global__ void fused_tail_kernel(int64_t M, int64_t N, int64_t K, int64_t nblk,
                                  const float* __restrict__ part1, const float* __restrict__ part2,
                                  const double* __restrict__ cr1, const double* __restrict__ cr2,
                                  const double* __restrict__ Tv, const double* __restrict__ bsum,
                                  const double* __restrict__ max_abs_a, int method, int aabft_t,
                                  double aabft_fixed_y, double aabft_conf, double floor_scale,
                                  double* T_out, vabft_verdicts v, int64_t* counts) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = i < M;
    bool det = false, located = false, isnan_row = false;
    if (valid) {
        // reduce_terms NativeBlocked(128): tot += part per block, in order.
        float r1 = 0.0f, r2 = 0.0f;
        for (int64_t b = 0; b < nblk; ++b) {
            r1 = __fadd_rn(r1, part1[b * M + i]);
            r2 = __fadd_rn(r2, part2[b * M + i]);
        }
        double t;
        if (method == 0) {
            t = Tv[i];
        } else {
            const double y = method == 1 ? aabft_fixed_y : __dmul_rn(*max_abs_a, bsum[3]);
            t = aabft_total(K, aabft_t, y, aabft_conf);
        }
        if (T_out && method != 0) T_out[i] = t;
        const double d1 = __dsub_rn(double(r1), cr1[i]);
        const double d2 = __dsub_rn(double(r2), cr2[i]);
        int64_t loc = -1;
        double res = 0.0;
        if (isnan(d1) || isnan(d2)) {
            det = true;
            isnan_row = true;
        } else {
            det = fabs(d1) > t;
            if (det && fabs(d1) > __dmul_rn(floor_scale, t)) {
                int64_t j;
                double rr;
                if (localize_dev(d1, d2, N, &j, &rr)) {
                    loc = j;
                    res = rr;
                    located = true;
                }
            }
        }
        if (v.diff1) v.diff1[i] = d1;
        if (v.diff2) v.diff2[i] = d2;
        if (v.detected) v.detected[i] = det ? 1 : 0;
        if (v.location) v.location[i] = loc;
        if (v.residual) v.residual[i] = res;
    }
    if (counts) {
        const unsigned mv = __ballot_sync(0xffffffffu, valid);
        const unsigned md = __ballot_sync(0xffffffffu, det);
        const unsigned ml = __ballot_sync(0xffffffffu, located);
        const unsigned mn = __ballot_sync(0xffffffffu, isnan_row);
        if ((threadIdx.x & 31) == 0) {
            if (mv) atomicAdd(reinterpret_cast<unsigned long long*>(counts + VABFT_COUNT_ROWS), __popc(mv));
            if (md) atomicAdd(reinterpret_cast<unsigned long long*>(counts + VABFT_COUNT_DETECTED), __popc(md));
            if (ml) atomicAdd(reinterpret_cast<unsigned long long*>(counts + VABFT_COUNT_LOCATED), __popc(ml));
            if (mn) atomicAdd(reinterpret_cast<unsigned long long*>(counts + VABFT_COUNT_NAN), __popc(mn));
        }
    }
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Per-thread, per-device side stream + fork/join events: the HBM-bound
// A-side statistics pass runs concurrently with the tensor-bound GEMM
// (its CTAs use no shared memory and co-reside with the persistent GEMM
// CTAs); the verify tail joins both. Capturable into CUDA graphs.
struct SideStream {
    int dev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

SideStream& side_stream() {
    thread_local SideStream ss;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (ss.dev != dev) {
        check_cuda(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking), "cudaStreamCreate");
        check_cuda(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming), "cudaEventCreate");
        check_cuda(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming), "cudaEventCreate");
        ss.dev = dev;
    }
    return ss;
}

struct FusedWs {
    float* part1;
    float* part2;
    double* cr1;
    double* cr2;
    double* Tv;
    double* max_abs_a;
    size_t bytes;
};

FusedWs carve(void* base, int64_t M, int64_t N) {
    const int64_t nblk = (N + 127) / 128;
    FusedWs w{};
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t sz) {
        char* p = b ? b + off : nullptr;
        off += align_up(sz);
        return p;
    };
    w.part1 = reinterpret_cast<float*>(take(sizeof(float) * size_t(nblk * M)));
    w.part2 = reinterpret_cast<float*>(take(sizeof(float) * size_t(nblk * M)));
    w.cr1 = reinterpret_cast<double*>(take(sizeof(double) * size_t(M)));
    w.cr2 = reinterpret_cast<double*>(take(sizeof(double) * size_t(M)));
    w.Tv = reinterpret_cast<double*>(take(sizeof(double) * size_t(M)));
    w.max_abs_a = reinterpret_cast<double*>(take(sizeof(double)));
    w.bytes = off;
    return w;
}

}  // namespace
}  // namespace vabft_dev

using namespace vabft_dev;

extern "C" vabft_status vabft_bside_create(int32_t format, int32_t mode, int64_t k, int64_t n,
                                           const void* B, vabft_bside_t* out, void* stream) {
    return guarded([&] {
        if (!out) fail(VABFT_INVALID_ARGUMENT, "vabft_bside_create: null handle pointer");
        if (format < VABFT_BF16 || format > VABFT_FP64) fail(VABFT_INVALID_ARGUMENT, "bad format");
        if (mode != VABFT_OFFLINE && mode != VABFT_ONLINE) fail(VABFT_INVALID_ARGUMENT, "bad mode");
        if (k < 1 || n < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        // ChecksumVectors::make: weights exact in FP32 (checksum.cpp:26-34)
        if (n > (int64_t(1) << 24)) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: weights exceed exact range");
        auto* h = new vabft_bside();
        h->fmt = format;
        h->mode = mode;
        h->b_kmajor = 0;
        h->k = k;
        h->n = n;
        h->B = B;
        const size_t K = size_t(k);
        const size_t KB = size_t(br_storage_floats(k));
        const size_t bytes = align_up(8 * K) * 3 + align_up(4 * KB) * 2 + align_up(8 * 4) + align_up(4);
        cudaError_t e = cudaMalloc(&h->storage, bytes);
        if (e != cudaSuccess) {
            delete h;
            fail(VABFT_CUDA_ERROR, std::string("cudaMalloc(bside): ") + cudaGetErrorString(e));
        }
        char* p = static_cast<char*>(h->storage);
        h->buf.mean = reinterpret_cast<double*>(p); p += align_up(8 * K);
        h->buf.vb = reinterpret_cast<double*>(p); p += align_up(8 * K);
        h->buf.rowsum_abs = reinterpret_cast<double*>(p); p += align_up(8 * K);
        h->buf.br1 = reinterpret_cast<float*>(p); p += align_up(4 * KB);
        h->buf.br2 = reinterpret_cast<float*>(p); p += align_up(4 * KB);
        h->buf.summary = reinterpret_cast<double*>(p); p += align_up(32);
        h->buf.nonfinite = reinterpret_cast<int*>(p);
        *out = h;
        if (B) {
            check_cuda(cudaMemsetAsync(h->buf.nonfinite, 0, sizeof(int), as_stream(stream)), "memset");
            launch_bside(format, k, n, B, mode == VABFT_OFFLINE ? 1 : 0, h->buf, as_stream(stream));
        }
    });
}

extern "C" vabft_status vabft_bside_update(vabft_bside_t h, const void* B, void* stream) {
    return guarded([&] {
        if (!h || !B) fail(VABFT_INVALID_ARGUMENT, "vabft_bside_update: null argument");
        h->B = B;
        check_cuda(cudaMemsetAsync(h->buf.nonfinite, 0, sizeof(int), as_stream(stream)), "memset");
        launch_bside(h->fmt, h->k, h->n, B, h->mode == VABFT_OFFLINE ? 1 : 0, h->buf, as_stream(stream));
    });
}

extern "C" vabft_status vabft_bside_destroy(vabft_bside_t h) {
    return guarded([&] {
        if (!h) return;
        cudaFree(h->storage);
        delete h;
    });
}

extern "C" vabft_status vabft_fused_workspace_size(int64_t m, int64_t n, int64_t k, size_t* bytes) {
    return guarded([&] {
        (void)k;
        if (!bytes) fail(VABFT_INVALID_ARGUMENT, "null bytes");
        if (m < 1 || n < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        *bytes = carve(nullptr, m, n).bytes;
    });
}

extern "C" vabft_status vabft_fused_gemm(const vabft_fused_opts* o, vabft_bside_t h, int64_t m,
                                         const void* A, void* C, double* T, vabft_verdicts verdicts,
                                         int64_t* counts, void* workspace, size_t ws_bytes,
                                         void* stream) {
    return guarded([&] {
        if (!o || !h || !A || !C || !h->B) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: null argument");
        if (h->fmt != VABFT_BF16 && h->fmt != VABFT_FP16)
            fail(VABFT_UNSUPPORTED, "vabft_fused_gemm: TENSOR engine needs BF16/FP16 (use the EXACT engine)");
        if (o->mode != h->mode) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: mode differs from the B-side handle");
        if (o->threshold_method < 0 || o->threshold_method > 2) fail(VABFT_INVALID_ARGUMENT, "bad threshold method");
        if (o->b_kmajor != h->b_kmajor)
            fail(VABFT_UNSUPPORTED, "vabft_fused_gemm: B layout differs from the B-side handle");
        if (m < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        if (m > (int64_t(1) << 24)) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: weights exceed exact range");
        const int64_t n = h->n, k = h->k;
        const FusedWs ws = carve(workspace, m, n);
        if (!workspace || ws_bytes < ws.bytes) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: workspace too small");
        cudaStream_t s = as_stream(stream);
        const bool offline = o->mode == VABFT_OFFLINE;
        double* Tv = (T && o->threshold_method == 0) ? T : ws.Tv;
        SideStream& side = side_stream();
        check_cuda(cudaEventRecord(side.fork, s), "cudaEventRecord");
        check_cuda(cudaStreamWaitEvent(side.s, side.fork, 0), "cudaStreamWaitEvent");
        TcEpilogue epi;
        epi.abft = offline ? 2 : 1;
        epi.part1 = ws.part1;
        epi.part2 = ws.part2;
        epi.fault_col = o->fault_col;
        epi.fault_bit = o->fault_bit;
        epi.fault_dir = o->fault_dir;
        epi.fault_records = o->fault_records;
        tc_gemm_launch(h->fmt, o->b_kmajor != 0, m, n, k, A, h->B, C, epi, s);
        // statistics pass on the side stream, overlapping the GEMM
        check_cuda(cudaMemsetAsync(ws.max_abs_a, 0, sizeof(double), side.s), "memset");
        launch_aside(h->fmt, m, k, n, A, h->buf, offline ? 1 : 0, o->e_max, o->c_sigma, Tv, ws.cr1, ws.cr2,
                     ws.max_abs_a, side.s);
        check_cuda(cudaEventRecord(side.join, side.s), "cudaEventRecord");
        check_cuda(cudaStreamWaitEvent(s, side.join, 0), "cudaStreamWaitEvent");
        const int64_t nblk = (n + 127) / 128;
        const int t_bits = o->aabft_mantissa_bits > 0 ? o->aabft_mantissa_bits
                                                      : (h->fmt == VABFT_BF16 ? 8 : 11);
        fused_tail_kernel<<<unsigned((m + 255) / 256), 256, 0, s>>>(
            m, n, k, nblk, ws.part1, ws.part2, ws.cr1, ws.cr2, Tv, h->buf.summary, ws.max_abs_a,
            o->threshold_method, t_bits, o->aabft_fixed_y, o->aabft_confidence > 0 ? o->aabft_confidence : 3.0,
            o->floor_scale, T, verdicts, counts);
        check_cuda(cudaGetLastError(), "fused tail launch");
    });
}
