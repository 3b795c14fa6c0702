// The hot path: V-ABFT fused GEMM (TENSOR engine).
//
//   vabft_bside_create   per-weight B state: precompute_b_stats +
//                        BStatsSummary::from (threshold_vabft.cpp:8-26), B r1 /
//                        B r2 (checksum.cpp:110-115), max_k |sum_j B| for A-ABFT
//                        computed y (threshold_aabft.cpp:38-48).
//   vabft_fused_gemm     1. tc_gemm (tcgen05), one persistent kernel:
//                           - MMA: C = A B, FP32 accumulators in TMEM;
//                           - epilogue warps: per-128-column row partials of
//                             the FP32 accumulator (online) or of the quantized
//                             output (offline), optional in-epilogue fault
//                             injection (faults.cpp:104-168), C store;
//                           - statistics warps: read the TMA-staged A tiles from
//                             shared memory and produce per-(row, 128-k-block)
//                             A (B r) partials and exact row-sum / max / min
//                             partials (threshold_vabft.cpp:54-61 inputs) —
//                             the A operand is never re-read from HBM.
//                        2. verify tail: A-row statistics -> V-ABFT T_i
//                           (exactness guard + sequential fallback), blocked:128
//                           combination of both partial sets, D1/D2, strict
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

__device__ __forceinline__ uint32_t pminu2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
template <int F>
__device__ __forceinline__ uint32_t pmax2(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (F == VABFT_BF16) asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
template <int F>
__device__ __forceinline__ uint32_t pmin2(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (F == VABFT_BF16) asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// n * max|x| < 2^(53 + lsb(min nonzero |x|)) => plain FP64 sums are exact in
// any order (see aside.cu); mnz_pat is (smallest nonzero magnitude - 1).
template <int F>
__device__ __forceinline__ bool guard_exact(float max_abs, uint32_t mnz_pat, int64_t n) {
    if (mnz_pat >= 0x7FFFu) return true;
    if (!isfinite(max_abs)) return false;
    const uint32_t pat = mnz_pat + 1;
    int lsb;
    if constexpr (F == VABFT_BF16) {
        const int ef = int((pat >> 7) & 0xFF);
        lsb = (ef == 0 ? 1 : ef) - 127 - 7;
    } else {
        const int ef = int((pat >> 10) & 0x1F);
        lsb = (ef == 0 ? 1 : ef) - 15 - 10;
    }
    const int top = ilogbf(max_abs) + 1 + (64 - __clzll(static_cast<unsigned long long>(n)));
    return top <= 53 + lsb;
}

struct TailArgs {
    int64_t M, N, K, nblkN, nblkK;
    const uint16_t* A;
    const float *part1, *part2;            // [nblkN][M] C row partials
    const float *sp1, *sp2;                // [nblkK][M] A (B r) partials
    const double* ssum;                    // [nblkK][M]
    const uint32_t *smax, *smin, *smnz;    // [nblkK][M]
    const double* bsum;                    // B summary (4)
    double* cr1;                           // [M] staged checksums (phase 1 -> 2)
    double* cr2;
    double* Tv;                            // [M] V-ABFT thresholds
    double* max_abs_a;
    int method, aabft_t, quantize_cr;
    double e_max, c_sigma, aabft_fixed_y, aabft_conf, floor_scale;
    double* T_out;
    vabft_verdicts v;
    int64_t* counts;
};

// phase bit 1: A-row statistics -> T_i, A (B r); bit 2: row sums + verify.
// A CTA owns 32 rows: its 4 warps stage the [block][row] partial arrays
// through shared memory with coalesced loads (many loads in flight), then
// warp 0 (lane = row) combines them in block order — NativeBlocked(128) for
// the checksum and row-sum partials — and runs the verify rules.
constexpr int kTailRows = 32;
constexpr int kTailChunk = 16;

template <int F>
__global__ void __launch_bounds__(128) fused_tail_kernel(const TailArgs a, int phase) {
    __shared__ float s_p1[kTailChunk][kTailRows], s_p2[kTailChunk][kTailRows];
    __shared__ double s_sum[kTailChunk][kTailRows];
    __shared__ uint32_t s_max[kTailChunk][kTailRows], s_min[kTailChunk][kTailRows], s_mnz[kTailChunk][kTailRows];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row0 = int64_t(blockIdx.x) * kTailRows;
    const int64_t i = row0 + lane;
    const bool valid = warp == 0 && i < a.M;
    bool det = false, located = false, isnan_row = false;
    double c1 = 0.0, c2 = 0.0, tv = 0.0;
    if (phase & 1) {
        float t1 = 0.0f, t2 = 0.0f;
        double sum = 0.0;
        uint32_t gmax = F == VABFT_BF16 ? 0xFF80FF80u : 0xFC00FC00u;
        uint32_t gmin = F == VABFT_BF16 ? 0x7F807F80u : 0x7C007C00u;
        uint32_t gmnz = 0x7FFF7FFFu;
        for (int64_t b0 = 0; b0 < a.nblkK; b0 += kTailChunk) {
            for (int e = threadIdx.x; e < kTailChunk * kTailRows; e += blockDim.x) {
                const int bb = e / kTailRows, rr = e % kTailRows;
                const int64_t b = b0 + bb, row = row0 + rr;
                if (b < a.nblkK && row < a.M) {
                    const int64_t o = b * a.M + row;
                    s_p1[bb][rr] = __ldg(a.sp1 + o);
                    s_p2[bb][rr] = __ldg(a.sp2 + o);
                    s_sum[bb][rr] = __ldg(a.ssum + o);
                    s_max[bb][rr] = __ldg(a.smax + o);
                    s_min[bb][rr] = __ldg(a.smin + o);
                    s_mnz[bb][rr] = __ldg(a.smnz + o);
                }
            }
            __syncthreads();
            if (valid) {
                const int cnt = int((a.nblkK - b0) < kTailChunk ? (a.nblkK - b0) : kTailChunk);
                for (int bb = 0; bb < cnt; ++bb) {  // block order
                    t1 = __fadd_rn(t1, s_p1[bb][lane]);
                    t2 = __fadd_rn(t2, s_p2[bb][lane]);
                    sum = __dadd_rn(sum, s_sum[bb][lane]);
                    gmax = pmax2<F>(gmax, s_max[bb][lane]);
                    gmin = pmin2<F>(gmin, s_min[bb][lane]);
                    gmnz = pminu2(gmnz, s_mnz[bb][lane]);
                }
            }
            __syncthreads();
        }
        if (valid) {
            const float mx = fmaxf(bits16_to_float<F>(uint16_t(gmax & 0xFFFFu)), bits16_to_float<F>(uint16_t(gmax >> 16)));
            const float mn = fminf(bits16_to_float<F>(uint16_t(gmin & 0xFFFFu)), bits16_to_float<F>(uint16_t(gmin >> 16)));
            const uint32_t mnz = min(gmnz & 0xFFFFu, gmnz >> 16);
            const float amax = fmaxf(fabsf(mx), fabsf(mn));
            if (!guard_exact<F>(amax, mnz, a.K)) {
                // the reference's sequential Neumaier pass over the row (stats.cpp:12-24)
                Neu ns;
                const uint16_t* row = a.A + i * a.K;
                for (int64_t q = 0; q < a.K; ++q) ns.add(double(bits16_to_float<F>(row[q])));
                sum = __dadd_rn(ns.s, ns.c);
            }
            Neu fin;
            fin.s = sum;
            double mean, vb;
            stats_finish(fin, double(mx), double(mn), a.K, &mean, &vb);
            tv = vabft_threshold_total(mean, vb, a.bsum[0], a.bsum[1], a.bsum[2], a.N, a.e_max, a.c_sigma);
            if (a.quantize_cr) {
                t1 = bits16_to_float<F>(quantize16_bits<F>(t1));
                t2 = bits16_to_float<F>(quantize16_bits<F>(t2));
            }
            c1 = double(t1);
            c2 = double(t2);
            a.Tv[i] = tv;
            if (phase == 1) {
                a.cr1[i] = c1;
                a.cr2[i] = c2;
            }
        }
        if (warp == 0) {  // one atomic per warp for max|A|
            float amax = 0.0f;
            if (valid) amax = float(fmax(fabs(double(bits16_to_float<F>(uint16_t(gmax & 0xFFFFu)))),
                                         fabs(double(bits16_to_float<F>(uint16_t(gmin & 0xFFFFu))))));
            if (valid) amax = fmaxf(amax, fmaxf(fabsf(bits16_to_float<F>(uint16_t(gmax >> 16))),
                                                fabsf(bits16_to_float<F>(uint16_t(gmin >> 16)))));
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, m));
            if (lane == 0) atomic_max_nonneg(a.max_abs_a, double(amax));
        }
    }
    if (!(phase & 2)) return;
    float r1 = 0.0f, r2 = 0.0f;
    for (int64_t b0 = 0; b0 < a.nblkN; b0 += kTailChunk) {
        for (int e = threadIdx.x; e < kTailChunk * kTailRows; e += blockDim.x) {
            const int bb = e / kTailRows, rr = e % kTailRows;
            const int64_t b = b0 + bb, row = row0 + rr;
            if (b < a.nblkN && row < a.M) {
                const int64_t o = b * a.M + row;
                s_p1[bb][rr] = __ldg(a.part1 + o);
                s_p2[bb][rr] = __ldg(a.part2 + o);
            }
        }
        __syncthreads();
        if (valid) {
            const int cnt = int((a.nblkN - b0) < kTailChunk ? (a.nblkN - b0) : kTailChunk);
            for (int bb = 0; bb < cnt; ++bb) {  // reduce_terms NativeBlocked(128), in order
                r1 = __fadd_rn(r1, s_p1[bb][lane]);
                r2 = __fadd_rn(r2, s_p2[bb][lane]);
            }
        }
        __syncthreads();
    }
    if (warp != 0) return;
    if (valid) {
        if (!(phase & 1)) {
            c1 = a.cr1[i];
            c2 = a.cr2[i];
            tv = a.Tv[i];
        }
        double t;
        if (a.method == 0) {
            t = tv;
        } else {
            const double y = a.method == 1 ? a.aabft_fixed_y : __dmul_rn(*a.max_abs_a, a.bsum[3]);
            t = aabft_total(a.K, a.aabft_t, y, a.aabft_conf);
        }
        if (a.T_out) a.T_out[i] = t;
        const double d1 = __dsub_rn(double(r1), c1);
        const double d2 = __dsub_rn(double(r2), c2);
        int64_t loc = -1;
        double res = 0.0;
        if (isnan(d1) || isnan(d2)) {
            det = true;
            isnan_row = true;
        } else {
            det = fabs(d1) > t;
            if (det && fabs(d1) > __dmul_rn(a.floor_scale, t)) {
                int64_t j;
                double rr;
                if (localize_dev(d1, d2, a.N, &j, &rr)) {
                    loc = j;
                    res = rr;
                    located = true;
                }
            }
        }
        if (a.v.diff1) a.v.diff1[i] = d1;
        if (a.v.diff2) a.v.diff2[i] = d2;
        if (a.v.detected) a.v.detected[i] = det ? 1 : 0;
        if (a.v.location) a.v.location[i] = loc;
        if (a.v.residual) a.v.residual[i] = res;
    }
    if (a.counts) {
        const unsigned mv = __ballot_sync(0xffffffffu, valid);
        const unsigned md = __ballot_sync(0xffffffffu, det);
        const unsigned ml = __ballot_sync(0xffffffffu, located);
        const unsigned mn = __ballot_sync(0xffffffffu, isnan_row);
        if (lane == 0) {
            if (mv) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_ROWS), __popc(mv));
            if (md) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_DETECTED), __popc(md));
            if (ml) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_LOCATED), __popc(ml));
            if (mn) atomicAdd(reinterpret_cast<unsigned long long*>(a.counts + VABFT_COUNT_NAN), __popc(mn));
        }
    }
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct FusedWs {
    float *part1, *part2, *sp1, *sp2;
    double* ssum;
    uint32_t *smax, *smin, *smnz;
    double *cr1, *cr2, *Tv, *max_abs_a;
    size_t bytes;
};

FusedWs carve(void* base, int64_t M, int64_t N, int64_t K) {
    const size_t nN = size_t((N + 127) / 128), nK = size_t((K + 127) / 128), m = size_t(M);
    FusedWs w{};
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t sz) {
        char* p = b ? b + off : nullptr;
        off += align_up(sz);
        return p;
    };
    w.part1 = reinterpret_cast<float*>(take(4 * nN * m));
    w.part2 = reinterpret_cast<float*>(take(4 * nN * m));
    w.sp1 = reinterpret_cast<float*>(take(4 * nK * m));
    w.sp2 = reinterpret_cast<float*>(take(4 * nK * m));
    w.ssum = reinterpret_cast<double*>(take(8 * nK * m));
    w.smax = reinterpret_cast<uint32_t*>(take(4 * nK * m));
    w.smin = reinterpret_cast<uint32_t*>(take(4 * nK * m));
    w.smnz = reinterpret_cast<uint32_t*>(take(4 * nK * m));
    w.cr1 = reinterpret_cast<double*>(take(8 * m));
    w.cr2 = reinterpret_cast<double*>(take(8 * m));
    w.Tv = reinterpret_cast<double*>(take(8 * m));
    w.max_abs_a = reinterpret_cast<double*>(take(8));
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
        if (!bytes) fail(VABFT_INVALID_ARGUMENT, "null bytes");
        if (m < 1 || n < 1 || k < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        *bytes = carve(nullptr, m, n, k).bytes;
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
        if (k % 8 != 0 || n % 8 != 0) fail(VABFT_UNSUPPORTED, "vabft_fused_gemm: K and N must be multiples of 8");
        const FusedWs ws = carve(workspace, m, n, k);
        if (!workspace || ws_bytes < ws.bytes) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: workspace too small");
        cudaStream_t s = as_stream(stream);
        const bool offline = o->mode == VABFT_OFFLINE;
        const int stages = o->stages == 0 ? 7 : o->stages;
        if (stages & 2) {
            TcEpilogue epi;
            epi.abft = offline ? 2 : 1;
            epi.part1 = ws.part1;
            epi.part2 = ws.part2;
            epi.fault_col = o->fault_col;
            epi.fault_bit = o->fault_bit;
            epi.fault_dir = o->fault_dir;
            epi.fault_records = o->fault_records;
            epi.br1 = h->buf.br1;
            epi.br2 = h->buf.br2;
            epi.sp1 = ws.sp1;
            epi.sp2 = ws.sp2;
            epi.ssum = ws.ssum;
            epi.smax = ws.smax;
            epi.smin = ws.smin;
            epi.smnz = ws.smnz;
            tc_gemm_launch(h->fmt, o->b_kmajor != 0, m, n, k, A, h->B, C, epi, s);
        }
        if (!(stages & 4)) return;
        TailArgs a;
        a.M = m;
        a.N = n;
        a.K = k;
        a.nblkN = (n + 127) / 128;
        a.nblkK = (k + 127) / 128;
        a.A = static_cast<const uint16_t*>(A);
        a.part1 = ws.part1;
        a.part2 = ws.part2;
        a.sp1 = ws.sp1;
        a.sp2 = ws.sp2;
        a.ssum = ws.ssum;
        a.smax = ws.smax;
        a.smin = ws.smin;
        a.smnz = ws.smnz;
        a.bsum = h->buf.summary;
        a.cr1 = ws.cr1;
        a.cr2 = ws.cr2;
        a.Tv = (T && o->threshold_method == 0) ? T : ws.Tv;
        a.max_abs_a = ws.max_abs_a;
        a.method = o->threshold_method;
        a.aabft_t = o->aabft_mantissa_bits > 0 ? o->aabft_mantissa_bits : (h->fmt == VABFT_BF16 ? 8 : 11);
        a.quantize_cr = offline ? 1 : 0;
        a.e_max = o->e_max;
        a.c_sigma = o->c_sigma;
        a.aabft_fixed_y = o->aabft_fixed_y;
        a.aabft_conf = o->aabft_confidence > 0 ? o->aabft_confidence : 3.0;
        a.floor_scale = o->floor_scale;
        a.T_out = T;
        a.v = verdicts;
        a.counts = counts;
        const unsigned grid = unsigned((m + kTailRows - 1) / kTailRows);
        check_cuda(cudaMemsetAsync(ws.max_abs_a, 0, sizeof(double), s), "memset");
        // computed-y A-ABFT needs the global max|A| before any verdict
        const bool two_phase = o->threshold_method == 2;
        if (h->fmt == VABFT_BF16) {
            if (two_phase) {
                fused_tail_kernel<VABFT_BF16><<<grid, 128, 0, s>>>(a, 1);
                fused_tail_kernel<VABFT_BF16><<<grid, 128, 0, s>>>(a, 2);
            } else {
                fused_tail_kernel<VABFT_BF16><<<grid, 128, 0, s>>>(a, 3);
            }
        } else {
            if (two_phase) {
                fused_tail_kernel<VABFT_FP16><<<grid, 128, 0, s>>>(a, 1);
                fused_tail_kernel<VABFT_FP16><<<grid, 128, 0, s>>>(a, 2);
            } else {
                fused_tail_kernel<VABFT_FP16><<<grid, 128, 0, s>>>(a, 3);
            }
        }
        check_cuda(cudaGetLastError(), "fused tail launch");
    });
}
