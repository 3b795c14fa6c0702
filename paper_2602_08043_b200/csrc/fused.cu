// The hot path: V-ABFT fused GEMM (TENSOR engine) — ONE persistent kernel.
//
//   vabft_bside_create   per-weight B state: precompute_b_stats +
//                        BStatsSummary::from (threshold_vabft.cpp:8-26), B r1 /
//                        B r2 (checksum.cpp:110-115), max_k |sum_j B| for A-ABFT
//                        computed y (threshold_aabft.cpp:38-48).
//   vabft_fused_gemm     tc_gemm (tcgen05), cooperative persistent launch:
//                         - MMA: C = A B, FP32 accumulators in TMEM;
//                         - epilogue warps: per-128-column row partials of the
//                           FP32 accumulator (online) or of the quantized output
//                           (offline), optional in-epilogue fault injection
//                           (faults.cpp:104-168), C store;
//                         - statistics warps: consume A tiles TMA-loaded into
//                           their own smem ring and produce per-(row, 128-k-
//                           block) A (B r) partials and exact row-sum / max / min
//                           partials (threshold_vabft.cpp:54-61);
//                         - after a grid barrier, every warp runs the verify
//                           tail (tail.cuh) on 32-row groups: A-row statistics
//                           -> V-ABFT T_i, blocked:128 combination of both
//                           partial sets, D1/D2, strict compare, NaN rule,
//                           localization (detect.cpp:9-55), counters.
// No host synchronization anywhere on this path.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "devcommon.cuh"
#include "exact.hpp"
#include "guard.hpp"
#include "internal.hpp"
#include "numerics.cuh"
#include "stats.hpp"
#include "tail.cuh"

struct vabft_bside {
    int fmt;
    int mode;
    int b_kmajor;
    int64_t k, n;
    int64_t ldb = 0;  // row stride of B (elements): n unless created by vabft_bside_create_ld
    const void* B;  // not owned
    vabft_dev::BsideBuffers buf;
    void* storage;  // one cudaMalloc holding every buffer
    unsigned int* gbar;  // grid-barrier state of the fused kernel (inside storage)
    // wide formats (FP32 / FP64): B r1 / B r2 in the working type (held as doubles)
    double* brd = nullptr;  // [2][K]
    bool rowsum_ready = false;  // wide formats: rowsum_abs / summary[3] (A-ABFT computed y) built
    // FP32 (3xTF32): the weight split once into hi / lo parts, transposed
    // ([2][N][K], K-major for kind::tf32), and
    // the activation's split buffers [2][M][K], grown on demand
    float* b_split = nullptr;
    float* a_split = nullptr;
    size_t a_split_elems = 0;
};

namespace vabft_dev {

namespace {

void destroy_bside(vabft_bside* h) {
    if (h->storage) cudaFree(h->storage);
    if (h->brd) cudaFree(h->brd);
    if (h->b_split) cudaFree(h->b_split);
    if (h->a_split) cudaFree(h->a_split);
    delete h;
}

// Workspace state across launches. The per-row statistics atomics and the
// streamed-verification counters of a 16-bit fused workspace hold their
// identities after every complete launch (the verify tail restores them), so
// a workspace the same handle used last at the same shape is launched without
// resetting anything. Any other history — first use, another handle, an
// FP32 / FP64 launch (whose carve overlays the same bytes), a stage-masked
// launch that ran the statistics warps without the tail, or
// vabft_fused_opts.workspace_fresh — resets them first (~20 B per row).
std::mutex g_ws_mu;
std::map<const void*, std::pair<const vabft_bside*, size_t>> g_ws_owner;  // workspace -> (handle, bytes)

// true when the workspace needs its identities written before this launch
bool claim_workspace(const void* ws, const vabft_bside* h, size_t bytes, bool fresh) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_ws_owner.find(ws);
    const bool ready = !fresh && it != g_ws_owner.end() && it->second.first == h && it->second.second == bytes;
    g_ws_owner[ws] = {h, bytes};
    return !ready;
}
void release_workspace(const void* ws) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    g_ws_owner.erase(ws);
}
void forget_workspaces(const vabft_bside* h) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto it = g_ws_owner.begin(); it != g_ws_owner.end();)
        it = it->second.first == h ? g_ws_owner.erase(it) : std::next(it);
}

// Standalone tail (profiling stage mask 4 without 2): 4 warps per CTA, one
// 32-row group per warp, each with its own 24 KiB shared-memory slice.
template <int F>
__global__ void __launch_bounds__(128) fused_tail_kernel(const TailArgs a, int phase) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bars[4];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        mbar_init(smem_u32(&bars[w]), 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t g = int64_t(blockIdx.x) * 4 + w;
    if (g * 32 >= a.M) return;
    uint32_t ph = 0;
    verify_rowgroup<F>(a, g, phase, reinterpret_cast<float*>(sm + size_t(w) * kTailWarpSmem),
                       smem_u32(&bars[w]), ph);
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct FusedWs {
    float *part1, *part2, *sp1, *sp2;
    double* rsum;                      // [M] per-row atomics (identities: 0, 0, ~0, ~0)
    uint32_t *rmax, *rmin, *rmnz;
    double *cr1, *cr2, *Tv, *max_abs_a;
    unsigned int* group_cnt;           // [ceil(M/32)][2] streamed-verification arrivals (identity 0)
    size_t bytes;
};

FusedWs carve(void* base, int64_t M, int64_t N, int64_t K) {
    const size_t nN = size_t((N + 127) / 128), nK = size_t((K + 127) / 128), m = size_t(M);
    const size_t ld = (m + 31) / 32 * 32;  // rows padded to whole 32-row groups
    FusedWs w{};
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t sz) {
        char* p = b ? b + off : nullptr;
        off += align_up(sz);
        return p;
    };
    w.part1 = reinterpret_cast<float*>(take(4 * nN * ld));
    w.part2 = reinterpret_cast<float*>(take(4 * nN * ld));
    w.sp1 = reinterpret_cast<float*>(take(4 * nK * ld));
    w.sp2 = reinterpret_cast<float*>(take(4 * nK * ld));
    w.rsum = reinterpret_cast<double*>(take(8 * m));
    w.rmax = reinterpret_cast<uint32_t*>(take(4 * m));
    w.rmin = reinterpret_cast<uint32_t*>(take(4 * m));  // rmin, rmnz adjacent: one 0xFF memset
    w.rmnz = reinterpret_cast<uint32_t*>(take(4 * m));
    w.cr1 = reinterpret_cast<double*>(take(8 * m));
    w.cr2 = reinterpret_cast<double*>(take(8 * m));
    w.Tv = reinterpret_cast<double*>(take(8 * m));
    w.max_abs_a = reinterpret_cast<double*>(take(8));
    w.group_cnt = reinterpret_cast<unsigned int*>(take(4 * 2 * (ld / 32)));
    w.bytes = off;
    return w;
}

// Workspace of the wide-format (FP32 / FP64) path, carved from the same buffer.
struct WideWs {
    void *part1, *part2;  // [ceil(N/128)][ld] working type
    void* cpart;          // [7][ceil(K/128)][ld] A-side block partials (wide.cu)
    int64_t ld;
    double *mean, *mx, *mn, *vb, *cr1, *cr2, *max_abs_a;
    unsigned* gcnt;       // [ld / 32] A-pass arrival counters (zero at rest)
    size_t bytes;
};

WideWs carve_wide(void* base, int64_t M, int64_t N, int64_t K) {
    const size_t nN = size_t((N + 127) / 128), nK = size_t((K + 127) / 128), m = size_t(M);
    const size_t ld = (m + 31) / 32 * 32;
    WideWs w{};
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t sz) {
        char* p = b ? b + off : nullptr;
        off += align_up(sz);
        return p;
    };
    w.ld = int64_t(ld);
    w.part1 = take(8 * nN * ld);
    w.part2 = take(8 * nN * ld);
    w.cpart = take(7 * 8 * nK * ld);
    w.mean = reinterpret_cast<double*>(take(8 * m));
    w.mx = reinterpret_cast<double*>(take(8 * m));
    w.mn = reinterpret_cast<double*>(take(8 * m));
    w.vb = reinterpret_cast<double*>(take(8 * m));
    w.cr1 = reinterpret_cast<double*>(take(8 * m));
    w.cr2 = reinterpret_cast<double*>(take(8 * m));
    w.max_abs_a = reinterpret_cast<double*>(take(8));
    w.gcnt = reinterpret_cast<unsigned*>(take(4 * (ld / 32)));
    w.bytes = off;
    return w;
}

bool is_wide(int fmt) { return fmt == VABFT_FP32 || fmt == VABFT_FP64; }


// vabft_fused_gemm for FP32 / FP64: the GEMM with the ABFT epilogue, the
// A-side pass (row statistics and A (B r) block partials, one read of A) and
// the verify tail, stream-ordered.
void wide_fused(const vabft_fused_opts* o, vabft_bside* h, int64_t m, const void* A, void* C, double* T,
                const vabft_verdicts& verdicts, int64_t* counts, void* workspace, cudaStream_t s) {
    if (o->tf32_passes != 0 && o->tf32_passes != 1 && o->tf32_passes != 3)
        fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: tf32_passes must be 0, 1 or 3");
    const int64_t n = h->n, k = h->k;
    const WideWs ws = carve_wide(workspace, m, n, k);
    const int stages = o->stages == 0 ? 7 : o->stages;
    const bool tail = (stages & 4) != 0;
    if (o->fault_target == 1 && (!o->fault_col || !o->fault_bit || !o->fault_dir))
        fail(VABFT_INVALID_ARGUMENT, "InputA faults need fault_col / fault_bit / fault_dir");
    if (o->fault_target == 2 && o->n_operand_faults > 0 && !o->operand_faults)
        fail(VABFT_INVALID_ARGUMENT, "InputB faults need operand_faults");
    if (stages & 2) {
        WideEpilogue epi;
        epi.abft = (stages & 8) ? 0 : 1;  // bit 8: the same GEMM with the ABFT epilogue off (overhead baseline)
        epi.part1 = ws.part1;
        epi.part2 = ws.part2;
        epi.ld = ws.ld;
        if (o->fault_target == 0) {
            epi.fault_col = o->fault_col;
            epi.fault_bit = o->fault_bit;
            epi.fault_dir = o->fault_dir;
            epi.fault_records = o->fault_records;
        }
        // Operand faults (FaultTarget InputA / InputB, faults.hpp:15): the GEMM
        // multiplies a copy of the operand with the planned bits flipped (what
        // the FP64 pipe / tensor cores see), while the A side and the checksums
        // read the clean operands. Campaign path: the copies come from the
        // stream-ordered allocator.
        const size_t es = h->fmt == VABFT_FP64 ? 8 : 4;
        const void* Ag = A;
        const void* Bg = h->B;
        void* scratch = nullptr;
        if (o->fault_target == 1) {
            check_cuda(cudaMallocAsync(&scratch, es * size_t(m) * size_t(k), s), "cudaMallocAsync(A')");
            check_cuda(cudaMemcpyAsync(scratch, A, es * size_t(m) * size_t(k), cudaMemcpyDeviceToDevice, s), "copy");
            launch_flip_rows(h->fmt, scratch, m, k, o->fault_col, o->fault_bit, o->fault_dir, o->fault_records, s);
            Ag = scratch;
        } else if (o->fault_target == 2 && o->n_operand_faults > 0) {
            // B' plus, for FP32, its transposed TF32 split
            const size_t nb = size_t(k) * size_t(n), extra = h->fmt == VABFT_FP32 ? 2 * nb : 0;
            check_cuda(cudaMallocAsync(&scratch, es * (nb + extra), s), "cudaMallocAsync(B')");
            check_cuda(cudaMemcpyAsync(scratch, h->B, es * nb, cudaMemcpyDeviceToDevice, s), "copy");
            launch_inject(h->fmt, n, scratch, o->operand_faults, o->n_operand_faults, o->operand_fault_records, s);
            Bg = scratch;
            if (h->fmt == VABFT_FP32) {
                float* t = static_cast<float*>(scratch) + nb;
                split_tf32_t(static_cast<const float*>(scratch), t, t + nb, k, n, s);
            }
        }
        const float* bsplit = (o->fault_target == 2 && o->n_operand_faults > 0 && h->fmt == VABFT_FP32)
                                  ? static_cast<const float*>(Bg) + size_t(k) * size_t(n)
                                  : h->b_split;
        if (h->fmt == VABFT_FP64) {
            dgemm_launch(m, n, k, static_cast<const double*>(Ag), static_cast<const double*>(Bg),
                         static_cast<double*>(C), epi, s);
        } else if (o->tf32_passes == 1) {
            tf32_gemm_launch(m, n, k, static_cast<const float*>(Ag), nullptr, bsplit, nullptr,
                             static_cast<float*>(C), epi, s);
        } else {
            const size_t need = 2 * size_t(m) * size_t(k);
            if (h->a_split_elems < need) {
                if (h->a_split) check_cuda(cudaFreeAsync(h->a_split, s), "cudaFreeAsync");
                h->a_split = nullptr;
                h->a_split_elems = 0;
                check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&h->a_split), need * sizeof(float), s),
                           "cudaMallocAsync(A split)");
                h->a_split_elems = need;
            }
            float* ahi = h->a_split;
            float* alo = h->a_split + size_t(m) * size_t(k);
            split_tf32(static_cast<const float*>(Ag), ahi, alo, m * k, s);
            tf32_gemm_launch(m, n, k, ahi, alo, bsplit, bsplit + size_t(k) * size_t(n), static_cast<float*>(C), epi, s);
        }
        if (scratch) check_cuda(cudaFreeAsync(scratch, s), "cudaFreeAsync");
    }
    if (!tail) return;
    // the A pass verifies each row group as it completes; A-ABFT computed y
    // needs the global max|A| first: stage the statistics, then a tail kernel
    const bool global_y = o->threshold_method == 2;
    if (global_y && !h->rowsum_ready) {  // max_k |sum_j B[k][j]| on first use (bside.cu)
        launch_bside_rowsum(h->fmt, h->k, h->n, h->B, h->buf, s, h->ldb);
        h->rowsum_ready = true;
    }
    if (claim_workspace(workspace, h, ws.bytes, o->workspace_fresh != 0))
        check_cuda(cudaMemsetAsync(ws.gcnt, 0, sizeof(unsigned) * size_t(ws.ld / 32), s), "memset");
    WideTail t{};
    t.M = m;
    t.N = n;
    t.K = k;
    t.nblk = (n + 127) / 128;
    t.ld = ws.ld;
    t.fmt = h->fmt;
    t.part1 = ws.part1;
    t.part2 = ws.part2;
    t.mean = ws.mean;
    t.vb = ws.vb;
    t.cr1 = ws.cr1;
    t.cr2 = ws.cr2;
    t.bsum = h->buf.summary;
    t.max_abs_a = ws.max_abs_a;
    t.method = o->threshold_method;
    t.t_in = o->t_in;
    t.ldt = o->ldt ? o->ldt : 1;
    t.aabft_t = o->aabft_mantissa_bits > 0 ? o->aabft_mantissa_bits : (h->fmt == VABFT_FP64 ? 53 : 23);
    t.e_max = o->e_max;
    t.c_sigma = o->c_sigma;
    t.aabft_fixed_y = o->aabft_fixed_y;
    t.aabft_conf = o->aabft_confidence > 0 ? o->aabft_confidence : 3.0;
    t.floor_scale = o->floor_scale;
    t.T_out = T;
    t.v = verdicts;
    t.counts = counts;
    t.C = C;
    t.correct = o->correct;
    t.A = A;
    t.qfmt = o->mode == VABFT_OFFLINE ? h->fmt : -1;
    const bool f32 = h->fmt == VABFT_FP32;  // B r in the working type: the pass's float copies for FP32
    launch_wide_aside(t, f32 ? static_cast<const void*>(h->buf.br1) : h->brd,
                      f32 ? static_cast<const void*>(h->buf.br2) : h->brd + k, ws.cpart, ws.gcnt, !global_y, ws.mean,
                      ws.vb, ws.mx, ws.mn, ws.cr1, ws.cr2, s);
    if (!global_y) return;
    check_cuda(cudaMemsetAsync(ws.max_abs_a, 0, sizeof(double), s), "memset");
    launch_max_abs_rows(m, ws.mx, ws.mn, ws.max_abs_a, s);
    launch_wide_tail(t, s);
}

}  // namespace
}  // namespace vabft_dev

using namespace vabft_dev;

extern "C" vabft_status vabft_bside_create(int32_t format, int32_t mode, int64_t k, int64_t n,
                                           const void* B, vabft_bside_t* out, void* stream) {
    return vabft_bside_create_ld(format, mode, k, n, B, 0, out, stream);
}

extern "C" vabft_status vabft_bside_create_ld(int32_t format, int32_t mode, int64_t k, int64_t n, const void* B,
                                              int64_t ldb, vabft_bside_t* out, void* stream) {
    return guarded([&] {
        if (ldb == 0) ldb = n;
        if (ldb < n) fail(VABFT_INVALID_ARGUMENT, "vabft_bside_create_ld: ldb < n");
        if (ldb != n && (format == VABFT_FP32 || format == VABFT_FP64))
            fail(VABFT_UNSUPPORTED, "vabft_bside_create_ld: strided weights are BF16 / FP16 only");
        if (!out) fail(VABFT_INVALID_ARGUMENT, "vabft_bside_create: null handle pointer");
        if (format < VABFT_BF16 || format > VABFT_FP64) fail(VABFT_INVALID_ARGUMENT, "bad format");
        if (mode != VABFT_OFFLINE && mode != VABFT_ONLINE) fail(VABFT_INVALID_ARGUMENT, "bad mode");
        if (k < 1 || n < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        // ChecksumVectors::make: weights exact in FP32 (checksum.cpp:26-34)
        if (n > (int64_t(1) << 24)) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: weights exceed exact range");
        if (format == VABFT_FP32 && (k * n) % 4 != 0)
            fail(VABFT_UNSUPPORTED, "FP32 weights: K x N must be a multiple of 4");
        // owned until handed out: every early exit below frees what was allocated
        std::unique_ptr<vabft_bside, void (*)(vabft_bside*)> hp(new vabft_bside(), destroy_bside);
        vabft_bside* h = hp.get();
        h->fmt = format;
        h->mode = mode;
        h->b_kmajor = 0;
        h->k = k;
        h->n = n;
        h->ldb = ldb;
        h->B = B;
        const size_t K = size_t(k);
        const size_t KB = size_t(br_storage_floats(k));
        const size_t gw = bside_group_words(k);
        const size_t bytes = align_up(8 * K) * 3 + align_up(4 * KB) * 2 + align_up(8 * 4) + align_up(4) + align_up(8) +
                             align_up(4 * gw) + align_up(bside_work_bytes(format, k, n));
        check_cuda(cudaMalloc(&h->storage, bytes), "cudaMalloc(bside)");
        char* p = static_cast<char*>(h->storage);
        h->buf.mean = reinterpret_cast<double*>(p); p += align_up(8 * K);
        h->buf.vb = reinterpret_cast<double*>(p); p += align_up(8 * K);
        h->buf.rowsum_abs = reinterpret_cast<double*>(p); p += align_up(8 * K);
        h->buf.br1 = reinterpret_cast<float*>(p); p += align_up(4 * KB);
        h->buf.br2 = reinterpret_cast<float*>(p); p += align_up(4 * KB);
        h->buf.summary = reinterpret_cast<double*>(p); p += align_up(32);
        h->buf.nonfinite = reinterpret_cast<int*>(p); p += align_up(4);
        h->gbar = reinterpret_cast<unsigned int*>(p); p += align_up(8);
        h->buf.groups = reinterpret_cast<unsigned int*>(p); p += align_up(4 * gw);
        h->buf.work = p;
        // grid barrier, B-side group counters / flags and the non-finite flag start at zero
        check_cuda(cudaMemset(h->buf.nonfinite, 0, size_t(p - reinterpret_cast<char*>(h->buf.nonfinite))),
                   "memset(bside state)");
        bside_init_work(format, k, n, h->buf.work, nullptr);
        check_cuda(cudaDeviceSynchronize(), "bside init");
        if (is_wide(format)) {
            check_cuda(cudaMalloc(&h->brd, 2 * sizeof(double) * K), "cudaMalloc(bside B r)");
            h->buf.brd1 = h->brd;
            h->buf.brd2 = h->brd + K;
            if (format == VABFT_FP32) {
                check_cuda(cudaMalloc(&h->b_split, 2 * sizeof(float) * K * size_t(n)), "cudaMalloc(B split)");
                // the B-side pass writes the transposed TF32 split as it streams B
                h->buf.split_hi = h->b_split;
                h->buf.split_lo = h->b_split + K * size_t(n);
            }
        }
        if (B) {
            launch_bside(format, k, n, B, mode == VABFT_OFFLINE ? 1 : 0, h->buf, as_stream(stream), ldb);
        }
        *out = hp.release();
    });
}

extern "C" vabft_status vabft_bside_update(vabft_bside_t h, const void* B, void* stream) {
    return guarded([&] {
        if (!h || !B) fail(VABFT_INVALID_ARGUMENT, "vabft_bside_update: null argument");
        h->B = B;
        h->rowsum_ready = false;
        launch_bside(h->fmt, h->k, h->n, B, h->mode == VABFT_OFFLINE ? 1 : 0, h->buf, as_stream(stream), h->ldb);
    });
}

extern "C" vabft_status vabft_bside_destroy(vabft_bside_t h) {
    return guarded([&] {
        if (!h) return;
        forget_workspaces(h);
        destroy_bside(h);
    });
}

extern "C" vabft_status vabft_fused_workspace_size(int64_t m, int64_t n, int64_t k, size_t* bytes) {
    return guarded([&] {
        if (!bytes) fail(VABFT_INVALID_ARGUMENT, "null bytes");
        if (m < 1 || n < 1 || k < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        *bytes = std::max(carve(nullptr, m, n, k).bytes, carve_wide(nullptr, m, n, k).bytes);
    });
}


extern "C" vabft_status vabft_fused_gemm(const vabft_fused_opts* o, vabft_bside_t h, int64_t m,
                                         const void* A, void* C, double* T, vabft_verdicts verdicts,
                                         int64_t* counts, void* workspace, size_t ws_bytes,
                                         void* stream) {
    // a launch that fails after the workspace was claimed may leave its
    // counters (per-row atomics, arrival counters, the A pass's task counter)
    // mid-flight: forget the claim so the next call resets them
    struct ReleaseOnError {
        const void* ws;
        bool armed = true;
        ~ReleaseOnError() {
            if (armed) release_workspace(ws);
        }
    } on_error{workspace};
    const vabft_status st = guarded([&] {
        if (!o || !h || !A || !C || !h->B) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: null argument");
        if (o->mode != h->mode) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: mode differs from the B-side handle");
        if (o->threshold_method < 0 || o->threshold_method > 3) fail(VABFT_INVALID_ARGUMENT, "bad threshold method");
        if (o->threshold_method == 3 && !o->t_in) fail(VABFT_INVALID_ARGUMENT, "threshold method 3 needs t_in");
        if (o->b_kmajor != h->b_kmajor)
            fail(VABFT_UNSUPPORTED, "vabft_fused_gemm: B layout differs from the B-side handle");
        if (m < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        if (m > (int64_t(1) << 24)) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: weights exceed exact range");
        const int64_t n = h->n, k = h->k;
        if (k % 8 != 0 || n % 8 != 0) fail(VABFT_UNSUPPORTED, "vabft_fused_gemm: K and N must be multiples of 8");
        const int64_t lda = o->lda ? o->lda : k, ldc = o->ldc ? o->ldc : n;
        if (lda < k || ldc < n) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: lda < K or ldc < N");
        if (is_wide(h->fmt) && (lda != k || ldc != n))
            fail(VABFT_UNSUPPORTED, "vabft_fused_gemm: strided A / C are BF16 / FP16 only");
        const size_t need = std::max(carve(nullptr, m, n, k).bytes, carve_wide(nullptr, m, n, k).bytes);
        if (!workspace || ws_bytes < need) fail(VABFT_INVALID_ARGUMENT, "vabft_fused_gemm: workspace too small");
        cudaStream_t s = as_stream(stream);
        if (o->fault_target < 0 || o->fault_target > 2) fail(VABFT_INVALID_ARGUMENT, "bad fault target");
        if (is_wide(h->fmt)) {
            wide_fused(o, h, m, A, C, T, verdicts, counts, workspace, s);
            return;
        }
        const FusedWs ws = carve(workspace, m, n, k);
        const bool offline = o->mode == VABFT_OFFLINE;
        const int stages = o->stages == 0 ? 7 : o->stages;

        TailArgs a;
        a.M = m;
        a.N = n;
        a.K = k;
        a.nblkN = (n + 127) / 128;
        a.nblkK = (k + 127) / 128;
        a.A = static_cast<const uint16_t*>(A);
        a.lda = lda;
        a.ldc = ldc;
        a.part1 = ws.part1;
        a.part2 = ws.part2;
        a.sp1 = ws.sp1;
        a.sp2 = ws.sp2;
        a.rsum = ws.rsum;
        a.rmax = ws.rmax;
        a.rmin = ws.rmin;
        a.rmnz = ws.rmnz;
        if (claim_workspace(workspace, h, ws.bytes, o->workspace_fresh != 0)) {
            // per-row atomics and group counters to their identities (the
            // verify tail restores them after every complete launch)
            check_cuda(cudaMemsetAsync(ws.rsum, 0, sizeof(double) * size_t(m), s), "memset");
            check_cuda(cudaMemsetAsync(ws.rmax, 0, sizeof(uint32_t) * size_t(m), s), "memset");
            check_cuda(cudaMemsetAsync(ws.rmin, 0xFF, size_t(reinterpret_cast<char*>(ws.rmnz + m) -
                                                             reinterpret_cast<char*>(ws.rmin)), s), "memset");
            check_cuda(cudaMemsetAsync(ws.group_cnt, 0, sizeof(unsigned int) * 2 * size_t((m + 31) / 32), s), "memset");
        }
        // a launch without the tail leaves the statistics atomics dirty
        if (!(stages & 4)) release_workspace(workspace);
        a.bsum = h->buf.summary;
        a.cr1 = ws.cr1;
        a.cr2 = ws.cr2;
        a.Tv = ws.Tv;
        a.max_abs_a = ws.max_abs_a;
        a.method = o->threshold_method;
        a.t_in = o->t_in;
        a.ldt = o->ldt ? o->ldt : 1;
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
        a.C = static_cast<uint16_t*>(C);
        a.correct = o->correct;
        if (o->fault_target < 0 || o->fault_target > 2) fail(VABFT_INVALID_ARGUMENT, "bad fault target");
        if (o->fault_target == 1 && (!o->fault_col || !o->fault_bit || !o->fault_dir))
            fail(VABFT_INVALID_ARGUMENT, "InputA faults need fault_col / fault_bit / fault_dir");
        if (o->fault_target == 2 && o->n_operand_faults > 0 && !o->operand_faults)
            fail(VABFT_INVALID_ARGUMENT, "InputB faults need operand_faults");
        // computed-y A-ABFT needs the global max|A| before any verdict: two passes
        const bool two_phase = o->threshold_method == 2;
        if (two_phase && (stages & 4)) check_cuda(cudaMemsetAsync(ws.max_abs_a, 0, sizeof(double), s), "memset");

        if (stages & 2) {
            TcEpilogue epi;
            epi.abft = offline ? 2 : 1;
            epi.part1 = ws.part1;
            epi.part2 = ws.part2;
            epi.fault_col = o->fault_col;
            epi.fault_bit = o->fault_bit;
            epi.fault_dir = o->fault_dir;
            epi.fault_records = o->fault_records;
            epi.fault_target = o->fault_target;
            epi.cta_mode = o->cta_mode;
            epi.n_operand_faults = o->n_operand_faults;
            epi.operand_faults = o->operand_faults;
            epi.operand_fault_records = o->operand_fault_records;
            epi.accum_out = o->accum_out;
            epi.br1 = h->buf.br1;
            epi.br2 = h->buf.br2;
            epi.sp1 = ws.sp1;
            epi.sp2 = ws.sp2;
            epi.rsum = ws.rsum;
            epi.rmax = ws.rmax;
            epi.rmin = ws.rmin;
            epi.rmnz = ws.rmnz;
            if (const char* dbg = std::getenv("VABFT_DEBUG_STATS")) epi.debug = std::atoi(dbg);
            if (stages & 4) {  // verification inside the same persistent kernel
                epi.tail = a;
                if (two_phase) {  // global max|A| first: grid-barrier tail in two passes
                    epi.tail_phases = 1;
                    epi.gbar = h->gbar;
                } else {          // streamed: each row group verified as it completes
                    epi.stream_verify = 1;
                    epi.group_cnt = ws.group_cnt;
                }
            }
            tc_gemm_launch(h->fmt, o->b_kmajor != 0, m, n, k, A, h->B, C, epi, s, lda, h->ldb, ldc);
            return;
        }
        if (!(stages & 4)) return;
        const unsigned grid = unsigned(((m + 31) / 32 + 3) / 4);
        const size_t smem = 4 * size_t(kTailWarpSmem);
        auto run = [&](auto kern) {
            ensure_smem_attr(reinterpret_cast<const void*>(kern), int(smem));
            if (two_phase) {
                kern<<<grid, 128, smem, s>>>(a, 1);
                kern<<<grid, 128, smem, s>>>(a, 2);
            } else {
                kern<<<grid, 128, smem, s>>>(a, 3);
            }
        };
        if (h->fmt == VABFT_BF16) run(fused_tail_kernel<VABFT_BF16>);
        else run(fused_tail_kernel<VABFT_FP16>);
        check_cuda(cudaGetLastError(), "fused tail launch");
    });
    if (st == VABFT_OK) on_error.armed = false;
    return st;
}

extern "C" int32_t vabft_fused_uses_cta_pairs(const vabft_fused_opts* o, int64_t m, int64_t n, int64_t k) {
    (void)m;
    (void)k;
    if (!o) return 0;
    TcEpilogue epi;
    epi.sp1 = reinterpret_cast<float*>(1);  // the fused kernel (statistics warps present)
    epi.fault_col = o->fault_col;
    epi.fault_target = o->fault_target;
    epi.n_operand_faults = o->n_operand_faults;
    epi.tail_phases = o->threshold_method == 2 ? 1 : 0;
    epi.cta_mode = o->cta_mode;
    return tc_gemm_uses_pairs(o->b_kmajor != 0, n, epi) ? 1 : 0;
}

