// Device C-ABI entry points that mirror the reference's value-level API
// (encode_and_multiply, row_sums, row_stats, vabft_thresholds,
// aabft_threshold, verify, inject). Temporaries come from the stream-ordered
// allocator; only entry points that must report data-dependent errors the
// reference throws (non-finite stats, negative thresholds, A-ABFT y) wait on
// the stream.
#include <cmath>
#include <mutex>
#include <vector>

#include "devcommon.cuh"
#include "exact.hpp"
#include "guard.hpp"
#include "internal.hpp"
#include "stats.hpp"

using namespace vabft_dev;

namespace {

// The stream-ordered pool keeps up to 1 GiB of freed temporaries mapped
// (default release threshold 0: every synchronising entry point handed its
// pages back and the next call re-mapped them — measured ~0.3-2.5 ms of host
// time per block-wise threshold call). Once per device.
void keep_pool_mapped() {
    static std::mutex mu;
    static std::vector<bool> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(mu);
    if (size_t(dev) >= done.size()) done.resize(size_t(dev) + 1, false);
    if (done[size_t(dev)]) return;
    done[size_t(dev)] = true;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = uint64_t(1) << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
}

struct Tmp {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Tmp(cudaStream_t st) : s(st) { keep_pool_mapped(); }
    template <class T>
    T* get(size_t count) {
        void* p = nullptr;
        check_cuda(cudaMallocAsync(&p, count * sizeof(T) + 16, s), "cudaMallocAsync");
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Tmp() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
};

void check_fmt(int f) {
    if (f < VABFT_BF16 || f > VABFT_FP64) fail(VABFT_INVALID_ARGUMENT, "bad format");
}

// checksum_precision_for (checksum.cpp:18-24)
void cs_prec(const vabft_precision& in, int mode, int* fmt, vabft_accum* acc) {
    *acc = in.accumulation;
    *fmt = mode == VABFT_OFFLINE ? in.format : (in.format == VABFT_FP64 ? VABFT_FP64 : VABFT_FP32);
}

// ChecksumVectors::make (checksum.cpp:26-34)
void check_weights(int64_t n, int fmt, int kind) {
    if (n < 1) fail(VABFT_INVALID_ARGUMENT, "ChecksumVectors: length must be >= 1");
    const int t = accumulates_in_float(fmt, kind) ? 24 : 53;
    if (n > (int64_t(1) << t))
        fail(VABFT_INVALID_ARGUMENT,
             "ChecksumVectors: position weights exceed the exact-integer range of the checksum precision");
}

// Stream-ordered B-side buffers for one call (the handle-less entry points).
BsideBuffers tmp_bside(Tmp& tmp, int fmt, int64_t k, int64_t n, cudaStream_t s) {
    BsideBuffers buf;
    buf.mean = tmp.get<double>(k);
    buf.vb = tmp.get<double>(k);
    buf.rowsum_abs = tmp.get<double>(k);
    buf.br1 = tmp.get<float>(size_t(br_storage_floats(k)));
    buf.br2 = tmp.get<float>(size_t(br_storage_floats(k)));
    buf.summary = tmp.get<double>(4);
    buf.nonfinite = tmp.get<int>(1);
    buf.groups = tmp.get<unsigned>(bside_group_words(k));
    buf.work = tmp.get<char>(bside_work_bytes(fmt, k, n));
    check_cuda(cudaMemsetAsync(buf.nonfinite, 0, sizeof(int), s), "memset");
    check_cuda(cudaMemsetAsync(buf.groups, 0, sizeof(unsigned) * bside_group_words(k), s), "memset");
    bside_init_work(fmt, k, n, buf.work, s);
    return buf;
}

__global__ void thresholds_from_stats_kernel(int64_t m, int64_t n, const double* mean,
                                             const double* vb, const double* bsum, double e_max,
                                             double c_sigma, double* T) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) T[i] = vabft_threshold_total(mean[i], vb[i], bsum[0], bsum[1], bsum[2], n, e_max, c_sigma);
}

__global__ void fill_kernel(double* x, int64_t n, double v) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

__global__ void max_abs_from_rows_kernel(int64_t m, const double* mx, const double* mn, double* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) atomic_max_nonneg(out, fmax(fabs(mx[i]), fabs(mn[i])));
}

}  // namespace

extern "C" vabft_status vabft_encode_workspace_size(int64_t m, int64_t n, int64_t k,
                                                    const vabft_precision* spec, size_t* bytes) {
    return guarded([&] {
        (void)m; (void)n; (void)k; (void)spec;
        if (!bytes) fail(VABFT_INVALID_ARGUMENT, "null bytes");
        *bytes = 0;  // temporaries come from the stream-ordered allocator
    });
}

extern "C" vabft_status vabft_encode_and_multiply(const vabft_precision* spec, int32_t mode,
                                                  int32_t engine, int64_t m, int64_t n, int64_t k,
                                                  const void* A, const void* B, void* C,
                                                  void* C_accum, double* rc1, double* rc2,
                                                  double* cc1, double* cc2, void* workspace,
                                                  size_t ws_bytes, void* stream) {
    return guarded([&] {
        (void)workspace; (void)ws_bytes;
        if (!spec || !A || !B) fail(VABFT_INVALID_ARGUMENT, "encode_and_multiply: null argument");
        check_fmt(spec->format);
        if (m < 1 || n < 1 || k < 1) fail(VABFT_INVALID_ARGUMENT, "Matrix: dims must be >= 1");
        if (mode != VABFT_OFFLINE && mode != VABFT_ONLINE) fail(VABFT_INVALID_ARGUMENT, "bad mode");
        const int f = spec->format;
        if ((f == VABFT_BF16 || f == VABFT_FP16) && spec->accumulation.kind != VABFT_ACCUM_FP32_ROUND_OUTPUT)
            fail(VABFT_INVALID_ARGUMENT, "gemm_emulated: 16-bit formats require fp32 accumulation");
        int csf;
        vabft_accum csa;
        cs_prec(*spec, mode, &csf, &csa);
        if (engine == VABFT_ENGINE_TENSOR) {
            // TENSOR engine checksum precision: FP32 arithmetic in blocked:128
            // order for both modes (an FP32 PrecisionSpec with NativeBlocked(128));
            // FP64 keeps FP64 arithmetic in the same order
            csf = f == VABFT_FP64 ? VABFT_FP64 : VABFT_FP32;
            csa = vabft_accum{VABFT_ACCUM_BLOCKED, 0, 128};
        }
        check_weights(n, csf, csa.kind);
        check_weights(m, csf, csa.kind);
        cudaStream_t s = as_stream(stream);
        Tmp tmp(s);
        const bool flt = accumulates_in_float(csf, csa.kind);
        const int qfmt = mode == VABFT_OFFLINE ? f : -1;

        if (engine == VABFT_ENGINE_TENSOR && (f == VABFT_FP64 || f == VABFT_FP32)) {
            // FP64: SIMT DFMA GEMM; FP32: tcgen05 3xTF32. C and C_accum hold
            // the same values (the accumulator is in the output format).
            const size_t es = f == VABFT_FP64 ? 8 : 4;
            void* c = C ? C : C_accum;
            if (c) {
                if (f == VABFT_FP64)
                    dgemm_launch(m, n, k, static_cast<const double*>(A), static_cast<const double*>(B),
                                 static_cast<double*>(c), WideEpilogue{}, s);
                else
                    tf32_gemm_run(m, n, k, static_cast<const float*>(A), static_cast<const float*>(B),
                                  static_cast<float*>(c), WideEpilogue{}, 3, s);
                if (C && C_accum)
                    check_cuda(cudaMemcpyAsync(C_accum, C, es * size_t(m * n), cudaMemcpyDeviceToDevice, s), "copy");
            }
            if (rc1 || rc2) {
                const bool fl = f == VABFT_FP32;
                double* br1 = tmp.get<double>(k);
                double* br2 = tmp.get<double>(k);
                launch_row_reduce(f, fl, 0, csa, k, n, B, nullptr, nullptr, qfmt, br1, br2, s);
                double* o1 = rc1 ? rc1 : tmp.get<double>(m);
                double* o2 = rc2 ? rc2 : tmp.get<double>(m);
                launch_row_reduce(f, fl, 1, csa, m, k, A, br1, br2, qfmt, o1, o2, s);
            }
        } else if (engine == VABFT_ENGINE_TENSOR) {
            if (f != VABFT_BF16 && f != VABFT_FP16)
                fail(VABFT_UNSUPPORTED, "TENSOR engine: unsupported format");
            void* c = C ? C : tmp.get<uint16_t>(size_t(m * n));
            TcEpilogue epi;
            epi.accum_out = static_cast<float*>(C_accum);
            tc_gemm_launch(f, false, m, n, k, A, B, c, epi, s);
            if (rc1 || rc2) {
                BsideBuffers buf = tmp_bside(tmp, f, k, n, s);
                launch_bside(f, k, n, B, mode == VABFT_OFFLINE, buf, s);
                double* T = tmp.get<double>(m);
                double* mx = tmp.get<double>(1);
                check_cuda(cudaMemsetAsync(mx, 0, sizeof(double), s), "memset");
                double* o1 = rc1 ? rc1 : tmp.get<double>(m);
                double* o2 = rc2 ? rc2 : tmp.get<double>(m);
                launch_aside(f, m, k, n, A, buf, mode == VABFT_OFFLINE, 0.0, 2.5, T, o1, o2, mx, s);
            }
        } else {
            if (C || C_accum) launch_exact_gemm(f, spec->accumulation, m, n, k, A, B, C, C_accum, s);
            if (rc1 || rc2) {
                double* br1 = tmp.get<double>(k);
                double* br2 = tmp.get<double>(k);
                launch_row_reduce(f, flt, 0, csa, k, n, B, nullptr, nullptr, qfmt, br1, br2, s);
                double* o1 = rc1 ? rc1 : tmp.get<double>(m);
                double* o2 = rc2 ? rc2 : tmp.get<double>(m);
                launch_row_reduce(f, flt, 1, csa, m, k, A, br1, br2, qfmt, o1, o2, s);
            }
        }
        if (cc1 || cc2) {
            double* ac1 = tmp.get<double>(k);
            double* ac2 = tmp.get<double>(k);
            launch_col_reduce(f, flt, 0, csa, m, k, A, nullptr, nullptr, qfmt, ac1, ac2, s);
            double* o1 = cc1 ? cc1 : tmp.get<double>(n);
            double* o2 = cc2 ? cc2 : tmp.get<double>(n);
            launch_col_reduce(f, flt, 1, csa, k, n, B, ac1, ac2, qfmt, o1, o2, s);
        }
    });
}

extern "C" vabft_status vabft_row_sums(const vabft_precision* sp, int32_t src_format, int64_t m,
                                       int64_t n, const void* source, double* r1, double* r2,
                                       void* stream) {
    return guarded([&] {
        if (!sp || !source || !r1 || !r2) fail(VABFT_INVALID_ARGUMENT, "row_sums: null argument");
        check_fmt(sp->format);
        check_fmt(src_format);
        if (m < 1 || n < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        check_weights(n, sp->format, sp->accumulation.kind);
        launch_row_reduce(src_format, accumulates_in_float(sp->format, sp->accumulation.kind), 0,
                          sp->accumulation, m, n, source, nullptr, nullptr, -1, r1, r2, as_stream(stream));
    });
}

extern "C" vabft_status vabft_row_stats(int32_t format, int64_t rows, int64_t cols, const void* X,
                                        double* mean, double* mx, double* mn, double* vb,
                                        void* stream) {
    return guarded([&] {
        check_fmt(format);
        if (!X) fail(VABFT_INVALID_ARGUMENT, "row_stats: null matrix");
        if (cols < 1) fail(VABFT_INVALID_ARGUMENT, "row_stats: empty row");
        if (rows < 1) return;
        cudaStream_t s = as_stream(stream);
        Tmp tmp(s);
        int* bad = tmp.get<int>(1);
        check_cuda(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
        launch_row_stats(format, rows, cols, X, mean, mx, mn, vb, bad, s);
        int h = 0;
        check_cuda(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "copy");
        check_cuda(cudaStreamSynchronize(s), "sync");
        if (h) fail(VABFT_DOMAIN_ERROR, "row_stats: non-finite value");
    });
}

extern "C" vabft_status vabft_vabft_thresholds(int32_t format, int64_t m, int64_t n, int64_t k,
                                               const void* A, const void* B, double e_max,
                                               double c_sigma, double* T, double* b_summary_out,
                                               void* stream) {
    return guarded([&] {
        check_fmt(format);
        if (!A || !B || !T) fail(VABFT_INVALID_ARGUMENT, "vabft_thresholds: null argument");
        if (m < 1 || n < 1 || k < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        cudaStream_t s = as_stream(stream);
        Tmp tmp(s);
        BsideBuffers buf = tmp_bside(tmp, format, k, n, s);
        launch_bside(format, k, n, B, 0, buf, s);
        double* mean = tmp.get<double>(m);
        double* vb = tmp.get<double>(m);
        launch_row_stats(format, m, k, A, mean, nullptr, nullptr, vb, buf.nonfinite, s);
        thresholds_from_stats_kernel<<<unsigned((m + 255) / 256), 256, 0, s>>>(m, n, mean, vb, buf.summary,
                                                                             e_max, c_sigma, T);
        check_cuda(cudaGetLastError(), "thresholds launch");
        if (b_summary_out)
            check_cuda(cudaMemcpyAsync(b_summary_out, buf.summary, 3 * sizeof(double),
                                       cudaMemcpyDeviceToDevice, s), "copy");
        int h = 0;
        check_cuda(cudaMemcpyAsync(&h, buf.nonfinite, sizeof(int), cudaMemcpyDeviceToHost, s), "copy");
        check_cuda(cudaStreamSynchronize(s), "sync");
        if (h) fail(VABFT_DOMAIN_ERROR, "row_stats: non-finite value");
    });
}

extern "C" vabft_status vabft_blockwise_thresholds(int32_t format, int64_t m, int64_t n, int64_t k,
                                                   const void* A, int64_t lda, const void* B, int64_t ldb,
                                                   int64_t tile_k, int64_t tile_n, const double* e_max_per_tile,
                                                   double c_sigma, double* T, void* stream) {
    return guarded([&] {
        check_fmt(format);
        if (!A || !B || !T || !e_max_per_tile) fail(VABFT_INVALID_ARGUMENT, "blockwise_thresholds: null argument");
        if (m < 1 || n < 1 || k < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        if (tile_k < 1 || tile_n < 1) fail(VABFT_INVALID_ARGUMENT, "blockwise_thresholds: tiles must be >= 1");
        if (lda == 0) lda = k;
        if (ldb == 0) ldb = n;
        if (lda < k || ldb < n) fail(VABFT_INVALID_ARGUMENT, "blockwise_thresholds: leading dimension too small");
        const int64_t nkt = (k + tile_k - 1) / tile_k;
        for (int64_t t = 0; t < nkt; ++t)  // threshold_row's e_max: the caller's model at dim = |kt|
            if (!(e_max_per_tile[t] >= 0.0)) fail(VABFT_INVALID_ARGUMENT, "blockwise_thresholds: e_max must be >= 0");
        cudaStream_t s = as_stream(stream);
        Tmp tmp(s);
        double* em = tmp.get<double>(size_t(nkt));
        check_cuda(cudaMemcpyAsync(em, e_max_per_tile, sizeof(double) * size_t(nkt), cudaMemcpyHostToDevice, s),
                   "copy");
        double* work = tmp.get<double>(blockwise_work_doubles(m, n, k, tile_k, tile_n));
        int* bad = tmp.get<int>(1);
        check_cuda(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
        launch_blockwise_thresholds(format, m, n, k, A, lda, B, ldb, tile_k, tile_n, em, c_sigma, T, work, bad, s);
        int h = 0;
        check_cuda(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "copy");
        check_cuda(cudaStreamSynchronize(s), "sync");
        if (h) fail(VABFT_DOMAIN_ERROR, "row_stats: non-finite value");
    });
}

extern "C" vabft_status vabft_aabft_threshold(int32_t format, int64_t m, int64_t n, int64_t k,
                                              const void* A, const void* B, int32_t t, double fixed_y,
                                              double conf, double* T, double* y_used,
                                              int32_t* degenerate, void* stream) {
    return guarded([&] {
        check_fmt(format);
        if (!A || !B || !T) fail(VABFT_INVALID_ARGUMENT, "aabft_threshold: null argument");
        if (m < 1 || n < 1 || k < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        cudaStream_t s = as_stream(stream);
        double y = fixed_y;
        if (std::isnan(fixed_y)) {
            // computed y = max|A| * max_k |sum_j B[k][j]| (threshold_aabft.cpp:38-48)
            Tmp tmp(s);
            BsideBuffers buf = tmp_bside(tmp, format, k, n, s);
            launch_bside(format, k, n, B, 0, buf, s);
            if (format == VABFT_FP32 || format == VABFT_FP64)  // plain row sums on demand (bside.cu)
                launch_bside_rowsum(format, k, n, B, buf, s);
            double* mx = tmp.get<double>(m);
            double* mn = tmp.get<double>(m);
            launch_row_stats(format, m, k, A, nullptr, mx, mn, nullptr, buf.nonfinite, s);
            double* amax = tmp.get<double>(1);
            check_cuda(cudaMemsetAsync(amax, 0, sizeof(double), s), "memset");
            max_abs_from_rows_kernel<<<unsigned((m + 255) / 256), 256, 0, s>>>(m, mx, mn, amax);
            double h[2];
            check_cuda(cudaMemcpyAsync(&h[0], amax, sizeof(double), cudaMemcpyDeviceToHost, s), "copy");
            check_cuda(cudaMemcpyAsync(&h[1], buf.summary + 3, sizeof(double), cudaMemcpyDeviceToHost, s), "copy");
            check_cuda(cudaStreamSynchronize(s), "sync");
            y = h[0] * h[1];
        }
        const double nn = double(k);
        const double poly = nn * (nn + 1.0) * (nn + 0.5) + 2.0 * nn;
        const double sig = std::sqrt(poly / 24.0) * std::ldexp(1.0, -t) * y;
        const double thr = conf * sig;  // the caller's multiplier as given (threshold_aabft.cpp:56)
        fill_kernel<<<unsigned((m + 255) / 256), 256, 0, s>>>(T, m, thr);
        check_cuda(cudaGetLastError(), "fill launch");
        if (y_used) *y_used = y;
        if (degenerate) *degenerate = y == 0.0;
    });
}

extern "C" vabft_status vabft_verify(const vabft_precision* cs, int32_t src_format, int64_t m,
                                     int64_t n, const void* source, const double* rc1,
                                     const double* rc2, const double* T, double floor_scale,
                                     vabft_verdicts v, int64_t* counts, void* stream) {
    return guarded([&] {
        if (!cs || !source || !rc1 || !rc2 || !T) fail(VABFT_INVALID_ARGUMENT, "verify: null argument");
        check_fmt(cs->format);
        check_fmt(src_format);
        if (m < 1 || n < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
        cudaStream_t s = as_stream(stream);
        // thresholds must be >= 0 (detect.cpp:24-27)
        std::vector<double> th(static_cast<size_t>(m));
        check_cuda(cudaMemcpyAsync(th.data(), T, sizeof(double) * size_t(m), cudaMemcpyDeviceToHost, s), "copy");
        check_cuda(cudaStreamSynchronize(s), "sync");
        for (double t : th)
            if (!(t >= 0.0)) fail(VABFT_INVALID_ARGUMENT, "verify: thresholds must be >= 0");
        check_weights(n, cs->format, cs->accumulation.kind);
        Tmp tmp(s);
        double* r1 = tmp.get<double>(m);
        double* r2 = tmp.get<double>(m);
        launch_row_reduce(src_format, accumulates_in_float(cs->format, cs->accumulation.kind), 0,
                          cs->accumulation, m, n, source, nullptr, nullptr, -1, r1, r2, s);
        launch_verify(m, n, r1, r2, rc1, rc2, T, floor_scale, v, counts, s);
    });
}

extern "C" vabft_status vabft_inject(int32_t format, int64_t m, int64_t n, void* X,
                                     const vabft_fault* faults, int64_t n_faults,
                                     vabft_fault_record* records, void* stream) {
    return guarded([&] {
        check_fmt(format);
        if (!X || (n_faults > 0 && !faults)) fail(VABFT_INVALID_ARGUMENT, "inject: null argument");
        const int width = format <= VABFT_FP16 ? 16 : format == VABFT_FP32 ? 32 : 64;
        for (int64_t q = 0; q < n_faults; ++q) {
            const vabft_fault& f = faults[q];
            if (f.bit < 0 || f.bit >= width)
                fail(VABFT_OUT_OF_RANGE, "inject: bit index outside the format's width");
            if (f.i < 0 || f.i >= m || f.j < 0 || f.j >= n)
                fail(VABFT_OUT_OF_RANGE, "inject: position out of range");
            if (f.direction < VABFT_FLIP || f.direction > VABFT_FLIP_SET1TO0)
                fail(VABFT_INVALID_ARGUMENT, "inject: direction ANY must be resolved by the caller");
        }
        if (n_faults == 0) return;
        cudaStream_t s = as_stream(stream);
        Tmp tmp(s);
        vabft_fault* df = tmp.get<vabft_fault>(size_t(n_faults));
        vabft_fault_record* dr = tmp.get<vabft_fault_record>(size_t(n_faults));
        check_cuda(cudaMemcpyAsync(df, faults, sizeof(vabft_fault) * size_t(n_faults), cudaMemcpyHostToDevice, s), "copy");
        launch_inject(format, n, X, df, n_faults, dr, s);
        if (records) {
            check_cuda(cudaMemcpyAsync(records, dr, sizeof(vabft_fault_record) * size_t(n_faults),
                                       cudaMemcpyDeviceToHost, s), "copy");
            check_cuda(cudaStreamSynchronize(s), "sync");
        }
    });
}
