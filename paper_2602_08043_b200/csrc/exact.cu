// K4 — order-exact ("EXACT" engine) kernels that reproduce the reference's
// emulated arithmetic bit for bit on the device:
//   gemm_emulated_with_accum / run_gemm / gemm_row_block / pairwise_block
//                                       proj/src/precision.cpp:208-338
//   ChecksumEngine plain / position_weighted / contract, encode_impl
//                                       proj/src/checksum.cpp:50-146
//   row_sums                            proj/src/checksum.cpp:160-187
// plus the shared verify (detect.cpp:19-55) and inject (faults.cpp:104-168)
// kernels used by both engines.
#include <map>
#include <mutex>
#include <vector>

#include "devcommon.cuh"
#include "exact.hpp"
#include "internal.hpp"
#include "numerics.cuh"
#include "reducers.cuh"

namespace vabft_dev {

// ------------------------------------------------------ pairwise schedules
// Merge counts of the balanced tree over [0, n) split at k0 + (k1-k0)/2
// (precision.cpp:222-236, 347-352): sched[k] = number of internal nodes
// whose right-most leaf is k.
static void build_sched(int64_t k0, int64_t k1, std::vector<uint8_t>& s) {
    if (k1 - k0 <= 1) return;
    const int64_t mid = k0 + (k1 - k0) / 2;
    build_sched(k0, mid, s);
    build_sched(mid, k1, s);
    s[size_t(k1 - 1)]++;
}

const uint8_t* pairwise_schedule(int64_t n) {
    static std::mutex mu;
    static std::map<std::pair<int, int64_t>, uint8_t*> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, n});
    if (it != cache.end()) return it->second;
    std::vector<uint8_t> s(size_t(n), 0);
    build_sched(0, n, s);
    uint8_t* d = nullptr;
    check_cuda(cudaMalloc(&d, size_t(n)), "cudaMalloc(schedule)");
    check_cuda(cudaMemcpy(d, s.data(), size_t(n), cudaMemcpyHostToDevice), "schedule upload");
    cache[{dev, n}] = d;
    return d;
}

namespace {

template <int F>
using ET = typename Elem<F>::T;

template <class T>
__device__ __forceinline__ T to_work(float x);
template <>
__device__ __forceinline__ float to_work<float>(float x) { return x; }
template <>
__device__ __forceinline__ double to_work<double>(float x) { return double(x); }

template <int F, class T>
__device__ __forceinline__ T load_work(const ET<F>* p) {
    if constexpr (F == VABFT_FP64) {
        return T(*p);
    } else {
        return to_work<T>(Elem<F>::f(*p));
    }
}

// Store one GEMM output with run_gemm's rules (precision.cpp:299-312):
// non-finite accumulator -> both outputs +-max_finite(format); otherwise the
// accumulator verbatim and C quantized when the formats differ.
template <int F, class T>
__device__ __forceinline__ void store_out(T acc, ET<F>* C, T* Caccum, int64_t idx) {
    if constexpr (F == VABFT_BF16 || F == VABFT_FP16) {
        const float a = saturate_accum<F>(acc);
        if (Caccum) Caccum[idx] = a;
        if (C) C[idx] = quantize16_bits<F>(a);
    } else if constexpr (F == VABFT_FP32) {
        const float a = isfinite(acc) ? acc : copysignf(3.40282346638528859812e+38f, acc);
        if (Caccum) Caccum[idx] = a;
        if (C) C[idx] = a;
    } else {
        const double a = isfinite(acc) ? acc : copysign(1.7976931348623157e308, acc);
        if (Caccum) Caccum[idx] = a;
        if (C) C[idx] = a;
    }
}

// ------------------------------------------------ exact GEMM, seq/blocked
// 16x16 threads, 4x4 outputs per thread (64x64 tile), BK = 16. Each output
// consumes k in increasing order: acc = acc + a*b with the product and the
// sum each rounded in T (no FMA). Blocked adds the per-block partials.
constexpr int kTile = 64, kBK = 16;

template <int F, class T, bool kBlocked>
__global__ void __launch_bounds__(256) exact_gemm_seq_kernel(const ET<F>* __restrict__ A,
                                                              const ET<F>* __restrict__ B, int64_t M,
                                                              int64_t N, int64_t K, int64_t bl,
                                                              ET<F>* C, T* Caccum) {
    __shared__ T As[kBK][kTile + 1];
    __shared__ T Bs[kBK][kTile + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t row0 = int64_t(blockIdx.y) * kTile, col0 = int64_t(blockIdx.x) * kTile;
    T acc[4][4], part[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = part[r][c] = T(0);
    for (int64_t k0 = 0; k0 < K; k0 += kBK) {
        for (int e = threadIdx.x; e < kBK * kTile; e += 256) {
            const int kk = e % kBK, rr = e / kBK;  // A tile: rows x k
            const int64_t gr = row0 + rr, gk = k0 + kk;
            As[kk][rr] = (gr < M && gk < K) ? load_work<F, T>(A + gr * K + gk) : T(0);
            const int cc = e % kTile, kb = e / kTile;  // B tile: k x cols
            const int64_t gk2 = k0 + kb, gc = col0 + cc;
            Bs[kb][cc] = (gk2 < K && gc < N) ? load_work<F, T>(B + gk2 * N + gc) : T(0);
        }
        __syncthreads();
        const int kmax = int((K - k0) < kBK ? (K - k0) : kBK);
        for (int kk = 0; kk < kmax; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = As[kk][ty + 16 * r];
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx + 16 * c];
            const int64_t kg = k0 + kk;
            if constexpr (kBlocked) {
                const bool flush = ((kg + 1) % bl == 0) || (kg + 1 == K);
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        part[r][c] = radd(part[r][c], rmul(a[r], b[c]));
                        if (flush) {
                            acc[r][c] = radd(acc[r][c], part[r][c]);
                            part[r][c] = T(0);
                        }
                    }
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = radd(acc[r][c], rmul(a[r], b[c]));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t gr = row0 + ty + 16 * r, gc = col0 + tx + 16 * c;
            if (gr < M && gc < N) store_out<F, T>(acc[r][c], C, Caccum, gr * N + gc);
        }
}

// --------------------------------------------------- exact GEMM, pairwise
// One output per thread (16x16 tile); the tree is evaluated with a stack in
// local memory following the merge schedule of length K.
template <int F, class T>
__global__ void __launch_bounds__(256) exact_gemm_pairwise_kernel(const ET<F>* __restrict__ A,
                                                                   const ET<F>* __restrict__ B,
                                                                   int64_t M, int64_t N, int64_t K,
                                                                   const uint8_t* __restrict__ sched,
                                                                   ET<F>* C, T* Caccum) {
    __shared__ T As[16][kBK + 1];
    __shared__ T Bs[kBK][16 + 1];
    __shared__ uint8_t Ss[kBK];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t gr = int64_t(blockIdx.y) * 16 + ty, gc = int64_t(blockIdx.x) * 16 + tx;
    T st[Reducer<T>::kMaxDepth];
    int sp = 0;
    for (int64_t k0 = 0; k0 < K; k0 += kBK) {
        {
            const int64_t ar = int64_t(blockIdx.y) * 16 + ty, ak = k0 + tx;
            As[ty][tx] = (ar < M && ak < K) ? load_work<F, T>(A + ar * K + ak) : T(0);
            const int64_t bk = k0 + ty, bc = int64_t(blockIdx.x) * 16 + tx;
            Bs[ty][tx] = (bk < K && bc < N) ? load_work<F, T>(B + bk * N + bc) : T(0);
            if (threadIdx.x < kBK && k0 + threadIdx.x < K) Ss[threadIdx.x] = sched[k0 + threadIdx.x];
        }
        __syncthreads();
        const int kmax = int((K - k0) < kBK ? (K - k0) : kBK);
        for (int kk = 0; kk < kmax; ++kk) {
            T v = rmul(As[ty][kk], Bs[kk][tx]);
            int c = Ss[kk];
            while (c-- > 0) v = radd(st[--sp], v);
            st[sp++] = v;
        }
        __syncthreads();
    }
    if (gr < M && gc < N) store_out<F, T>(st[0], C, Caccum, gr * N + gc);
}

// Offline checksum quantization (checksum.cpp:112-115, 129-134). qfmt < 0:
// none. Non-finite values are kept so the host can raise quantize's
// domain_error; FP32/FP64 quantization of a finite value is the identity.
__device__ __forceinline__ double quantize_checksum(double x, int qfmt) {
    if (qfmt < 0 || !isfinite(x)) return x;
    if (qfmt == VABFT_BF16) return double(bits16_to_float<VABFT_BF16>(quantize16_bits<VABFT_BF16>(float(x))));
    if (qfmt == VABFT_FP16) return double(bits16_to_float<VABFT_FP16>(quantize16_bits<VABFT_FP16>(float(x))));
    return x;
}

// ----------------------------------------------------- row-wise reductions
// One warp handles 32 rows; 32x32 tiles are staged through shared memory
// (coalesced loads), then each lane walks its own row in order.
//   kTerm 0: out1 = reduce(T(x_j)), out2 = reduce(T(j+1) * T(x_j))
//   kTerm 1: out1 = reduce(w1_j * T(x_j)), out2 = reduce(w2_j * T(x_j))
// Optional quantization of the results to `qfmt` (offline checksums).
template <int F, class T, int kTerm>
__global__ void exact_row_reduce_kernel(const ET<F>* __restrict__ X, int64_t rows, int64_t cols,
                                        int kind, int64_t bl, const uint8_t* sched,
                                        const double* __restrict__ w1, const double* __restrict__ w2,
                                        int qfmt, double* out1, double* out2) {
    __shared__ T tile[4][32][33];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t(blockIdx.x) * 4 + w) * 32;
    if (r0 >= rows) return;
    const int64_t my_row = r0 + lane;
    Reducer<T> red1(kind, bl, sched), red2(kind, bl, sched);
    for (int64_t c0 = 0; c0 < cols; c0 += 32) {
        for (int rr = 0; rr < 32; ++rr) {
            const int64_t r = r0 + rr, c = c0 + lane;
            tile[w][rr][lane] = (r < rows && c < cols) ? load_work<F, T>(X + r * cols + c) : T(0);
        }
        __syncwarp();
        const int cmax = int((cols - c0) < 32 ? (cols - c0) : 32);
        if (my_row < rows) {
            for (int jj = 0; jj < cmax; ++jj) {
                const int64_t j = c0 + jj;
                const T x = tile[w][lane][jj];
                if constexpr (kTerm == 0) {
                    red1.push(x, cols);
                    red2.push(rmul(T(j + 1), x), cols);
                } else {
                    red1.push(rmul(T(w1[j]), x), cols);
                    red2.push(rmul(T(w2[j]), x), cols);
                }
            }
        }
        __syncwarp();
    }
    if (my_row < rows) {
        double a = double(red1.result()), b = double(red2.result());
        out1[my_row] = quantize_checksum(a, qfmt);
        out2[my_row] = quantize_checksum(b, qfmt);
    }
}

// Warp per row for term 0 in NativeBlocked(128) order with the storage type
// as working type (FP32 / FP64 B r1 / B r2 of the fused path's weights):
// lane l sums blocks l, l + 32, ... in order (radd / rmul exactly as
// Reducer's BLOCKED path), then the block partials are added in block order.
// exact_row_reduce_kernel's thread-per-row walk took 1.9 ms for a 4096 x 4096
// FP32 weight (32 CTAs); this is one read of the matrix.
template <class T>
__global__ void __launch_bounds__(256) blocked128_row_reduce_kernel(const T* __restrict__ X, int64_t rows,
                                                                   int64_t cols, int qfmt, double* out1,
                                                                   double* out2) {
    const int lane = threadIdx.x & 31;
    const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (r >= rows) return;
    const T* row = X + r * cols;
    const int64_t nblk = (cols + 127) / 128;
    T acc1 = T(0), acc2 = T(0);
    for (int64_t b0 = 0; b0 < nblk; b0 += 32) {
        T p1 = T(0), p2 = T(0);
        const int64_t b = b0 + lane;
        if (b < nblk) {
            const int64_t j0 = b * 128, j1 = cols < j0 + 128 ? cols : j0 + 128;
#pragma unroll 8
            for (int64_t j = j0; j < j1; ++j) {
                const T x = __ldg(row + j);
                p1 = radd(p1, x);
                p2 = radd(p2, rmul(T(j + 1), x));
            }
        }
        const int cnt = int(nblk - b0 < 32 ? nblk - b0 : 32);
        for (int l = 0; l < cnt; ++l) {
            acc1 = radd(acc1, __shfl_sync(0xffffffffu, p1, l));
            acc2 = radd(acc2, __shfl_sync(0xffffffffu, p2, l));
        }
    }
    if (lane == 0) {
        out1[r] = quantize_checksum(double(acc1), qfmt);
        out2[r] = quantize_checksum(double(acc2), qfmt);
    }
}

// ---------------------------------------------------- column reductions
// One thread per column j of an R x L matrix (coalesced across threads),
// reducing over rows in order:
//   kTerm 0: out1 = reduce_i T(x_ij), out2 = reduce_i T(i+1) T(x_ij)
//   kTerm 1: out1 = reduce_i w1_i T(x_ij), out2 = reduce_i w2_i T(x_ij)
template <int F, class T, int kTerm>
__global__ void exact_col_reduce_kernel(const ET<F>* __restrict__ X, int64_t rows, int64_t cols,
                                        int kind, int64_t bl, const uint8_t* sched,
                                        const double* __restrict__ w1, const double* __restrict__ w2,
                                        int qfmt, double* out1, double* out2) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    Reducer<T> red1(kind, bl, sched), red2(kind, bl, sched);
    for (int64_t i = 0; i < rows; ++i) {
        const T x = load_work<F, T>(X + i * cols + j);
        if constexpr (kTerm == 0) {
            red1.push(x, rows);
            red2.push(rmul(T(i + 1), x), rows);
        } else {
            red1.push(rmul(T(w1[i]), x), rows);
            red2.push(rmul(T(w2[i]), x), rows);
        }
    }
    out1[j] = quantize_checksum(double(red1.result()), qfmt);
    out2[j] = quantize_checksum(double(red2.result()), qfmt);
}

// -------------------------------------------------------------- verify
// detect.cpp:19-55 on precomputed row sums r1/r2 (double holding the
// working-type value). Counters are accumulated with warp-aggregated atomics.
__global__ void verify_kernel(int64_t m, int64_t n, const double* __restrict__ r1,
                              const double* __restrict__ r2, const double* __restrict__ rc1,
                              const double* __restrict__ rc2, const double* __restrict__ T,
                              double floor_scale, vabft_verdicts v, int64_t* counts) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool det = false, located = false, isnan_row = false, valid = i < m;
    if (valid) {
        const double d1 = __dsub_rn(r1[i], rc1[i]);
        const double d2 = __dsub_rn(r2[i], rc2[i]);
        const double t = T[i];
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
                if (localize_dev(d1, d2, n, &j, &rr)) {
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

// --------------------------------------------------------------- inject
// Fixed-position faults applied in order by one thread (faults.cpp:104-168,
// positions given). Canonical encodings: BF16/FP16 raw 16-bit patterns,
// FP32/FP64 IEEE patterns.
__global__ void inject_kernel(int fmt, int64_t n, void* X, const vabft_fault* faults, int64_t nf,
                              vabft_fault_record* rec) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int64_t f = 0; f < nf; ++f) {
        const vabft_fault ft = faults[f];
        const int64_t idx = ft.i * n + ft.j;
        uint64_t bits;
        double before, after;
        if (fmt == VABFT_BF16 || fmt == VABFT_FP16) {
            uint16_t* p = static_cast<uint16_t*>(X) + idx;
            bits = *p;
            before = fmt == VABFT_BF16 ? double(bits16_to_float<VABFT_BF16>(uint16_t(bits)))
                                       : double(bits16_to_float<VABFT_FP16>(uint16_t(bits)));
        } else if (fmt == VABFT_FP32) {
            float* p = static_cast<float*>(X) + idx;
            bits = __float_as_uint(*p);
            before = double(*p);
        } else {
            double* p = static_cast<double*>(X) + idx;
            bits = uint64_t(__double_as_longlong(*p));
            before = *p;
        }
        const bool ok = bit_eligible(bits, ft.bit, ft.direction);
        const uint64_t nb = ok ? (bits ^ (uint64_t(1) << ft.bit)) : bits;
        if (fmt == VABFT_BF16 || fmt == VABFT_FP16) {
            static_cast<uint16_t*>(X)[idx] = uint16_t(nb);
            after = fmt == VABFT_BF16 ? double(bits16_to_float<VABFT_BF16>(uint16_t(nb)))
                                      : double(bits16_to_float<VABFT_FP16>(uint16_t(nb)));
        } else if (fmt == VABFT_FP32) {
            static_cast<float*>(X)[idx] = __uint_as_float(uint32_t(nb));
            after = double(__uint_as_float(uint32_t(nb)));
        } else {
            static_cast<double*>(X)[idx] = __longlong_as_double(int64_t(nb));
            after = __longlong_as_double(int64_t(nb));
        }
        if (rec) {  // records are optional for campaign callers
            rec[f].value_before = before;
            rec[f].value_after = after;
            rec[f].applied = ok ? 1 : 0;
            rec[f].reserved = 0;
        }
    }
}

}  // namespace

// ================================================================ launchers
bool accumulates_in_float(int fmt, int kind) {
    return kind == VABFT_ACCUM_FP32_ROUND_OUTPUT || fmt == VABFT_FP32;
}

template <int F, class T>
static void gemm_exact_t(const vabft_accum& acc, int64_t M, int64_t N, int64_t K, const void* A,
                         const void* B, void* C, void* Caccum, cudaStream_t s) {
    const ET<F>* a = static_cast<const ET<F>*>(A);
    const ET<F>* b = static_cast<const ET<F>*>(B);
    ET<F>* c = static_cast<ET<F>*>(C);
    T* ca = static_cast<T*>(Caccum);
    if (acc.kind == VABFT_ACCUM_PAIRWISE) {
        const dim3 grid(unsigned((N + 15) / 16), unsigned((M + 15) / 16));
        exact_gemm_pairwise_kernel<F, T><<<grid, 256, 0, s>>>(a, b, M, N, K, pairwise_schedule(K), c, ca);
    } else {
        const dim3 grid(unsigned((N + kTile - 1) / kTile), unsigned((M + kTile - 1) / kTile));
        if (acc.kind == VABFT_ACCUM_BLOCKED)
            exact_gemm_seq_kernel<F, T, true><<<grid, 256, 0, s>>>(a, b, M, N, K, acc.block_len > 0 ? acc.block_len : 128, c, ca);
        else
            exact_gemm_seq_kernel<F, T, false><<<grid, 256, 0, s>>>(a, b, M, N, K, 1, c, ca);
    }
    check_cuda(cudaGetLastError(), "exact gemm launch");
}

void launch_exact_gemm(int fmt, const vabft_accum& acc, int64_t M, int64_t N, int64_t K,
                       const void* A, const void* B, void* C, void* Caccum, cudaStream_t s) {
    if ((fmt == VABFT_BF16 || fmt == VABFT_FP16) && acc.kind != VABFT_ACCUM_FP32_ROUND_OUTPUT)
        fail(VABFT_INVALID_ARGUMENT, "gemm_emulated: 16-bit formats require fp32 accumulation");
    const bool flt = accumulates_in_float(fmt, acc.kind);
    switch (fmt) {
        case VABFT_BF16: gemm_exact_t<VABFT_BF16, float>(acc, M, N, K, A, B, C, Caccum, s); break;
        case VABFT_FP16: gemm_exact_t<VABFT_FP16, float>(acc, M, N, K, A, B, C, Caccum, s); break;
        case VABFT_FP32: gemm_exact_t<VABFT_FP32, float>(acc, M, N, K, A, B, C, Caccum, s); break;
        case VABFT_FP64:
            if (flt) fail(VABFT_UNSUPPORTED, "FP64 with FP32 accumulation");
            gemm_exact_t<VABFT_FP64, double>(acc, M, N, K, A, B, C, Caccum, s);
            break;
        default: fail(VABFT_INVALID_ARGUMENT, "bad format");
    }
}

template <int F, class T>
static void row_reduce_t(int term, const vabft_accum& acc, int64_t rows, int64_t cols, const void* X,
                         const double* w1, const double* w2, int qfmt, double* o1, double* o2,
                         cudaStream_t s) {
    const uint8_t* sched = acc.kind == VABFT_ACCUM_PAIRWISE ? pairwise_schedule(cols) : nullptr;
    const unsigned grid = unsigned((rows + 127) / 128);
    const ET<F>* x = static_cast<const ET<F>*>(X);
    if (term == 0)
        exact_row_reduce_kernel<F, T, 0><<<grid, 128, 0, s>>>(x, rows, cols, acc.kind, acc.block_len, sched, w1, w2, qfmt, o1, o2);
    else
        exact_row_reduce_kernel<F, T, 1><<<grid, 128, 0, s>>>(x, rows, cols, acc.kind, acc.block_len, sched, w1, w2, qfmt, o1, o2);
    check_cuda(cudaGetLastError(), "row reduce launch");
}

template <int F, class T>
static void col_reduce_t(int term, const vabft_accum& acc, int64_t rows, int64_t cols, const void* X,
                         const double* w1, const double* w2, int qfmt, double* o1, double* o2,
                         cudaStream_t s) {
    const uint8_t* sched = acc.kind == VABFT_ACCUM_PAIRWISE ? pairwise_schedule(rows) : nullptr;
    const unsigned grid = unsigned((cols + 127) / 128);
    const ET<F>* x = static_cast<const ET<F>*>(X);
    if (term == 0)
        exact_col_reduce_kernel<F, T, 0><<<grid, 128, 0, s>>>(x, rows, cols, acc.kind, acc.block_len, sched, w1, w2, qfmt, o1, o2);
    else
        exact_col_reduce_kernel<F, T, 1><<<grid, 128, 0, s>>>(x, rows, cols, acc.kind, acc.block_len, sched, w1, w2, qfmt, o1, o2);
    check_cuda(cudaGetLastError(), "col reduce launch");
}

#define VABFT_DISPATCH_RED(fn, fmt, flt, ...)                                                   \
    do {                                                                                         \
        switch (fmt) {                                                                           \
            case VABFT_BF16:                                                                     \
                if (flt) fn<VABFT_BF16, float>(__VA_ARGS__); else fn<VABFT_BF16, double>(__VA_ARGS__); \
                break;                                                                           \
            case VABFT_FP16:                                                                     \
                if (flt) fn<VABFT_FP16, float>(__VA_ARGS__); else fn<VABFT_FP16, double>(__VA_ARGS__); \
                break;                                                                           \
            case VABFT_FP32:                                                                     \
                if (flt) fn<VABFT_FP32, float>(__VA_ARGS__); else fn<VABFT_FP32, double>(__VA_ARGS__); \
                break;                                                                           \
            case VABFT_FP64:                                                                     \
                if (flt) fn<VABFT_FP64, float>(__VA_ARGS__); else fn<VABFT_FP64, double>(__VA_ARGS__); \
                break;                                                                           \
            default: fail(VABFT_INVALID_ARGUMENT, "bad format");                                 \
        }                                                                                        \
    } while (0)

void launch_row_reduce(int src_fmt, bool flt, int term, const vabft_accum& acc, int64_t rows,
                       int64_t cols, const void* X, const double* w1, const double* w2, int qfmt,
                       double* o1, double* o2, cudaStream_t s) {
    const bool blocked128 = acc.kind == VABFT_ACCUM_BLOCKED && (acc.block_len <= 0 || acc.block_len == 128);
    if (term == 0 && blocked128 && rows > 0 && cols > 0 &&
        ((src_fmt == VABFT_FP32 && flt) || (src_fmt == VABFT_FP64 && !flt))) {
        const unsigned grid = unsigned((rows + 7) / 8);
        if (src_fmt == VABFT_FP32)
            blocked128_row_reduce_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(X), rows, cols, qfmt, o1, o2);
        else
            blocked128_row_reduce_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(X), rows, cols, qfmt, o1, o2);
        check_cuda(cudaGetLastError(), "blocked row reduce launch");
        return;
    }
    VABFT_DISPATCH_RED(row_reduce_t, src_fmt, flt, term, acc, rows, cols, X, w1, w2, qfmt, o1, o2, s);
}

void launch_col_reduce(int src_fmt, bool flt, int term, const vabft_accum& acc, int64_t rows,
                       int64_t cols, const void* X, const double* w1, const double* w2, int qfmt,
                       double* o1, double* o2, cudaStream_t s) {
    VABFT_DISPATCH_RED(col_reduce_t, src_fmt, flt, term, acc, rows, cols, X, w1, w2, qfmt, o1, o2, s);
}

void launch_verify(int64_t m, int64_t n, const double* r1, const double* r2, const double* rc1,
                   const double* rc2, const double* T, double floor_scale, const vabft_verdicts& v,
                   int64_t* counts, cudaStream_t s) {
    const unsigned grid = unsigned((m + 255) / 256);
    verify_kernel<<<grid, 256, 0, s>>>(m, n, r1, r2, rc1, rc2, T, floor_scale, v, counts);
    check_cuda(cudaGetLastError(), "verify launch");
}

void launch_inject(int fmt, int64_t n, void* X, const vabft_fault* d_faults, int64_t nf,
                   vabft_fault_record* d_rec, cudaStream_t s) {
    inject_kernel<<<1, 32, 0, s>>>(fmt, n, X, d_faults, nf, d_rec);
    check_cuda(cudaGetLastError(), "inject launch");
}

}  // namespace vabft_dev
