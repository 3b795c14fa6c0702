// FP32 GEMM on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with
// FP32 accumulation in TMEM, plus the V-ABFT epilogue of the wide-format
// fused path (FP32 row partials, FP32 accumulator fault injection).
//
// FP32 accuracy (the reference multiplies FP32 operands in FP32,
// precision.cpp:222-236) comes from 3xTF32 error compensation: every operand
// is split once in HBM into hi = rna_tf32(x) and lo = rna_tf32(x - hi) (the
// weight B when its handle is created — stored transposed, N x K, because
// kind::tf32 reads only K-major operands — the activation A per call), and each
// k step issues D += a_lo b_hi, D += a_hi b_lo, D += a_hi b_hi. The dropped
// a_lo b_lo term and the rounding of lo are below 2^-22 |a b|. A single-pass
// TF32 mode (passes = 1) multiplies the raw A by the rounded B.
//
// Structure (one CTA per SM, persistent over 128 x 256 output tiles):
//   warp 0      TMA producer: per 16-deep k block, A_hi / A_lo boxes {16 k,
//               128 rows} and B_hi / B_lo boxes {16 k, 256 n} (all K-major,
//               SWIZZLE_64B); single pass: 32-deep k blocks, SWIZZLE_128B.
//               4-stage ring of 48 KiB stages.
//   warp 1      TMEM allocation (2 x 256 FP32 columns) and the single-thread
//               MMA issuer (M = 128, N = 256, K = 8; 3 MMAs per k step).
//   warps 2..5  epilogue: tcgen05.ld -> saturate -> optional bit flip ->
//               blocked:128 FP32 row partials -> C store.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "internal.hpp"
#include "numerics.cuh"
#include "ptx.cuh"

namespace vabft_dev {

namespace {

constexpr int kBM = 128, kBN = 256;
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;
// 3xTF32: 16-deep k blocks (64-byte rows, SWIZZLE_64B), 4 stages of hi + lo
// tiles; one pass: 32-deep k blocks (128-byte rows, SWIZZLE_128B), 4 stages.
// 48 KiB per stage either way (6 resp. 4 MMAs of 128 x 256 x 8 per stage).
template <bool kSplit>
struct TfCfg {
    static constexpr int kBK = kSplit ? 16 : 32;
    static constexpr uint32_t kATile = kBM * kBK * 4;
    static constexpr uint32_t kBTile = kBN * kBK * 4;
    static constexpr uint32_t kStage = (kSplit ? 2 : 1) * (kATile + kBTile);
    static constexpr int kStages = 4;
};
constexpr size_t kSmem = size_t(4) * 49152 + 1024 + 256;
static_assert(TfCfg<true>::kStage == 49152 && TfCfg<false>::kStage == 49152, "stage size");

struct Tf32Params {
    int M, N, K;
    int num_m, num_n, num_k, num_tiles;
    int group;  // row blocks per raster group
    float* C;
    WideEpilogue epi;
};

__device__ __forceinline__ uint64_t desc_sw64_kmajor(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t(1) << 16;                 // LBO (unused for swizzled K-major)
    d |= uint64_t(512 >> 4) << 32;          // SBO: 8 rows x 64 B
    d |= uint64_t(1) << 46;                 // descriptor version (sm_100)
    d |= uint64_t(4) << 61;                 // SWIZZLE_64B
    return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// grouped raster: 8 row blocks per group, so concurrently running tiles share
// A row panels and B column panels in L2
__device__ __forceinline__ void tile_mn(const Tf32Params& p, int t, int& m, int& n) {
    const int G = p.group;
    const int gsz = G * p.num_n;
    const int g = t / gsz, first = g * G;
    const int gm = p.num_m - first < G ? p.num_m - first : G;
    const int r = t % gsz;
    m = first + r % gm;
    n = r / gm;
}

template <bool kSplit, bool kAbft, bool kInject>
__global__ void __launch_bounds__(kThreads, 1)
    tf32_gemm_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                     const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl,
                     const __grid_constant__ Tf32Params p) {
    using Cfg = TfCfg<kSplit>;
    constexpr int kST = Cfg::kStages, kBK = Cfg::kBK;
    constexpr uint32_t kSB = Cfg::kStage, kATile = Cfg::kATile, kBTile = Cfg::kBTile;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // stage s: [A_hi | A_lo | B_hi | B_lo]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(kST) * kSB);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kST;
    uint64_t* tfull_bar = bars + 2 * kST;
    uint64_t* tempty_bar = bars + 2 * kST + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kST + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto a_hi = [&](int s) { return smem + size_t(s) * kSB; };
    auto a_lo = [&](int s) { return smem + size_t(s) * kSB + kATile; };
    auto b_hi = [&](int s) { return smem + size_t(s) * kSB + (kSplit ? 2 : 1) * kATile; };
    auto b_lo = [&](int s) { return smem + size_t(s) * kSB + 2 * kATile + kBTile; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kST; ++s) {
            mbar_init(smem_u32(&full_bar[s]), 1);
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&tfull_bar[a]), 1);
            mbar_init(smem_u32(&tempty_bar[a]), 4);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tAh);
        tma_prefetch_desc(&tBh);
        if constexpr (kSplit) {
            tma_prefetch_desc(&tAl);
            tma_prefetch_desc(&tBl);
        }
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // the wide A pass that follows (programmatic launch) may start on SMs this
    // grid leaves idle; it waits for the grid's completion before reading C
    griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                int mb, nb;
                tile_mn(p, t, mb, nb);
                for (int kb = 0; kb < p.num_k; ++kb) {
                    mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full_bar[stage]);
                    mbar_arrive_expect_tx(fb, kSB);
                    tma_load_2d(smem_u32(a_hi(stage)), &tAh, fb, kb * kBK, mb * kBM);
                    if constexpr (kSplit) tma_load_2d(smem_u32(a_lo(stage)), &tAl, fb, kb * kBK, mb * kBM);
                    tma_load_2d(smem_u32(b_hi(stage)), &tBh, fb, kb * kBK, nb * kBN);
                    if constexpr (kSplit) tma_load_2d(smem_u32(b_lo(stage)), &tBl, fb, kb * kBK, nb * kBN);
                    if (++stage == kST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // both operands K-major: kind::tf32 takes no MN-major (transposed)
            // operand on sm_100a — measured: the MMA leaves D untouched
            constexpr uint32_t idesc = umma_idesc_f16(2u /*TF32*/, false, kBM, kBN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                mbar_wait(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * kBN);
                for (int kb = 0; kb < p.num_k; ++kb) {
                    mbar_wait(smem_u32(&full_bar[stage]), phase);
                    tc_fence_after();
                    auto kdesc = [](uint32_t a) {
                        return kSplit ? desc_sw64_kmajor(a) : umma_desc_sw128(a, 16, 1024);
                    };
                    const uint64_t ah = kdesc(smem_u32(a_hi(stage)));
                    const uint64_t bh = kdesc(smem_u32(b_hi(stage)));
#pragma unroll
                    for (int k = 0; k < kBK / 8; ++k) {
                        // K-major operands: +32 bytes per 8 elements inside the swizzled row
                        const uint64_t ao = uint64_t((k * 32) >> 4), bo = ao;
                        const uint32_t first = (kb > 0 || k > 0) ? 1u : 0u;
                        if constexpr (kSplit) {
                            const uint64_t al = desc_sw64_kmajor(smem_u32(a_lo(stage)));
                            const uint64_t bl = desc_sw64_kmajor(smem_u32(b_lo(stage)));
                            umma_tf32(d, al + ao, bh + bo, idesc, first);
                            umma_tf32(d, ah + ao, bl + bo, idesc, 1u);
                            umma_tf32(d, ah + ao, bh + bo, idesc, 1u);
                        } else {
                            umma_tf32(d, ah + ao, bh + bo, idesc, first);
                        }
                    }
                    umma_commit(smem_u32(&empty_bar[stage]));
                    if (++stage == kST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(smem_u32(&tfull_bar[acc]));
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ------------------------------------------------------ epilogue
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            int mb, nb;
            tile_mn(p, t, mb, nb);
            const int row = mb * kBM + quad * 32 + lane;
            const int n0 = nb * kBN;
            const bool row_ok = row < p.M;
            int fcol = -1, fbit = 0, fdir = 0;
            if constexpr (kInject) {
                if (row_ok) {
                    fcol = p.epi.fault_col[row];
                    fbit = p.epi.fault_bit[row];
                    fdir = p.epi.fault_dir[row];
                }
            }
            mbar_wait(smem_u32(&tfull_bar[acc]), acc_phase);
            tc_fence_after();
            float s1 = 0.0f, s2 = 0.0f;
#pragma unroll 1
            for (int c = 0; c < kBN; c += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + (uint32_t(quad * 32) << 16) + uint32_t(acc * kBN + c), v);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    float x = saturate_accum<VABFT_FP32>(__uint_as_float(v[e]));
                    const int col = n0 + c + e;
                    if constexpr (kInject) {
                        if (col == fcol) {
                            const uint32_t bb = __float_as_uint(x);
                            const bool ok = bit_eligible(bb, fbit, fdir);
                            const uint32_t b2 = ok ? (bb ^ (1u << fbit)) : bb;
                            if (p.epi.fault_records) {
                                vabft_fault_record rr;
                                rr.value_before = double(x);
                                rr.value_after = double(__uint_as_float(b2));
                                rr.applied = ok ? 1 : 0;
                                rr.reserved = 0;
                                p.epi.fault_records[row] = rr;
                            }
                            x = __uint_as_float(b2);
                        }
                    }
                    if constexpr (kAbft) {
                        if (col < p.N) {
                            s1 = __fadd_rn(s1, x);
                            s2 = __fadd_rn(s2, __fmul_rn(float(col + 1), x));
                        }
                    }
                    v[e] = __float_as_uint(x);
                }
                if (row_ok) {
                    float* dst = p.C + size_t(row) * p.N + n0 + c;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        if (n0 + c + g * 4 + 4 <= p.N)
                            __stcs(reinterpret_cast<float4*>(dst + g * 4),
                                   make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]),
                                               __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3])));
                    }
                }
                if constexpr (kAbft) {
                    if ((c + 32) % 128 == 0) {
                        const int blk = (n0 + c) / 128;
                        if (row_ok && blk * 128 < p.N) {
                            const size_t o = size_t(blk) * size_t(p.epi.ld) + size_t(row);
                            static_cast<float*>(p.epi.part1)[o] = s1;
                            static_cast<float*>(p.epi.part2)[o] = s2;
                        }
                        s1 = 0.0f;
                        s2 = 0.0f;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[acc]));
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// hi = rna_tf32(x), lo = rna_tf32(x - hi) (lo = 0 for non-finite x)
__global__ void split_tf32_kernel(const float4* __restrict__ x, float4* __restrict__ hi, float4* __restrict__ lo,
                                  int64_t n4) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = x[i];
        float h[4], l[4];
        const float in[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint32_t hb, lb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(in[e]));
            h[e] = __uint_as_float(hb);
            const float r = isfinite(in[e]) ? __fsub_rn(in[e], h[e]) : 0.0f;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(r));
            l[e] = __uint_as_float(lb);
        }
        hi[i] = make_float4(h[0], h[1], h[2], h[3]);
        lo[i] = make_float4(l[0], l[1], l[2], l[3]);
    }
}

// The same split of a K x N row-major weight, written transposed (N x K,
// K-major) for the MMA's B operand: 32 x 32 tiles through shared memory.
__global__ void split_tf32_t_kernel(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                                    int64_t K, int64_t N) {
    __shared__ float th[32][33], tl[32][33];
    const int64_t k0 = int64_t(blockIdx.y) * 32, n0 = int64_t(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    for (int r = ty; r < 32; r += 8) {
        const int64_t k = k0 + r, n = n0 + tx;
        float h = 0.0f, l = 0.0f;
        if (k < K && n < N) {
            const float v = x[k * N + n];
            uint32_t hb, lb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
            h = __uint_as_float(hb);
            const float rr = isfinite(v) ? __fsub_rn(v, h) : 0.0f;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(rr));
            l = __uint_as_float(lb);
        }
        th[r][tx] = h;
        tl[r][tx] = l;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t n = n0 + r, k = k0 + tx;
        if (n < N && k < K) {
            hi[n * K + k] = th[tx][r];
            lo[n * K + k] = tl[tx][r];
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    if (!fn) fail(VABFT_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap map_f32(const float* base, uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows,
                    CUtensorMapSwizzle sw) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(VABFT_CUDA_ERROR, "cuTensorMapEncodeTiled(FP32) failed");
    return m;
}

template <bool kSplit, bool kAbft, bool kInject>
void launch_tf32(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh, const CUtensorMap& bl,
                 const Tf32Params& p, cudaStream_t s) {
    auto kern = tf32_gemm_kernel<kSplit, kAbft, kInject>;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), int(kSmem));
    const int grid = p.num_tiles < sm_count() ? p.num_tiles : sm_count();
    kern<<<grid, kThreads, kSmem, s>>>(ah, al, bh, bl, p);
    check_cuda(cudaGetLastError(), "tf32 gemm launch");
}

}  // namespace

void split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s) {
    if (n % 4 != 0) fail(VABFT_UNSUPPORTED, "split_tf32: element count must be a multiple of 4");
    const int64_t n4 = n / 4;
    const int64_t blocks = (n4 + 255) / 256;
    const unsigned grid = unsigned(blocks < 8 * 148 ? blocks : 8 * 148);
    split_tf32_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(reinterpret_cast<const float4*>(x),
                                                          reinterpret_cast<float4*>(hi),
                                                          reinterpret_cast<float4*>(lo), n4);
    check_cuda(cudaGetLastError(), "split_tf32 launch");
}

void split_tf32_t(const float* x, float* hi_t, float* lo_t, int64_t K, int64_t N, cudaStream_t s) {
    const dim3 grid(unsigned((N + 31) / 32), unsigned((K + 31) / 32));
    split_tf32_t_kernel<<<grid, 256, 0, s>>>(x, hi_t, lo_t, K, N);
    check_cuda(cudaGetLastError(), "split_tf32_t launch");
}

void tf32_gemm_launch(int64_t M, int64_t N, int64_t K, const float* a_hi, const float* a_lo, const float* b_hi,
                      const float* b_lo, float* C, const WideEpilogue& epi, cudaStream_t s) {
    if (M < 1 || N < 1 || K < 1) fail(VABFT_INVALID_ARGUMENT, "dims must be >= 1");
    if (K % 4 != 0 || N % 4 != 0) fail(VABFT_UNSUPPORTED, "FP32 tensor-core GEMM: K and N must be multiples of 4");
    if (M > (int64_t(1) << 30) || N > (int64_t(1) << 30) || K > (int64_t(1) << 30))
        fail(VABFT_UNSUPPORTED, "FP32 tensor-core GEMM: dims too large");
    const bool split = a_lo != nullptr;
    if (split != (b_lo != nullptr)) fail(VABFT_INVALID_ARGUMENT, "3xTF32 needs both lo parts");
    Tf32Params p{};
    p.M = int(M);
    p.N = int(N);
    p.K = int(K);
    p.num_m = int((M + kBM - 1) / kBM);
    p.num_n = int((N + kBN - 1) / kBN);
    const int bk = split ? TfCfg<true>::kBK : TfCfg<false>::kBK;
    const CUtensorMapSwizzle sw = split ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    p.num_k = int((K + bk - 1) / bk);
    p.num_tiles = p.num_m * p.num_n;
    static const int grp_env = [] {  // developer override (VABFT_TF32_GROUP)
        const char* e = std::getenv("VABFT_TF32_GROUP");
        return e ? std::atoi(e) : 0;
    }();
    p.group = grp_env > 0 ? grp_env : 8;
    p.C = C;
    p.epi = epi;
    const CUtensorMap ah = map_f32(a_hi, M, K, bk, kBM, sw);
    const CUtensorMap bh = map_f32(b_hi, N, K, bk, kBN, sw);
    const CUtensorMap al = split ? map_f32(a_lo, M, K, bk, kBM, sw) : ah;
    const CUtensorMap bl = split ? map_f32(b_lo, N, K, bk, kBN, sw) : bh;
    const bool inj = epi.abft && epi.fault_col != nullptr;
    if (split) {
        if (!epi.abft) launch_tf32<true, false, false>(ah, al, bh, bl, p, s);
        else if (inj) launch_tf32<true, true, true>(ah, al, bh, bl, p, s);
        else launch_tf32<true, true, false>(ah, al, bh, bl, p, s);
    } else {
        if (!epi.abft) launch_tf32<false, false, false>(ah, al, bh, bl, p, s);
        else if (inj) launch_tf32<false, true, true>(ah, al, bh, bl, p, s);
        else launch_tf32<false, true, false>(ah, al, bh, bl, p, s);
    }
}

void tf32_gemm_run(int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* C, const WideEpilogue& epi,
                   int passes, cudaStream_t s) {
    float* buf = nullptr;
    const size_t na = size_t(M) * size_t(K), nb = size_t(K) * size_t(N);
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * (na + nb) * sizeof(float), s), "cudaMallocAsync");
    split_tf32_t(B, buf + 2 * na, buf + 2 * na + nb, K, N, s);
    if (passes == 1) {
        tf32_gemm_launch(M, N, K, A, nullptr, buf + 2 * na, nullptr, C, epi, s);
    } else {
        split_tf32(A, buf, buf + na, int64_t(na), s);
        tf32_gemm_launch(M, N, K, buf, buf + na, buf + 2 * na, buf + 2 * na + nb, C, epi, s);
    }
    check_cuda(cudaFreeAsync(buf, s), "cudaFreeAsync");
}

}  // namespace vabft_dev
