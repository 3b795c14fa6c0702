// tcgen05 fused ABFT-GEMM for BF16/FP16 inputs with FP32 accumulation in
// TMEM — the B200 replacement of gemm_emulated_with_accum's 16-bit path
// (proj/src/precision.cpp:238-338) plus the epilogue half of row_sums
// (proj/src/checksum.cpp:160-187), the accumulator/output fault injector
// (proj/src/faults.cpp:104-168) and, fused into the operand stream, the A-side
// statistics of vabft_thresholds / encode (threshold_vabft.cpp:54-61,
// checksum.cpp:103-146).
//
// Structure (one CTA per SM, persistent over 128 x 256 output tiles):
//   warp 0      TMA producer: A tile 128x64 (K-major, SW128) and B tile
//               64x256 (N-major 4 x [64k x 64n] boxes, or K-major 256x64)
//               into a 4-stage smem ring guarded by full/empty mbarriers.
//   warp 1      TMEM allocator (512 cols = 2 accumulators of 256 FP32 cols)
//               and single-thread tcgen05.mma issuer (M=128, N=256, K=16).
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers; saturate; optional
//               bit-flip injection; quantize (RNE, satfinite); store C; row
//               partials r1 = sum_j v, r2 = sum_j (j+1) v in FP32, one
//               partial per 128-column block (the reference's blocked:128
//               reduction order), written as [block][M] for the verify tail.
//   warps 6..9  (fused path only) A statistics: see stats_warps below.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "internal.hpp"
#include "numerics.cuh"
#include "ptx.cuh"
#include "tail.cuh"

namespace vabft_dev {

// developer timeline buffer (VABFT_TRACE): 8 stamps per CTA, read back with
// vabft_debug_trace
__device__ unsigned long long g_trace[1024 * 8];

namespace {

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kBM = 128;
constexpr int kBN = 256;
constexpr int kBK = 64;
#ifndef VABFT_STAGES
#define VABFT_STAGES 4
#endif
constexpr int kStages = VABFT_STAGES;
constexpr int kThreads = 192;       // TMA, MMA, 4 epilogue warps
#ifndef VABFT_STATS_REMAP
#define VABFT_STATS_REMAP 0
#endif
// + 4 A-statistics warps + 1 statistics producer; with VABFT_STATS_REMAP the
// statistics warps are 6, 7, 8, 10 and the producer 11 (warp 9 idle), so the
// MMA issuer's SM sub-partition (warp % 4 == 1) hosts no statistics warp
constexpr int kThreadsStats = VABFT_STATS_REMAP ? 384 : 352;
constexpr int kStatsProducerWarp = VABFT_STATS_REMAP ? 11 : 10;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KiB
constexpr uint32_t kBBytes = kBN * kBK * 2;  // 32 KiB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kTmemCols = 512;
constexpr size_t kSmemBytes = size_t(kStages) * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
static_assert(size_t(kStages) * kStageBytes + 2 * (kABytes + 2 * kBK * 4) + 1024 + 256 <= 232448, "smem budget");
// + the statistics warps' private 2-slot A ring (fused path)
constexpr uint32_t kSlotBytes = kABytes + 2 * kBK * 4;  // A tile + B r1/B r2 segments
constexpr size_t kSmemBytesStats = kSmemBytes + 2 * size_t(kSlotBytes);
// CTA-pair kernel: 16 KiB of A + 16 KiB of B per stage per CTA
constexpr int kStagesPair = 6;
constexpr size_t kSmemBytesPair = size_t(kStagesPair) * (kABytes + kBBytes / 2) + 1024 + 256;
constexpr size_t kSmemBytesPairStats = kSmemBytesPair + 2 * size_t(kSlotBytes);
static_assert(kSmemBytesPairStats <= 232448, "pair smem budget");
static_assert((2 * kStagesPair + 9 + 9) * 8 <= 256, "pair barrier area");
// warps running the in-kernel verify tail, each with a 24 KiB slice of the
// (then idle) pipeline shared memory
constexpr int kTailWarps = 9;
static_assert(kTailWarps * kTailWarpSmem <= kStages * kStageBytes + 2 * kSlotBytes, "tail smem slices");
static_assert((2 * kStages + 9 + kTailWarps) * 8 <= 256, "barrier area");

struct TcParams {
    int M, N, K;
    int num_m_blk, num_n_blk, num_k_blk, num_tiles;
    // work units of the persistent loop: tiles [0, split_from) whole, each
    // later tile as two 128-column halves (pair mode's under-filled last wave)
    int split_from, num_units;
    int group_m;  // tile raster: groups of group_m row blocks, n-major inside a group
    int pair;     // 1: CTA-pair kernel (tiles of 256 rows, num_m_blk in 256-row blocks)
    uint16_t* C;
    int64_t ldc;  // row stride of C (elements)
    TcEpilogue epi;
};

// Grouped raster: tiles run through groups of group_m consecutive 128-row
// blocks; inside a group the row block varies fastest, so the CTAs of one
// wave share B tiles across the group and every row block of a group
// completes (all N tiles done) at the same time, group after group, which is
// what lets streamed verification run while later groups are still in the
// tensor cores. group_m = num_m_blk is the plain n-major order.
__device__ __forceinline__ void tile_coords(const TcParams& p, int tile, int& m_blk, int& n_blk) {
    const int per_group = p.group_m * p.num_n_blk;
    const int grp = tile / per_group;
    const int rem = tile - grp * per_group;
    const int m0 = grp * p.group_m;
    const int gm = p.num_m_blk - m0 < p.group_m ? p.num_m_blk - m0 : p.group_m;
    m_blk = m0 + rem % gm;
    n_blk = rem / gm;
}

// This CTA's persistent tile loop. In pair mode (2 x 1 clusters, cta_group::2)
// both CTAs of a pair walk the same pair tiles (256 x 256 outputs; num_m_blk
// counts 256-row blocks) and each owns one 128-row half, so everything
// downstream of the MMA sees 128-row blocks either way.
__device__ __forceinline__ int tile_first(const TcParams& p) {
    return p.pair ? int(blockIdx.x >> 1) : int(blockIdx.x);
}
__device__ __forceinline__ int tile_stride(const TcParams& p) {
    return p.pair ? int(gridDim.x >> 1) : int(gridDim.x);
}
__device__ __forceinline__ void cta_tile(const TcParams& p, int tile, int& m_blk, int& n_blk) {
    tile_coords(p, tile, m_blk, n_blk);
    if (p.pair) m_blk = 2 * m_blk + int(cluster_ctarank());
}
// Work unit u: its tile, and half = -1 (whole 256-column tile) or 0 / 1 (the
// tile's left / right 128 columns). Splitting the last wave's tiles when it
// would leave more than half the pairs idle: 4096^3 is 256 pair tiles = 3
// waves of 74 + 34, and the 34 become 68 half tiles (each CTA then streams
// 8 KiB of B per k-block; the whole tile would stream 16).
__device__ __forceinline__ void cta_unit(const TcParams& p, int u, int& m_blk, int& n_blk, int& half) {
    int tile = u;
    half = -1;
    if (u >= p.split_from) {
        tile = p.split_from + ((u - p.split_from) >> 1);
        half = (u - p.split_from) & 1;
    }
    cta_tile(p, tile, m_blk, n_blk);
}
// arrival weight of a unit on the streamed-verification counters: a whole
// tile counts 2, a half 1 (targets are 2 per N tile)
__device__ __forceinline__ unsigned int unit_weight(int half) { return half < 0 ? 2u : 1u; }

// Streamed verification (see TcEpilogue::stream_verify). Per 32-row group g
// two self-resetting counters: group_cnt[2g] counts statistics arrivals (one
// per N tile), group_cnt[2g+1] final arrivals (one per N tile from the
// epilogue + one from the statistics half). __syncwarp orders every lane's
// partial / atomic writes before lane 0's acq_rel RMW at GPU scope (release
// is cumulative); the acquire side orders the verifier's L2 reads after all
// earlier arrivals. (A __threadfence per lane is fence.sc + L1 invalidate.)
__device__ __forceinline__ unsigned int warp_arrive(unsigned int* cnt, unsigned int w) {
    __syncwarp();
    unsigned int old = 0;
    if ((threadIdx.x & 31) == 0) old = atom_add_acq_rel_gpu(cnt, w);
    return __shfl_sync(0xffffffffu, old, 0);
}

template <int F>
__device__ __forceinline__ void final_arrive(const TcParams& p, int64_t g, unsigned int w) {
    unsigned int* cnt = p.epi.group_cnt + 2 * g + 1;
    // target 2 num_n_blk (epilogue units) + 2 (the statistics half)
    if (warp_arrive(cnt, w) + w != 2u * unsigned(p.num_n_blk) + 2u) return;
    if (p.epi.debug != 7 && p.epi.debug != 9) final_half_direct<F>(p.epi.tail, g);  // 7: no verification, 9: no final half
    __syncwarp();
    if ((threadIdx.x & 31) == 0) *cnt = 0u;  // ready for the next launch
}

template <int F>
__device__ __forceinline__ void stats_arrive(const TcParams& p, int64_t g, unsigned int w) {
    unsigned int* cnt = p.epi.group_cnt + 2 * g;
    if (warp_arrive(cnt, w) + w != 2u * unsigned(p.num_n_blk)) return;
    const unsigned long long t0 = p.epi.trace ? gtime() : 0ull;
    if (p.epi.debug != 7 && p.epi.debug != 8) stats_half_direct<F>(p.epi.tail, g);
    if (p.epi.trace && (threadIdx.x & 31) == 0) {
        atomicAdd(p.epi.trace + blockIdx.x * 8 + 6, gtime() - t0);
        atomicAdd(p.epi.trace + blockIdx.x * 8 + 7, 1ull);
    }  // 8: no statistics half
    __syncwarp();
    if ((threadIdx.x & 31) == 0) *cnt = 0u;
    final_arrive<F>(p, g, 2u);
}

// ----------------------------------------------------- operand faults
// inject (faults.cpp:104-168) on an operand element as the tensor cores see
// it: one 16-bit pattern in a swizzled shared-memory tile.
template <int F>
__device__ __forceinline__ void flip16(uint16_t* e, int bit, int dir, vabft_fault_record* rec) {
    const uint16_t before = *e;
    const bool ok = bit_eligible(before, bit, dir);
    const uint16_t after = ok ? uint16_t(before ^ (1u << bit)) : before;
    *e = after;
    if (rec) {
        vabft_fault_record r;
        r.value_before = double(bits16_to_float<F>(before));
        r.value_after = double(bits16_to_float<F>(after));
        r.applied = ok ? 1 : 0;
        r.reserved = 0;
        *rec = r;
    }
}

// Apply the planned operand faults that fall into k-stage kb of tile
// (m_blk, n_blk) to the stage's A / B tiles (called by all lanes of the MMA
// warp after the stage's full barrier, before the MMAs). SWIZZLE_128B: a
// 128-byte row r keeps 16-byte chunk c at chunk c ^ (r & 7). A is K-major
// (row = A row, 64 k per row); B is N-major as 4 boxes of 64 k-rows x 64 n
// (8 KiB each) or K-major (row = B column). Every tile of the row / column
// block gets the same flip (the element as seen by all MMAs); the record is
// written once. The statistics warps read their own A copy and the B-side
// checksums come from the clean B, so the checksums stay clean.
template <int F, bool kBKMajor>
__device__ __forceinline__ void operand_faults_stage(const TcParams& p, uint8_t* sa, uint8_t* sb, int m_blk,
                                                     int n_blk, int kb) {
    const int lane = threadIdx.x & 31;
    const int k0 = kb * 64;
    bool wrote = false;
    if (p.epi.fault_target == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = q * 32 + lane;
            const int row = m_blk * 128 + r;
            if (row >= p.M) continue;
            const int k = p.epi.fault_col[row];
            if (k < k0 || k >= k0 + 64) continue;
            const int kk = k - k0;
            uint16_t* e = reinterpret_cast<uint16_t*>(sa + r * 128 + ((((kk >> 3) ^ (r & 7))) << 4) + (kk & 7) * 2);
            flip16<F>(e, p.epi.fault_bit[row], p.epi.fault_dir[row],
                      (n_blk == 0 && p.epi.fault_records) ? p.epi.fault_records + row : nullptr);
            wrote = true;
        }
    } else {
        for (int t = lane; t < p.epi.n_operand_faults; t += 32) {
            const vabft_fault f = p.epi.operand_faults[t];
            if (f.i < k0 || f.i >= k0 + 64 || f.j < int64_t(n_blk) * 256 || f.j >= int64_t(n_blk) * 256 + 256) continue;
            const int kk = int(f.i - k0), jj = int(f.j - int64_t(n_blk) * 256);
            uint8_t* a = kBKMajor ? sb + jj * 128 + ((((kk >> 3) ^ (jj & 7))) << 4) + (kk & 7) * 2
                                  : sb + (jj >> 6) * 8192 + kk * 128 + (((((jj & 63) >> 3) ^ (kk & 7))) << 4) +
                                        (jj & 7) * 2;
            flip16<F>(reinterpret_cast<uint16_t*>(a), f.bit, f.direction,
                      (m_blk == 0 && p.epi.operand_fault_records) ? p.epi.operand_fault_records + t : nullptr);
            wrote = true;
        }
    }
    // generic-proxy writes -> the tensor cores' async-proxy reads
    if (wrote) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// N tiles of a row block that compute its statistics: K block b belongs to
// tile b mod stats_tiles (all N tiles: concentrating the blocks on fewer
// tiles was measured to put the statistics warps on the critical path).
__device__ __forceinline__ int stats_tiles(const TcParams& p) { return p.num_n_blk; }

// ------------------------------------------------ in-GEMM A statistics
// Four statistics warps (thread = row of the 128-row A tile). The 128-column
// K blocks b are spread over the N tiles: the CTA computing tile
// (m_blk, n_blk) owns the blocks with b % num_n_blk == n_blk, so each
// (row, block) is processed exactly once and the work is balanced. For an
// owned k-stage the TMA producer issues a second load of the same A tile
// into the statistics warps' private 2-slot ring (own full/empty barriers),
// so the MMA ring never waits on statistics; the next owned pair of stages
// is ~2*num_n_blk stages away, far more than the arithmetic needs. Per
// (row, b) the warps write the blocked:128 checksum partials
// sum_k fl(br[k] A[i][k]) (sequential in k) and the exact FP64 row-sum
// partial with packed max / min / min-nonzero trackers (the order-independent
// exactness guard, see aside.cu). A tile row r lives at byte r*128 of a slot
// with 16-byte chunk c stored at chunk c ^ (r & 7) (SWIZZLE_128B), so 8
// consecutive threads hit 8 distinct bank groups.
__device__ __forceinline__ uint32_t pminu2_(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t pmaxu2_(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
template <int F>
__device__ __forceinline__ uint32_t pmax2_(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (F == VABFT_BF16) asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
template <int F>
__device__ __forceinline__ uint32_t pmin2_(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (F == VABFT_BF16) asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// Exact row sums without FP64 arithmetic. FP64 instructions issued next to a
// running tcgen05 pipeline cost tensor-pipe cycles on B200 (measured: an FP64
// add per element in these warps cut the GEMM's flops/cycle by ~12%, the
// same work in integer/FP32 ~3%), so each 64-element stage of a row is summed
// as an integer: element = m * 2^(e - bias) with the stage anchored at
// ebase = (stage max exponent) - 48, i.e. m << (e - ebase) < 2^56 and 64 terms
// < 2^62. Under the exactness guard (tail.cuh guard_exact: every nonzero
// element's lsb is within 45 bits of the row maximum) no element falls below
// the anchor and the stage sum is exactly representable in FP64, so the one
// int64 -> double conversion per stage is exact and equals the reference's
// Neumaier sum once all stages are added. Rows that fail the guard take the
// sequential fallback, so what this computes for them is irrelevant.
// FP16's exponent range is narrow enough for a fixed anchor (ebase = 1).
template <int F>
struct StatsAcc {
    static constexpr int kFracBits = F == VABFT_BF16 ? 7 : 10;
    static constexpr int kExpMask = F == VABFT_BF16 ? 0xFF : 0x1F;
    static constexpr int kBias = F == VABFT_BF16 ? 127 + 7 : 15 + 10;  // value = m * 2^(e - kBias)
    float p1, p2;
    double s;  // exact FP64 sum of the finished stages
    uint32_t vmax, vmin, vmnz;
    __device__ __forceinline__ void reset() {
        p1 = p2 = 0.0f;
        s = 0.0;
        vmax = F == VABFT_BF16 ? 0xFF80FF80u : 0xFC00FC00u;
        vmin = F == VABFT_BF16 ? 0x7F807F80u : 0x7C007C00u;
        vmnz = 0x7FFF7FFFu;
    }
    // pass 1 over a granule: max / min / min-nonzero trackers and the stage's
    // largest magnitude pattern (packed u16 max)
    __device__ __forceinline__ void track(const uint4 w, uint32_t& amx) {
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            vmax = pmax2_<F>(vmax, ws[h]);
            vmin = pmin2_<F>(vmin, ws[h]);
            const uint32_t mag = ws[h] & 0x7FFF7FFFu;
            vmnz = pminu2_(vmnz, ((mag | 0x80008000u) - 0x00010001u) & 0x7FFF7FFFu);
            if constexpr (F == VABFT_BF16) amx = pmaxu2_(amx, mag);
        }
    }
    __device__ __forceinline__ static int anchor(uint32_t amx) {
        if constexpr (F == VABFT_BF16) {
            const int e0 = int((amx >> 7) & 0xFFu), e1 = int((amx >> 23) & 0xFFu);
            return (e0 > e1 ? e0 : e1) - 48;
        } else {
            return 1;  // m < 2^11, shift <= 30: 64 terms < 2^47
        }
    }
    __device__ __forceinline__ static void isum(uint32_t x, int ebase, uint64_t& pos, uint64_t& neg) {
        const uint32_t e = (x >> kFracBits) & uint32_t(kExpMask);
        const uint32_t m = (x & ((1u << kFracBits) - 1u)) | (e ? (1u << kFracBits) : 0u);
        const int sh = int(e ? e : 1u) - ebase;
        const uint64_t t = sh >= 0 ? (uint64_t(m) << sh) : 0ull;  // sh < 0 only for guard failures
        if (x & 0x8000u) neg += t;
        else pos += t;
    }
    // pass 2 over a granule (8 consecutive elements k .. k+7): blocked:128
    // checksum partials in FP32 (reference order, no FMA) and the integer sum
    __device__ __forceinline__ void sums(const uint4 w, const float* br1, const float* br2, int k, int ebase,
                                         uint64_t& pos, uint64_t& neg) {
        const float4* g1 = reinterpret_cast<const float4*>(br1 + k);  // shared memory (broadcast)
        const float4* g2 = reinterpret_cast<const float4*>(br2 + k);
        const float4 u0 = g1[0], u1 = g1[1], v0 = g2[0], v1 = g2[1];
        const float b1[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
        const float b2[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        // the element's integer image m * 2^(e - ebase) = x * 2^(kBias - ebase):
        // one exact power-of-two FMUL and one float -> int64 conversion (exact
        // for every element at or above the anchor, truncated below it like the
        // shift path — such rows fail the guard) instead of ~12 integer
        // instructions; the shift path remains for stages too small for the
        // float scale (stage maximum below 2^-72)
        const int se = kBias - ebase + 127;
        const bool fast = se >= 1 && se <= 254;
        const float S = __int_as_float((fast ? se : 127) << 23);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float xa = bits16_to_float<F>(uint16_t(ws[h] & 0xFFFFu));
            const float xb = bits16_to_float<F>(uint16_t(ws[h] >> 16));
            if (fast) {
                pos += static_cast<uint64_t>(__float2ll_rz(__fmul_rn(xa, S)));
                pos += static_cast<uint64_t>(__float2ll_rz(__fmul_rn(xb, S)));
            } else {
                isum(ws[h] & 0xFFFFu, ebase, pos, neg);
                isum(ws[h] >> 16, ebase, pos, neg);
            }
            // the two checksum chains' sums as one packed FADD2 per element.
            // Products stay scalar FMUL: ptxas (12.9) contracts mul.rn.f32x2 +
            // add.rn.f32x2 into FFMA2, which would change the rounding.
            float2 pp = make_float2(p1, p2);
            pp = __fadd2_rn(pp, make_float2(__fmul_rn(b1[2 * h], xa), __fmul_rn(b2[2 * h], xa)));
            pp = __fadd2_rn(pp, make_float2(__fmul_rn(b1[2 * h + 1], xb), __fmul_rn(b2[2 * h + 1], xb)));
            p1 = pp.x;
            p2 = pp.y;
        }
    }
    // close a stage: s += (pos - neg) * 2^(ebase - kBias), exact under the guard
    __device__ __forceinline__ void close_stage(uint64_t pos, uint64_t neg, int ebase) {
        const double scale = __longlong_as_double(static_cast<long long>(ebase - kBias + 1023) << 52);
        s = __dadd_rn(s, __dmul_rn(__ll2double_rn(static_cast<long long>(pos - neg)), scale));
    }
};

// Statistics producer (one thread): walks the CTA's owned (tile, 128-block,
// k-stage) sequence and TMA-loads each A tile + its B r segments into the
// 2-slot statistics ring, independently of the main MMA ring.
__device__ __forceinline__ void stats_producer(const TcParams& p, const CUtensorMap* tmA, uint8_t* smS,
                                               uint64_t* sfull_bar, uint64_t* sempty_bar) {
    uint32_t cnt = 0;
    const int nblk = (p.K + 127) / 128;
    for (int u = tile_first(p); u < p.num_units; u += tile_stride(p)) {
        int m_blk, n_blk, half;
        cta_unit(p, u, m_blk, n_blk, half);
        // a half tile takes every other one of its tile's blocks
        const int st = stats_tiles(p) * (half < 0 ? 1 : 2);
        for (int b = n_blk + (half > 0 ? stats_tiles(p) : 0); n_blk < stats_tiles(p) && b < nblk; b += st) {
            for (int kb = 2 * b; kb < 2 * b + 2 && kb < p.num_k_blk; ++kb, ++cnt) {
                const int slot = int(cnt & 1u);
                mbar_wait_sleep(smem_u32(&sempty_bar[slot]), ((cnt >> 1) & 1u) ^ 1u, 1000000u);
                const uint32_t sb = smem_u32(&sfull_bar[slot]);
                // slot layout: [A tile 0][A tile 1] (1024-aligned for SW128), then the
                // [B r1 | B r2] segments; the br arrays are padded to 128 entries
                const uint32_t adst = smem_u32(smS + slot * kABytes);
                const uint32_t bdst = smem_u32(smS + 2 * kABytes + slot * (2 * kBK * 4));
                if (p.epi.debug == 1 || p.epi.debug == 10) {  // ablation: no statistics loads (10: nor math)
                    mbar_arrive(sb);
                    continue;
                }
                mbar_arrive_expect_tx(sb, kSlotBytes);
                tma_load_2d(adst, tmA, sb, kb * kBK, m_blk * kBM);
                bulk_load(bdst, p.epi.br1 + kb * kBK, kBK * 4, sb);
                bulk_load(bdst + kBK * 4, p.epi.br2 + kb * kBK, kBK * 4, sb);
            }
        }
    }
}

template <int kFmt>
__device__ __forceinline__ void stats_warps(const TcParams& p, const uint8_t* smS, uint64_t* sfull_bar,
                                            uint64_t* sempty_bar, int sw, int lane) {
    const int r = sw * 32 + lane;  // row within the 128-row tile
    StatsAcc<kFmt> acc;
    acc.reset();
    uint32_t cnt = 0;  // statistics stages consumed: slot = cnt & 1, phase = (cnt >> 1) & 1
    const int nblk = (p.K + 127) / 128;
    for (int u = tile_first(p); u < p.num_units; u += tile_stride(p)) {
        int m_blk, n_blk, half;
        cta_unit(p, u, m_blk, n_blk, half);
        const int row = m_blk * kBM + r;
        const int st = stats_tiles(p) * (half < 0 ? 1 : 2);  // as stats_producer
        for (int b = n_blk + (half > 0 ? stats_tiles(p) : 0); n_blk < stats_tiles(p) && b < nblk; b += st) {
            for (int kb = 2 * b; kb < 2 * b + 2 && kb < p.num_k_blk; ++kb, ++cnt) {
                const int slot = int(cnt & 1u);
                mbar_wait_sleep(smem_u32(&sfull_bar[slot]), (cnt >> 1) & 1u, 1000000u);
                const uint8_t* trow = smS + slot * kABytes + r * 128;
                const float* sbr1 = reinterpret_cast<const float*>(smS + 2 * kABytes + slot * (2 * kBK * 4));
                const float* sbr2 = sbr1 + kBK;
                const int kbase = kb * kBK;
                const int ng = (p.K - kbase) >= kBK ? 8 : (p.K - kbase) / 8;  // K % 8 == 0: whole granules
                if (p.epi.debug != 2 && p.epi.debug != 10) {  // 2 / 10: ablation, no math
                    if (ng == 8) {  // whole stage: one shared-memory pass into registers
                        uint4 v[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) v[c] = *reinterpret_cast<const uint4*>(trow + ((c ^ (r & 7)) << 4));
                        uint32_t amx = 0;
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc.track(v[c], amx);
                        const int ebase = StatsAcc<kFmt>::anchor(amx);
                        uint64_t pos = 0, neg = 0;
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc.sums(v[c], sbr1, sbr2, c * 8, ebase, pos, neg);
                        acc.close_stage(pos, neg, ebase);
                    } else {
                        uint32_t amx = 0;
                        for (int c = 0; c < ng; ++c)
                            acc.track(*reinterpret_cast<const uint4*>(trow + ((c ^ (r & 7)) << 4)), amx);
                        const int ebase = StatsAcc<kFmt>::anchor(amx);
                        uint64_t pos = 0, neg = 0;
                        for (int c = 0; c < ng; ++c)
                            acc.sums(*reinterpret_cast<const uint4*>(trow + ((c ^ (r & 7)) << 4)), sbr1, sbr2,
                                     c * 8, ebase, pos, neg);
                        acc.close_stage(pos, neg, ebase);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&sempty_bar[slot]));
            }
            if (row < p.M) {  // end of the 128-column block b
                const size_t o = part_index(b, row, nblk);
                p.epi.sp1[o] = acc.p1;
                p.epi.sp2[o] = acc.p2;
                // order-independent statistics: per-row atomics (exact sum under
                // the guard; max / min / min-nonzero via order keys)
                atomicAdd(p.epi.rsum + row, acc.s);
                const float hx = fmaxf(bits16_to_float<kFmt>(uint16_t(acc.vmax & 0xFFFFu)),
                                       bits16_to_float<kFmt>(uint16_t(acc.vmax >> 16)));
                const float hn = fminf(bits16_to_float<kFmt>(uint16_t(acc.vmin & 0xFFFFu)),
                                       bits16_to_float<kFmt>(uint16_t(acc.vmin >> 16)));
                atomicMax(p.epi.rmax + row, fkey(hx));
                atomicMin(p.epi.rmin + row, fkey(hn));
                const uint32_t mz = min(acc.vmnz & 0xFFFFu, acc.vmnz >> 16);
                if (mz < 0x7FFFu) atomicMin(p.epi.rmnz + row, mz);
            }
            acc.reset();
        }
        if (p.epi.stream_verify && (int64_t(m_blk) * 4 + sw) * 32 < p.M)
            stats_arrive<kFmt>(p, int64_t(m_blk) * 4 + sw, unit_weight(half));
    }
    if (p.epi.trace && lane == 0) atomicMax(p.epi.trace + blockIdx.x * 8 + 3, gtime());
}

template <int kFmt, bool kBKMajor, int kAbft, bool kInject, bool kStats, bool kPair = false>
__global__ void __launch_bounds__(kThreadsStats, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ TcParams p) {
    // Pair mode: the leader's tcgen05.mma.cta_group::2 (M = 256) reads 128 A
    // rows and 128 B columns from each CTA's ring, so a CTA stages 32 KiB per
    // k-block instead of 48 and holds kStagesPair stages in the same space.
    constexpr int kST = kPair ? kStagesPair : kStages;
    constexpr uint32_t kBB = kPair ? kBBytes / 2 : kBBytes;
    constexpr uint32_t kSB = kABytes + kBB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* smA = smem;
    uint8_t* smB = smem + kST * kABytes;
    uint8_t* smS = smem + kST * kSB;  // statistics ring (kStats only)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smS + (kStats ? 2 * kSlotBytes : 0));
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kST;
    uint64_t* tfull_bar = bars + 2 * kST;
    uint64_t* tempty_bar = bars + 2 * kST + 2;
    uint64_t* sfull_bar = bars + 2 * kST + 4;
    uint64_t* sempty_bar = bars + 2 * kST + 6;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kST + 8);
    uint64_t* tail_bar = bars + 2 * kST + 9;  // kTailWarps verify-tail barriers

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = kPair ? cluster_ctarank() : 0u;  // 0 = the pair's MMA leader

    if (threadIdx.x == 0) {
        for (int s = 0; s < kST; ++s) {
            // pair: the leader's full barrier takes an arrival from each CTA's
            // producer and the transaction bytes of both halves
            mbar_init(smem_u32(&full_bar[s]), kPair ? 2 : 1);
            mbar_init(smem_u32(&empty_bar[s]), 1);  // MMA commit (multicast to both CTAs in pair mode)
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&tfull_bar[a]), 1);
            mbar_init(smem_u32(&tempty_bar[a]), kPair ? 8 : 4);  // both CTAs' epilogue warps (leader's)
            mbar_init(smem_u32(&sfull_bar[a]), 1);
            mbar_init(smem_u32(&sempty_bar[a]), 4);  // the 4 statistics warps
        }
        if constexpr (kStats) {
            for (int w = 0; w < kTailWarps; ++w) mbar_init(smem_u32(&tail_bar[w]), 1);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) {
        if constexpr (kPair) tmem_alloc_pair(smem_u32(tmem_slot), kTmemCols);
        else tmem_alloc(smem_u32(tmem_slot), kTmemCols);
    }
    tc_fence_before();
    if constexpr (kPair) cluster_sync_all();  // barriers initialised in both CTAs before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (p.epi.trace && threadIdx.x == 0) p.epi.trace[blockIdx.x * 8 + 0] = gtime();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int u = tile_first(p); u < p.num_units; u += tile_stride(p)) {
                int m_blk, n_blk, half;
                cta_unit(p, u, m_blk, n_blk, half);
                const int nw = half < 0 ? kBN : kBN / 2;              // unit width
                const int n0 = n_blk * kBN + (half > 0 ? kBN / 2 : 0);  // first column
                for (int kb = 0; kb < p.num_k_blk; ++kb) {
                    mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full_bar[stage]);
                    const uint32_t adst = smem_u32(smA + stage * kABytes);
                    const uint32_t bdst = smem_u32(smB + stage * kBB);
                    if constexpr (kPair) {
                        // this CTA's 128 A rows and nw / 2 of the unit's nw B columns,
                        // completion bytes on the leader's full barrier
                        if (rank == 0) mbar_arrive_expect_tx(fb, 2 * (kABytes + uint32_t(nw) * kBK));
                        else mbar_arrive_cluster_relaxed(mapa_shared(fb, 0));
                        tma_load_2d_pair(adst, &tmA, fb, kb * kBK, m_blk * kBM);
                        for (int c = 0; c < nw / 128; ++c)
                            tma_load_2d_pair(bdst + c * 8192, &tmB, fb, n0 + int(rank) * (nw / 2) + c * 64, kb * kBK);
                    } else {
                        mbar_arrive_expect_tx(fb, kStageBytes);
                        tma_load_2d(adst, &tmA, fb, kb * kBK, m_blk * kBM);
                        if constexpr (kBKMajor) {
                            tma_load_2d(bdst, &tmB, fb, kb * kBK, n_blk * kBN);
                        } else {
#pragma unroll
                            for (int c = 0; c < kBN / 64; ++c)
                                tma_load_2d(bdst + c * 8192, &tmB, fb, n_blk * kBN + c * 64, kb * kBK);
                        }
                    }
                    if (++stage == kST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // With operand faults (campaign instantiations only) the whole warp
        // walks the stages: its lanes flip the planned operand bits in the
        // freshly loaded shared-memory tiles before lane 0 issues the MMAs.
        const bool opf = kInject && !kPair && p.epi.fault_target != 0;  // operand faults: one-CTA kernel only
        // pair mode: only the leader issues (cta_group::2, M = 256)
        if ((lane == 0 || opf) && rank == 0) {
            // --------------------------------------------------- MMA issuer
            constexpr uint32_t idesc =
                umma_idesc_f16(kFmt == VABFT_BF16 ? 1u : 0u, !kBKMajor, kPair ? 2 * kBM : kBM, kBN);
            constexpr uint32_t idesc_half =
                umma_idesc_f16(kFmt == VABFT_BF16 ? 1u : 0u, !kBKMajor, kPair ? 2 * kBM : kBM, kBN / 2);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int u = tile_first(p); u < p.num_units; u += tile_stride(p)) {
                int m_blk = 0, n_blk = 0, half = -1;
                cta_unit(p, u, m_blk, n_blk, half);
                const uint32_t id = half < 0 ? idesc : idesc_half;
                if (lane == 0) {
                    mbar_wait(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
                    tc_fence_after();
                }
                const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
                for (int kb = 0; kb < p.num_k_blk; ++kb) {
                    mbar_wait(smem_u32(&full_bar[stage]), phase);
                    if constexpr (kInject) {
                        if (opf) {
                            operand_faults_stage<kFmt, kBKMajor>(p, smA + stage * kABytes, smB + stage * kBBytes,
                                                                m_blk, n_blk, kb);
                            __syncwarp();
                        }
                    }
                    if (lane == 0) {
                        tc_fence_after();
                        const uint64_t adesc = umma_desc_sw128(smem_u32(smA + stage * kABytes), 16, 1024);
                        const uint64_t bdesc =
                            kBKMajor ? umma_desc_sw128(smem_u32(smB + stage * kBB), 16, 1024)
                                     : umma_desc_sw128(smem_u32(smB + stage * kBB), 8192, 1024);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            // K-major: +32 bytes per 16 elements inside the 128B swizzle row.
                            // N-major: +16 k-rows = 2 swizzle atoms = 2048 bytes.
                            const uint64_t a_off = uint64_t((k * 32) >> 4);
                            const uint64_t b_off = kBKMajor ? uint64_t((k * 32) >> 4) : uint64_t((k * 2048) >> 4);
                            if constexpr (kPair)
                                umma_f16_pair(d_tmem, adesc + a_off, bdesc + b_off, id, (kb > 0 || k > 0) ? 1u : 0u);
                            else
                                umma_f16(d_tmem, adesc + a_off, bdesc + b_off, id, (kb > 0 || k > 0) ? 1u : 0u);
                        }
                        // frees the stage in both CTAs of a pair
                        if constexpr (kPair) umma_commit_pair(smem_u32(&empty_bar[stage]), 0x3);
                        else umma_commit(smem_u32(&empty_bar[stage]));
                    }
                    if (++stage == kST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) {
                    if constexpr (kPair) umma_commit_pair(smem_u32(&tfull_bar[acc]), 0x3);
                    else umma_commit(smem_u32(&tfull_bar[acc]));
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
            if (p.epi.trace && lane == 0) p.epi.trace[blockIdx.x * 8 + 1] = gtime();
        }
    } else if (warp == kStatsProducerWarp) {
        if constexpr (kStats) {
            if (lane == 0) stats_producer(p, &tmA, smS, sfull_bar, sempty_bar);
        }
    } else if (warp >= 6) {
        if constexpr (kStats) {
            if (!VABFT_STATS_REMAP || warp != 9)
                stats_warps<kFmt>(p, smS, sfull_bar, sempty_bar, (VABFT_STATS_REMAP && warp == 10) ? 3 : warp - 6,
                                  lane);
        }
    } else {
        // ------------------------------------------------------- epilogue
        const int quad = warp & 3;  // TMEM lanes [32*quad, 32*quad+32) are addressable by this warp
        const int row_in_tile = quad * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = tile_first(p); u < p.num_units; u += tile_stride(p)) {
            int m_blk, n_blk, half;
            cta_unit(p, u, m_blk, n_blk, half);
            const int row = m_blk * kBM + row_in_tile;
            const bool row_ok = row < p.M;
            const int nw = half < 0 ? kBN : kBN / 2;
            const int n0 = n_blk * kBN + (half > 0 ? kBN / 2 : 0);

            int fcol = -1, fbit = 0, fdir = 0;
            if constexpr (kInject) {
                if (row_ok && p.epi.fault_target == 0) {
                    fcol = p.epi.fault_col[row];
                    if (fcol >= n0 && fcol < n0 + nw) {
                        fbit = p.epi.fault_bit[row];
                        fdir = p.epi.fault_dir[row];
                    } else {
                        fcol = -1;
                    }
                }
            }

            mbar_wait_sleep(smem_u32(&tfull_bar[acc]), acc_phase, 1000000u);
            tc_fence_after();

            float s1 = 0.0f, s2 = 0.0f;
#pragma unroll 1
            for (int c = 0; c < nw; c += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + (uint32_t(quad * 32) << 16) + uint32_t(acc * kBN + c), v);
                tmem_wait_ld();
                uint32_t packed[16];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int col = n0 + c + e;
                    float x = saturate_accum<kFmt>(__uint_as_float(v[e]));
                    uint16_t q;
                    if constexpr (kAbft == 2) {
                        q = quantize16_bits<kFmt>(x);
                        if constexpr (kInject) {
                            if (col == fcol) {
                                const bool ok = bit_eligible(q, fbit, fdir);
                                const uint16_t q2 = ok ? uint16_t(q ^ (1u << fbit)) : q;
                                if (p.epi.fault_records) {
                                    vabft_fault_record rr;
                                    rr.value_before = double(bits16_to_float<kFmt>(q));
                                    rr.value_after = double(bits16_to_float<kFmt>(q2));
                                    rr.applied = ok ? 1 : 0;
                                    rr.reserved = 0;
                                    p.epi.fault_records[row] = rr;
                                }
                                q = q2;
                            }
                        }
                        const float f = bits16_to_float<kFmt>(q);
                        if (col < p.N) {
                            // (s1, s2) += (f, (col + 1) f) as one FADD2 (scalar product, see sums)
                            const float2 sp =
                                __fadd2_rn(make_float2(s1, s2), make_float2(f, __fmul_rn(float(col + 1), f)));
                            s1 = sp.x;
                            s2 = sp.y;
                        }
                    } else {
                        if constexpr (kAbft == 1 && kInject) {
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
                        if constexpr (kAbft == 1) {
                            if (col < p.N) {
                                const float2 sp =
                                    __fadd2_rn(make_float2(s1, s2), make_float2(x, __fmul_rn(float(col + 1), x)));
                                s1 = sp.x;
                                s2 = sp.y;
                            }
                        }
                        q = quantize16_bits<kFmt>(x);
                    }
                    if (e & 1)
                        packed[e >> 1] |= uint32_t(q) << 16;
                    else
                        packed[e >> 1] = uint32_t(q);
                }
                if (p.epi.accum_out != nullptr && row_ok) {
                    // parity dump of the (saturated, post-injection) FP32 accumulator
                    float* dst = p.epi.accum_out + size_t(row) * p.N + n0 + c;
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        if (n0 + c + e < p.N) {
                            float x = saturate_accum<kFmt>(__uint_as_float(v[e]));
                            if constexpr (kAbft == 1 && kInject) {
                                if (n0 + c + e == fcol && bit_eligible(__float_as_uint(x), fbit, fdir))
                                    x = __uint_as_float(__float_as_uint(x) ^ (1u << fbit));
                            }
                            dst[e] = x;
                        }
                    }
                }
                if (row_ok) {
                    uint16_t* dst = p.C + size_t(row) * size_t(p.ldc) + n0 + c;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (n0 + c + g * 8 + 8 <= p.N) {
                            uint4 w = make_uint4(packed[4 * g], packed[4 * g + 1], packed[4 * g + 2],
                                                 packed[4 * g + 3]);
                            *reinterpret_cast<uint4*>(dst + g * 8) = w;
                        }
                    }
                }
                if constexpr (kAbft != 0) {
                    if ((c + 32) % 128 == 0) {
                        const int blk = (n0 + c) / 128;
                        if (row_ok && blk * 128 < p.N) {
                            const size_t o = part_index(blk, row, (p.N + 127) / 128);
                            p.epi.part1[o] = s1;
                            p.epi.part2[o] = s2;
                        }
                        s1 = 0.0f;
                        s2 = 0.0f;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                // pair: the leader's MMA waits for both CTAs' epilogues
                if (kPair && rank != 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
                else mbar_arrive(smem_u32(&tempty_bar[acc]));
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
            if constexpr (kStats) {
                if (p.epi.stream_verify && (int64_t(m_blk) * 4 + quad) * 32 < p.M)
                    final_arrive<kFmt>(p, int64_t(m_blk) * 4 + quad, unit_weight(half));
            }
        }
        if (p.epi.trace && lane == 0) atomicMax(p.epi.trace + blockIdx.x * 8 + 2, gtime());
    }

    if (p.epi.trace && threadIdx.x == 0) p.epi.trace[blockIdx.x * 8 + 4] = gtime();
    tc_fence_before();
    if constexpr (kPair) cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
    else __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        if constexpr (kPair) tmem_dealloc_pair(tmem_base, kTmemCols);
        else tmem_dealloc(tmem_base, kTmemCols);
    }
    if (p.epi.trace && threadIdx.x == 0) p.epi.trace[blockIdx.x * 8 + 5] = gtime();
    if constexpr (kStats) {
        // ---------------------------------------------- in-kernel verify tail
        // every tile's C partials and statistics partials are in global memory
        // once all CTAs pass the barrier; then all warps of the grid verify
        // 32-row groups (lane = row).
        if (p.epi.tail_phases) {
            unsigned int* gcount = p.epi.gbar;
            volatile unsigned int* ggen = p.epi.gbar + 1;
            grid_barrier(gcount, ggen);
            const int64_t ngroups = (int64_t(p.M) + 31) / 32;
            const int64_t g0 = int64_t(blockIdx.x) * kTailWarps + warp, gs = int64_t(gridDim.x) * kTailWarps;
            const bool tw = warp < kTailWarps;
            float* sbuf = reinterpret_cast<float*>(smem + size_t(warp) * kTailWarpSmem);
            const uint32_t tb = smem_u32(&tail_bar[tw ? warp : 0]);
            uint32_t tph = 0;
            if (p.epi.tail_phases == 3) {
                if (tw)
                    for (int64_t g = g0; g < ngroups; g += gs) verify_rowgroup<kFmt>(p.epi.tail, g, 3, sbuf, tb, tph);
            } else {
                if (tw)
                    for (int64_t g = g0; g < ngroups; g += gs) verify_rowgroup<kFmt>(p.epi.tail, g, 1, sbuf, tb, tph);
                grid_barrier(gcount, ggen);
                if (tw)
                    for (int64_t g = g0; g < ngroups; g += gs) verify_rowgroup<kFmt>(p.epi.tail, g, 2, sbuf, tb, tph);
            }
        }
    }
}

// ---------------------------------------------------------- host helpers
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    if (!fn) fail(VABFT_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2D row-major tensor [rows][cols] of 16-bit elements, row stride ld
// elements, box {box_cols, box_rows}.
CUtensorMap make_map_2d(int fmt, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                        uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt =
        fmt == VABFT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUresult r = get_encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(VABFT_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

template <int kFmt, bool kBKMajor, int kAbft, bool kInject, bool kStats = false, bool kPair = false>
void launch_inst(const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& p,
                 cudaStream_t stream) {
    auto kern = tc_gemm_kernel<kFmt, kBKMajor, kAbft, kInject, kStats, kPair>;
    constexpr size_t smem = kPair ? (kStats ? kSmemBytesPairStats : kSmemBytesPair)
                                  : (kStats ? kSmemBytesStats : kSmemBytes);
    constexpr unsigned threads = kStats ? kThreadsStats : kThreads;
    ensure_smem_attr(reinterpret_cast<const void*>(kern), int(smem));
    if constexpr (kPair) {
        // 2 x 1 clusters: the two CTAs of a pair share one TPC. A persistent
        // grid must fit in ONE wave: size it by the co-resident cluster count
        // (not every TPC can host a pair at one 227 KiB CTA per SM).
        cudaLaunchConfig_t cfg{};
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // per (kernel, device): a process may drive several GPUs
        const int max_clusters = cached_cluster_count(
            reinterpret_cast<const void*>(kern),
            [](const void* fn, void* ctx) {
                cudaLaunchConfig_t q = *static_cast<cudaLaunchConfig_t*>(ctx);
                q.gridDim = dim3(unsigned(sm_count() & ~1));
                int n = 0;
                check_cuda(cudaOccupancyMaxActiveClusters(&n, fn, &q), "cudaOccupancyMaxActiveClusters");
                return n > 0 ? n : 1;
            },
            &cfg);
        static const int cap_env = [] {
            const char* e = std::getenv("VABFT_MAX_PAIRS");  // developer cap (tools/l2_probe.py)
            return e ? std::atoi(e) : 0;
        }();
        const int avail = cap_env > 0 && cap_env < max_clusters ? cap_env : max_clusters;
        const int pairs = p.num_units < avail ? p.num_units : avail;
        cfg.gridDim = dim3(unsigned(2 * pairs));
        check_cuda(cudaLaunchKernelEx(&cfg, kern, ta, tb, p), "tc_gemm pair launch");
    } else {
        const int grid = p.num_units < sm_count() ? p.num_units : sm_count();
        if (kStats && p.epi.tail_phases) {
            // the in-kernel verify tail synchronizes the grid: cooperative launch
            // guarantees every CTA is co-resident (grid <= #SMs, 1 CTA/SM)
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(unsigned(grid));
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            check_cuda(cudaLaunchKernelEx(&cfg, kern, ta, tb, p), "tc_gemm cooperative launch");
        } else {
            kern<<<grid, threads, smem, stream>>>(ta, tb, p);
        }
    }
    check_cuda(cudaGetLastError(), "tc_gemm launch");
}

// pair-mode kernels exist for N-major B (with accumulator / output faults,
// not operand faults: tc_gemm_uses_pairs)
template <int kFmt, bool kBKMajor, int kAbft, bool kInject, bool kStats = false>
void launch_sel(const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& p, cudaStream_t stream) {
    if constexpr (!kBKMajor) {
        if (p.pair) {
            launch_inst<kFmt, kBKMajor, kAbft, kInject, kStats, true>(ta, tb, p, stream);
            return;
        }
    }
    if (p.pair) fail(VABFT_LOGIC_ERROR, "tc_gemm: no CTA-pair kernel for this configuration");
    launch_inst<kFmt, kBKMajor, kAbft, kInject, kStats, false>(ta, tb, p, stream);
}

template <int kFmt, bool kBKMajor>
void dispatch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& p,
                  cudaStream_t stream) {
    const bool inj = p.epi.fault_col != nullptr || (p.epi.fault_target == 2 && p.epi.n_operand_faults > 0);
    const bool st = p.epi.sp1 != nullptr && p.epi.debug != 3;  // 3: ablation, ABFT epilogue only
    switch (p.epi.abft) {
        case 0: launch_sel<kFmt, kBKMajor, 0, false>(ta, tb, p, stream); break;
        case 1:
            if (st) {
                if (inj) launch_sel<kFmt, kBKMajor, 1, true, true>(ta, tb, p, stream);
                else launch_sel<kFmt, kBKMajor, 1, false, true>(ta, tb, p, stream);
            } else {
                if (inj) launch_sel<kFmt, kBKMajor, 1, true>(ta, tb, p, stream);
                else launch_sel<kFmt, kBKMajor, 1, false>(ta, tb, p, stream);
            }
            break;
        default:
            if (st) {
                if (inj) launch_sel<kFmt, kBKMajor, 2, true, true>(ta, tb, p, stream);
                else launch_sel<kFmt, kBKMajor, 2, false, true>(ta, tb, p, stream);
            } else {
                if (inj) launch_sel<kFmt, kBKMajor, 2, true>(ta, tb, p, stream);
                else launch_sel<kFmt, kBKMajor, 2, false>(ta, tb, p, stream);
            }
            break;
    }
}

}  // namespace

bool tc_gemm_uses_pairs(bool b_kmajor, int64_t N, const TcEpilogue& epi) {
    static const int pair_env = [] {
        const char* e = std::getenv("VABFT_PAIR");  // developer override of the automatic choice
        return e ? std::atoi(e) : -1;
    }();
    // operand faults flip bits in one CTA's shared-memory tiles: one-CTA kernel
    const bool operand_inj = epi.fault_target != 0 && (epi.fault_col != nullptr || epi.n_operand_faults > 0);
    const bool eligible = !b_kmajor && !operand_inj && epi.tail_phases == 0 && sm_count() >= 2;
    const int mode = epi.cta_mode >= 0 ? epi.cta_mode : pair_env;
    (void)N;
    // automatic: CTA pairs whenever eligible — measured faster for the plain
    // and (with the fused kernel's raster of 32-row-block groups) the fused
    // kernel at every bench shape
    const bool want = mode >= 0 ? mode != 0 : true;
    return eligible && want;
}

bool tc_gemm_supported(int fmt, int64_t M, int64_t N, int64_t K) {
    if (fmt != VABFT_BF16 && fmt != VABFT_FP16) return false;
    if (M < 1 || N < 1 || K < 1) return false;
    if (N % 8 != 0 || K % 8 != 0) return false;  // 16-byte TMA global strides
    if (M > (int64_t(1) << 31) - 1 || N > (int64_t(1) << 24) || K > (int64_t(1) << 31) - 1) return false;
    return true;
}

void tc_gemm_launch(int fmt, bool b_kmajor, int64_t M, int64_t N, int64_t K, const void* A,
                    const void* B, void* C, const TcEpilogue& epi, cudaStream_t stream, int64_t lda, int64_t ldb,
                    int64_t ldc) {
    if (!tc_gemm_supported(fmt, M, N, K))
        fail(VABFT_UNSUPPORTED, "tcgen05 GEMM: needs BF16/FP16 with N % 8 == 0 and K % 8 == 0");
    const int64_t bcols = b_kmajor ? K : N;
    if (lda == 0) lda = K;
    if (ldb == 0) ldb = bcols;
    if (ldc == 0) ldc = N;
    if (lda < K || ldb < bcols || ldc < N || lda % 8 || ldb % 8 || ldc % 8)
        fail(VABFT_UNSUPPORTED, "tcgen05 GEMM: leading dimensions must cover the rows and be multiples of 8");
    TcParams p;
    p.M = int(M);
    p.N = int(N);
    p.K = int(K);
    p.num_m_blk = int((M + kBM - 1) / kBM);
    p.num_n_blk = int((N + kBN - 1) / kBN);
    p.num_k_blk = int((K + kBK - 1) / kBK);
    p.num_tiles = p.num_m_blk * p.num_n_blk;
    p.split_from = p.num_tiles;
    p.num_units = p.num_tiles;
    static const int raster_env = [] {
        const char* e = std::getenv("VABFT_RASTER_GROUP");  // developer override
        return e ? std::atoi(e) : 0;
    }();
    // measured (bench C2, interleaved A/B per group size): the plain kernel is
    // fastest with groups of 8 row blocks, the fused kernel (statistics warps)
    // with groups of 32 (+2-4 %: 1126-1178 vs 1077-1160 TFLOP/s)
    const int raster = raster_env ? raster_env : (epi.sp1 != nullptr ? 32 : 8);
    p.group_m = raster <= 0 || raster > p.num_m_blk ? p.num_m_blk : raster;
    p.C = static_cast<uint16_t*>(C);
    p.ldc = ldc;
    p.epi = epi;
    static unsigned long long* trace_buf = [] {
        unsigned long long* t = nullptr;
        if (std::getenv("VABFT_TRACE")) {  // developer timeline, see tools/trace_probe.py
            void* sym = nullptr;
            check_cuda(cudaGetSymbolAddress(&sym, g_trace), "trace symbol");
            t = static_cast<unsigned long long*>(sym);
        }
        return t;
    }();
    p.epi.trace = trace_buf;
    // CTA pairs (cta_group::2, 256 x 256 tiles over two SMs): N-major B, no
    // no operand faults, no grid-barrier tail. Policy (measured):
    // pairs whenever eligible, plain and fused (the fused kernel lost to the
    // one-CTA kernel at N = 4096 only with groups of 4 pair-row blocks; with
    // its 16-pair-block groups it wins at every bench shape).
    // VABFT_PAIR = 0 / 1 forces the 1-CTA / pair kernels.
    p.pair = tc_gemm_uses_pairs(b_kmajor, N, epi) ? 1 : 0;
    if (p.pair) {
        p.num_m_blk = int((M + 2 * kBM - 1) / (2 * kBM));
        p.num_tiles = p.num_m_blk * p.num_n_blk;
        const int g = raster / 2;
        p.group_m = g <= 0 || g > p.num_m_blk ? p.num_m_blk : g;
        // split the last wave's tiles into halves when it would leave more
        // than half the pairs idle (VABFT_SPLIT_LAST = 0 disables)
        static const bool split_env = [] {
            const char* e = std::getenv("VABFT_SPLIT_LAST");
            return !(e && std::atoi(e) == 0);
        }();
        const int pairs = sm_count() / 2;
        const int rem = p.num_tiles % pairs;
        p.split_from = p.num_tiles;
        if (split_env && p.num_tiles > pairs && rem > 0 && 2 * rem <= pairs && N > kBN / 2) p.split_from = p.num_tiles - rem;
        p.num_units = p.split_from + 2 * (p.num_tiles - p.split_from);
    }
    const CUtensorMap ta = make_map_2d(fmt, A, uint64_t(M), uint64_t(K), uint64_t(lda), kBK, kBM);
    const CUtensorMap tb = b_kmajor ? make_map_2d(fmt, B, uint64_t(N), uint64_t(K), uint64_t(ldb), kBK, kBN)
                                    : make_map_2d(fmt, B, uint64_t(K), uint64_t(N), uint64_t(ldb), 64, kBK);
    if (fmt == VABFT_BF16) {
        if (b_kmajor) dispatch_epi<VABFT_BF16, true>(ta, tb, p, stream);
        else dispatch_epi<VABFT_BF16, false>(ta, tb, p, stream);
    } else {
        if (b_kmajor) dispatch_epi<VABFT_FP16, true>(ta, tb, p, stream);
        else dispatch_epi<VABFT_FP16, false>(ta, tb, p, stream);
    }
}

}  // namespace vabft_dev

// developer timeline read-back (not part of the C-ABI header)
extern "C" int vabft_debug_tail(unsigned long long* out4, int reset) {
    if (cudaMemcpyFromSymbol(out4, vabft_dev::g_tail_dbg, sizeof(unsigned long long) * 4) != cudaSuccess) return 1;
    if (reset) {
        const unsigned long long z[4] = {0, 0, 0, 0};
        if (cudaMemcpyToSymbol(vabft_dev::g_tail_dbg, z, sizeof(z)) != cudaSuccess) return 1;
    }
    return 0;
}

extern "C" int vabft_debug_trace(unsigned long long* out, int n, int reset) {
    if (cudaMemcpyFromSymbol(out, vabft_dev::g_trace, sizeof(unsigned long long) * size_t(n)) != cudaSuccess) return 1;
    if (reset) {
        static unsigned long long zeros[1024 * 8] = {};
        if (cudaMemcpyToSymbol(vabft_dev::g_trace, zeros, sizeof(zeros)) != cudaSuccess) return 1;
    }
    return 0;
}
