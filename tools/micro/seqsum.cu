// micro (negative result, DESIGN B-side): a warp-parallel exact reproduction of the sequential FP64 sum of
// non-negative terms (integer increments within a binade, events at binade crossings / ties) vs the
// sequential loop: bit-identical, but ~1.4-2x SLOWER (per-iteration latency of one warp: 32 iterations
// for 4096 terms at 1700-2500 cycles each vs 9.7 cycles per sequential add).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ int g_iters;
template <int kWhich>
__device__ __forceinline__ double chain_term(double x) {
    if constexpr (kWhich == 0) return fabs(x);
    else if constexpr (kWhich == 1) return __dmul_rn(x, x);
    else return x;
}

// The sequential FP64 sum acc = fl(acc + t_j), j = 0 .. n-1 (n <= 256), of
// non-negative terms t_j = chain_term(x[j]) (x in shared memory), by the whole
// warp, bit-identical to the sequential loop. While acc stays in one binade
// [2^e, 2^(e+1)) its quantum is ulp = 2^(e-52), so fl(acc + t) = acc +
// RN(t / ulp) ulp — independent of acc — except at an exact tie (t / ulp
// with fraction 1/2: the even neighbour depends on acc's last bit) or when
// the rounded sum leaves the binade. So the increments q_j = RN(t_j / ulp)
// are integers, their warp prefix sum commits every term up to the first
// such event exactly (acc = (M + Q_j) ulp, M = acc / ulp), the event term is
// added with one IEEE add, and the scan resumes in the new binade. Events:
// ~one per binade crossed (the partial sums grow monotonically: ~log2 K
// crossings) plus rare ties; acc zero, subnormal or non-finite takes plain
// sequential steps. Replaces K dependent FP64 adds (~8 cycles each: the
// B-side pass's latency floor) by ~K/256 warp scans.
template <int kWhich>
__device__ double warp_seq_sum_nonneg_impl(double acc, const double* x, int n) {
    const int lane = threadIdx.x & 31;
    constexpr long long kTop = 1ll << 53;
    int p = 0;  // terms [0, p) are in acc
    while (p < n) {
        if (threadIdx.x == 0) atomicAdd(&g_iters, 1);
        const long long ab = __double_as_longlong(acc);
        const int eb = int((ab >> 52) & 0x7FF);  // biased exponent of acc (acc >= +0)
        if (ab <= 0 || eb == 0 || eb >= 2046) {  // zero, subnormal, huge, non-finite: plain steps
            if (acc == 0.0) {
                int j = p;
                while (j < n && chain_term<kWhich>(x[j]) == 0.0) ++j;
                if (j == n) return acc;
                acc = chain_term<kWhich>(x[j]);
                p = j + 1;
            } else {
                acc = __dadd_rn(acc, chain_term<kWhich>(x[p]));
                ++p;
            }
            continue;
        }
        // acc = M 2^(eb - 1075), M in [2^52, 2^53); a term t = mt 2^(et - 1075)
        // (et >= 1) has t / ulp = mt 2^(et - eb): q = RN(mt >> (eb - et)),
        // integer ops only
        const long long M = (ab & ((1ll << 52) - 1)) | (1ll << 52);
        long long inc[8], q[8];
        bool ev[8];
        long long run = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = 8 * lane + u;
            const bool act = j >= p && j < n;
            const long long tb = act ? __double_as_longlong(chain_term<kWhich>(x[j])) : 0ll;
            const int et = int((tb >> 52) & 0x7FF);
            const long long mt = (tb & ((1ll << 52) - 1)) | (et ? (1ll << 52) : 0ll);
            const int sh = eb - (et ? et : 1);  // t / ulp = mt >> sh (sh < 0: t >= 2 ulp 2^52: event)
            long long qq = 0;
            bool tie = false;
            if (sh >= 64) {
                qq = 0;  // t < ulp / 2^11: rounds to 0, never a tie
            } else if (sh > 0) {
                const long long half = 1ll << (sh - 1);
                const long long rem = mt & ((1ll << sh) - 1);
                qq = (mt >> sh) + (rem > half ? 1 : 0);
                tie = rem == half;
            } else {
                qq = sh > -11 ? (mt << -sh) : kTop;  // >= 2^53 quanta: the binade is left anyway
            }
            q[u] = qq;
            ev[u] = act && (tie || et == 0x7FF);
            run += qq;
            inc[u] = run;
        }
        long long excl = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long o = __shfl_up_sync(0xffffffffu, excl, d);
            if (lane >= d) excl += o;
        }
        excl -= run;
        int first = 256;
#pragma unroll
        for (int u = 7; u >= 0; --u) {
            const int j = 8 * lane + u;
            const bool act = j >= p && j < n;
            if (act && (ev[u] || M + excl + inc[u] >= kTop)) first = j;
        }
        first = __reduce_min_sync(0xffffffffu, first);
        const long long ulpb = static_cast<long long>(eb - 52) << 52;  // ulp = 2^(eb - 1075)
        if (first >= n) {
            const long long tot = __shfl_sync(0xffffffffu, excl + run, 31);
            return __dmul_rn(static_cast<double>(M + tot), __longlong_as_double(ulpb));
        }
        long long before = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (8 * lane + u == first) before = excl + inc[u] - q[u];
        before = __shfl_sync(0xffffffffu, before, first >> 3);
        acc = __dadd_rn(__dmul_rn(static_cast<double>(M + before), __longlong_as_double(ulpb)),
                        chain_term<kWhich>(x[first]));
        p = first + 1;
    }
    return acc;
}

__global__ void run(const double* g, int n, double* out, long long* cyc) {
    __shared__ double x[4096];
    for (int i = threadIdx.x; i < n; i += 32) x[i] = g[i];
    __syncwarp();
    long long t0 = clock64();
    double acc = 0.0;
    for (int c = 0; c < n; c += 256) acc = warp_seq_sum_nonneg_impl<0>(acc, x + c, n - c < 256 ? n - c : 256);
    long long t1 = clock64();
    double ref = 0.0;
    if (threadIdx.x == 0) for (int i = 0; i < n; ++i) ref = __dadd_rn(ref, fabs(x[i]));
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = acc; out[1] = ref; cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
    const int n = 4096;
    double h[n];
    srand(1);
    for (int i = 0; i < n; ++i) { double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0);
        h[i] = sqrt(-2 * log(u)) * cos(6.283185307179586 * v) / 64.0; }
    double *g, *out; long long* cyc; cudaMalloc(&g, n * 8); cudaMallocManaged(&out, 16); cudaMallocManaged(&cyc, 16);
    cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice);
    int z = 0; cudaMemcpyToSymbol(g_iters, &z, 4);
    run<<<1, 32>>>(g, n, out, cyc); cudaDeviceSynchronize();
    int it; cudaMemcpyFromSymbol(&it, g_iters, 4);
    printf("par %.17g seq %.17g equal %d | cycles par %lld seq %lld | iterations %d | %s\n", out[0], out[1], out[0] == out[1],
           cyc[0], cyc[1], it, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
