/*
 * vabft_c.h — C-ABI of the B200-native V-ABFT fault-tolerant GEMM.
 *
 * This is the drop-in seam under the reference's C++ API (namespace vabft,
 * proj/include/vabft/*.hpp in arxiv/paper_2602_08043). Every entry point
 * names the reference interface it replaces. All matrix arguments are
 * caller-owned DEVICE pointers in native storage (BF16/FP16 as uint16
 * patterns, FP32 as float, FP64 as double), row-major, and every device
 * entry point is stream-ordered on the cudaStream_t passed as `stream`
 * (NULL = legacy default stream). Host-only helpers are marked [host].
 *
 * Errors: every function returns a vabft_status whose values map 1:1 to the
 * exception classes the reference throws (see vabft_status below);
 * vabft_last_error() returns the message of the calling thread's last error.
 * There is no CPU fallback: without a usable sm_100 device the device entry
 * points return VABFT_CUDA_ERROR.
 */
#ifndef VABFT_C_H_
#define VABFT_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VABFT_C_API_VERSION 3

/* Status codes <-> reference exception types (proj/src/*.cpp throw sites). */
typedef enum vabft_status {
    VABFT_OK = 0,
    VABFT_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    VABFT_DOMAIN_ERROR = 2,     /* std::domain_error     */
    VABFT_RANGE_ERROR = 3,      /* std::range_error      */
    VABFT_OUT_OF_RANGE = 4,     /* std::out_of_range     */
    VABFT_LOGIC_ERROR = 5,      /* std::logic_error      */
    VABFT_CUDA_ERROR = 6,       /* device / driver failure */
    VABFT_UNSUPPORTED = 7       /* shape or option outside a kernel's envelope */
} vabft_status;

/* vabft::Format (proj/include/vabft/precision.hpp:10) */
typedef enum vabft_format { VABFT_BF16 = 0, VABFT_FP16 = 1, VABFT_FP32 = 2, VABFT_FP64 = 3 } vabft_format;

/* vabft::AccumKind (precision.hpp:15-26) */
typedef enum vabft_accum_kind {
    VABFT_ACCUM_FP32_ROUND_OUTPUT = 0,
    VABFT_ACCUM_SEQUENTIAL = 1,
    VABFT_ACCUM_BLOCKED = 2,
    VABFT_ACCUM_PAIRWISE = 3
} vabft_accum_kind;

/* vabft::VerifyMode (proj/include/vabft/checksum.hpp:10) */
typedef enum vabft_verify_mode { VABFT_OFFLINE = 0, VABFT_ONLINE = 1 } vabft_verify_mode;

/* vabft::FlipDirection (proj/include/vabft/faults.hpp:17) */
typedef enum vabft_flip_direction {
    VABFT_FLIP = 0,
    VABFT_FLIP_SET0TO1 = 1,
    VABFT_FLIP_SET1TO0 = 2,
    VABFT_FLIP_ANY = 3
} vabft_flip_direction;

/* Which device GEMM engine computes C.
 *  EXACT  : order-exact SIMT kernels that reproduce gemm_emulated_with_accum
 *           (precision.cpp:222-338) bit for bit (no FMA, reference order).
 *  TENSOR : tcgen05/TMEM fused ABFT-GEMM (BF16/FP16 only); FP32 accumulation
 *           order is the tensor core's, checksums/row sums use blocked:128. */
typedef enum vabft_engine { VABFT_ENGINE_EXACT = 0, VABFT_ENGINE_TENSOR = 1 } vabft_engine;

/* vabft::AccumStrategy (precision.hpp:28-33) */
typedef struct vabft_accum {
    int32_t kind;      /* vabft_accum_kind */
    int32_t reserved;
    int64_t block_len; /* NativeBlocked only; <= 0 means 128 */
} vabft_accum;

/* vabft::PrecisionSpec (precision.hpp:54-85), flattened. */
typedef struct vabft_precision {
    int32_t format;        /* vabft_format */
    int32_t mantissa_bits; /* t incl. implicit bit */
    double unit_roundoff;  /* 2^-t */
    vabft_accum accumulation;
    int32_t emax_kind;     /* 0 = Constant, 1 = SqrtScaled (EmaxModel) */
    int32_t overflow;      /* 0 = Saturate, 1 = Error */
    double emax_scale;
    double emax_offset;
} vabft_precision;

/* Per-row verdict arrays (RowVerdict, proj/include/vabft/detect.hpp:14-23),
 * structure-of-arrays in device memory, each of length M. Any pointer may be
 * NULL to skip that output. location[i] = -1 when absent; correction is
 * diff1 whenever location >= 0 (detect.cpp:50). */
typedef struct vabft_verdicts {
    double* diff1;
    double* diff2;
    uint8_t* detected;
    int64_t* location;
    double* residual;
    double* row_check1; /* EncodedProduct::row_check1/2 (fused path only; may be NULL) */
    double* row_check2;
} vabft_verdicts;

/* Aggregate counters written by the verify tails (device, int64). Layout of
 * the `counts` array: [0] rows verified, [1] rows detected, [2] rows with a
 * location, [3] rows with NaN differences. */
#define VABFT_COUNT_ROWS 0
#define VABFT_COUNT_DETECTED 1
#define VABFT_COUNT_LOCATED 2
#define VABFT_COUNT_NAN 3
#define VABFT_COUNT_SLOW_STATS 4 /* rows whose A-row mean needed the sequential fallback */
#define VABFT_COUNT_CORRECTED 5  /* rows corrected in the kernel (vabft_fused_opts.correct) */
#define VABFT_NUM_COUNTS 6

/* One planned fault (InjectionRecord inputs, faults.hpp:21-35). */
typedef struct vabft_fault {
    int64_t i, j;
    int32_t bit;
    int32_t direction; /* vabft_flip_direction; ANY must be resolved by the caller */
} vabft_fault;

/* Outcome of one planned fault (InjectionRecord, faults.hpp:27-35). */
typedef struct vabft_fault_record {
    double value_before;
    double value_after;
    int32_t applied;
    int32_t reserved;
} vabft_fault_record;

/* ------------------------------------------------------------------ host */

/* [host] Last error message of the calling thread ("" if none). */
const char* vabft_last_error(void);
/* [host] VABFT_C_API_VERSION. */
int32_t vabft_api_version(void);
/* [host] PrecisionSpec::of (precision.cpp:84-92). */
vabft_status vabft_precision_default(int32_t format, vabft_precision* out);
/* [host] quantize (precision.cpp:129-159). */
vabft_status vabft_quantize(double x, const vabft_precision* fmt, double* out);
/* [host] resolve_e_max (threshold_vabft.cpp:49-52). */
vabft_status vabft_resolve_e_max(const vabft_precision* spec, int64_t dim, double* out);
/* [host] aabft_sigma (threshold_aabft.cpp:31-36). */
vabft_status vabft_aabft_sigma(int64_t n, int32_t mantissa_bits, double y, double* out);
/* [host] threshold_row over a BStatsSummary (threshold_vabft.cpp:28-42).
 * a_stats = {mean, max, min, var_bound}; b_summary = {sum_abs_mean,
 * sum_mean_sq, sum_var}; out = {det, var23, var4, total}. */
vabft_status vabft_threshold_row(const double a_stats[4], const double b_summary[3], int64_t n,
                                 double e_max, double c_sigma, double out[4]);
/* [host] localize (detect.cpp:9-17). Returns 1 with *j/*residual set when a
 * location exists, 0 otherwise. */
int32_t vabft_localize(double d1, double d2, int64_t n_cols, int64_t* j, double* residual);
/* [host] encode_bits / decode_bits (faults.cpp:66-87). */
vabft_status vabft_encode_bits(double value, int32_t format, uint64_t* out);
vabft_status vabft_decode_bits(uint64_t bits, int32_t format, double* out);

/* --------------------------------------------------------------- device */

/* Number of SMs and compute capability of the current device. */
vabft_status vabft_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* gemm_emulated_with_accum + encode_impl + quantize (precision.cpp:320-338,
 * checksum.cpp:103-158) — encode_and_multiply.
 *   A: M x K, B: K x N in `spec.format` native storage.
 *   C: M x N output format. C_accum: M x N FP32 (BF16/FP16/FP32) or FP64
 *   (FP64), may be NULL. row_check1/2: M doubles, col_check1/2: N doubles
 *   (either pair may be NULL).
 * engine EXACT reproduces the reference bit for bit; engine TENSOR requires
 * BF16/FP16 and uses the tcgen05 kernel (checksums blocked:128).
 * Workspace: vabft_encode_workspace_size bytes of device memory. */
vabft_status vabft_encode_workspace_size(int64_t m, int64_t n, int64_t k,
                                         const vabft_precision* spec, size_t* bytes);
vabft_status vabft_encode_and_multiply(const vabft_precision* spec, int32_t mode, int32_t engine,
                                       int64_t m, int64_t n, int64_t k, const void* A,
                                       const void* B, void* C, void* C_accum, double* row_check1,
                                       double* row_check2, double* col_check1,
                                       double* col_check2, void* workspace, size_t ws_bytes,
                                       void* stream);

/* row_sums (checksum.cpp:160-187): r1 = C r1, r2 = C r2 over rows of the
 * M x N source, accumulated in `sum_precision`'s arithmetic and order.
 * src_format is the storage format of `source` (FP32 for an FP32 accumulator). */
vabft_status vabft_row_sums(const vabft_precision* sum_precision, int32_t src_format, int64_t m,
                            int64_t n, const void* source, double* r1, double* r2, void* stream);

/* row_stats over every row of an R x L matrix (stats.cpp:9-32). Outputs are
 * device arrays of R doubles (any may be NULL). Non-finite input ->
 * VABFT_DOMAIN_ERROR (checked on the host after the stream syncs). */
vabft_status vabft_row_stats(int32_t format, int64_t rows, int64_t cols, const void* X,
                             double* mean, double* max, double* min, double* var_bound,
                             void* stream);

/* vabft_thresholds (threshold_vabft.cpp:54-61): T_i for every row of A
 * (n = N). Out: M doubles on device. Optional b_summary_out: 3 doubles on
 * device (BStatsSummary::from). Synchronizes `stream` to report errors. */
vabft_status vabft_vabft_thresholds(int32_t format, int64_t m, int64_t n, int64_t k, const void* A,
                                    const void* B, double e_max, double c_sigma, double* T,
                                    double* b_summary_out, void* stream);

/* Block-wise (tile-level) V-ABFT thresholds (PAPER.md "Integration with
 * Block-wise ABFT"): the composition of vabft_thresholds
 * (threshold_vabft.cpp:54-61) over slices, T[i][J] = sum over the k-tiles kt,
 * in order, of the V-ABFT threshold of row i of A[:, kt] against B[kt, J]
 * with n = |J| and e_max_per_tile[kt] (HOST array of ceil(K / tile_k)
 * values). T: device array M x ceil(N / tile_n), row-major. lda / ldb: row
 * strides in elements (0 = dense). Replaces the host loop over slice pairs
 * (paper_2602_08043_b200/blockwise.py) by three launches. Synchronizes
 * `stream` to report non-finite input (VABFT_DOMAIN_ERROR). */
vabft_status vabft_blockwise_thresholds(int32_t format, int64_t m, int64_t n, int64_t k, const void* A,
                                        int64_t lda, const void* B, int64_t ldb, int64_t tile_k,
                                        int64_t tile_n, const double* e_max_per_tile, double c_sigma,
                                        double* T, void* stream);

/* aabft_threshold (threshold_aabft.cpp:50-60): fills M doubles with the
 * row-independent bound confidence_multiplier * aabft_sigma(K, t, y);
 * *y_used / *degenerate (y == 0) are host outputs. fixed_y = NaN selects
 * computed y = max|A| * max_k |sum_j B[k][j]| (AabftParams::fixed_y empty);
 * any other value, zero and negative included, is used as the fixed y. */
vabft_status vabft_aabft_threshold(int32_t format, int64_t m, int64_t n, int64_t k, const void* A,
                                   const void* B, int32_t mantissa_bits, double fixed_y,
                                   double confidence_multiplier, double* T, double* y_used,
                                   int32_t* degenerate, void* stream);

/* verify (detect.cpp:19-55): row sums of `source` in checksum precision
 * `cs_prec`, D1/D2 against row_check1/2, strict `> T`, NaN always detected,
 * localization above floor_scale*T. counts (device int64[VABFT_NUM_COUNTS],
 * may be NULL) are accumulated, not overwritten. Synchronizes `stream` when
 * it validates thresholds (T >= 0, detect.cpp:24-27). */
vabft_status vabft_verify(const vabft_precision* cs_prec, int32_t src_format, int64_t m,
                          int64_t n, const void* source, const double* row_check1,
                          const double* row_check2, const double* T, double floor_scale,
                          vabft_verdicts verdicts, int64_t* counts, void* stream);

/* inject (faults.cpp:104-168) at fixed positions: flips/sets one bit of the
 * canonical encoding of element (i, j) of an M x N device matrix in
 * `format` storage, for each of `n_faults` host-side fault plans (applied in
 * order). records (host, may be NULL) receive the InjectionRecord fields. */
vabft_status vabft_inject(int32_t format, int64_t m, int64_t n, void* X, const vabft_fault* faults,
                          int64_t n_faults, vabft_fault_record* records, void* stream);

/* ------------------------------------------------ fused ABFT-GEMM (hot) */

/* Cached per-weight B-side state (B r1, B r2, B row-stat summary, A-ABFT
 * max_k|sum_j B|). Opaque device allocation owned by the handle. */
typedef struct vabft_bside* vabft_bside_t;

/* Build the B-side state for a K x N weight (precompute_b_stats +
 * BStatsSummary::from + encode's B r1/B r2, threshold_vabft.cpp:8-26,
 * checksum.cpp:110-115) with the checksum precision of `mode`. */
vabft_status vabft_bside_create(int32_t format, int32_t mode, int64_t k, int64_t n, const void* B,
                                vabft_bside_t* out, void* stream);
/* [v2] The same for a weight stored with row stride ldb >= n elements (0 = n;
 * BF16 / FP16, a multiple of 8), e.g. a column slice of a wider matrix. */
vabft_status vabft_bside_create_ld(int32_t format, int32_t mode, int64_t k, int64_t n, const void* B,
                                   int64_t ldb, vabft_bside_t* out, void* stream);
vabft_status vabft_bside_update(vabft_bside_t h, const void* B, void* stream);
vabft_status vabft_bside_destroy(vabft_bside_t h);

/* Options of one fused launch. */
typedef struct vabft_fused_opts {
    int32_t mode;              /* vabft_verify_mode */
    int32_t threshold_method;  /* 0 = V-ABFT, 1 = A-ABFT fixed y, 2 = A-ABFT computed y,
                                  3 = [v3] given thresholds t_in (e.g. vabft_blockwise_thresholds) */
    double e_max;              /* V-ABFT e_max (caller-resolved) */
    double c_sigma;            /* 2.5 */
    double floor_scale;        /* DetectOptions::localization_floor_scale, 1e-3 */
    int32_t aabft_mantissa_bits;
    int32_t b_kmajor;          /* 1: B is stored N x K (K-major, nn.Linear weight layout) */
    double aabft_fixed_y;
    double aabft_confidence;   /* 3.0 */
    /* Optional planned faults, one per row at most: device int32 arrays of
     * length M (fault_col[i] < 0 = none). Injected into the FP32 accumulator
     * (online) or the quantized output bits (offline) inside the epilogue. */
    const int32_t* fault_col;
    const int32_t* fault_bit;
    const int32_t* fault_dir;
    vabft_fault_record* fault_records; /* device, length M, may be NULL */
    /* Stage mask for profiling (0 = all): 1 statistics pass, 2 GEMM with the
     * ABFT epilogue, 4 verify tail; FP32 / FP64 handles: 8 with 2 runs the
     * same GEMM kernel with the ABFT epilogue off (overhead baseline). */
    int32_t stages;
    /* Where the planned faults land (FaultTarget, faults.hpp:15):
     *  0 OutputC: fault_col/bit/dir per row as above (accumulator online,
     *    output bits offline);
     *  1 InputA: fault_col[i] = k — bit fault_bit[i] of A[i][k] is flipped in
     *    the shared-memory operand tiles the tensor cores read (every N tile
     *    of row i), while the checksums and statistics use the clean A;
     *  2 InputB: operand_faults[t] = {i = k, j = column, bit, direction} —
     *    B[k][j] flipped in the operand tiles of every M tile; the checksums
     *    come from the clean B of the B-side handle.
     * Operand bits are the BF16/FP16 patterns (0..15); FP32 / FP64 handles
     * flip IEEE bits (0..31 / 0..63) in a copy of the operand the GEMM reads
     * (FP32: before its TF32 split). Records: fault_records per row for
     * InputA, operand_fault_records per fault for InputB. */
    int32_t fault_target;
    int32_t n_operand_faults;
    int32_t correct;  /* 1: rows with a located single error (residual < 0.5 - 0.1,
                         DetectOptions::residual_margin) get C[i][j] = quantize(C[i][j] - diff1)
                         in the kernel (correct, detect.cpp:57-64); counted in
                         counts[VABFT_COUNT_CORRECTED] */
    const vabft_fault* operand_faults;
    vabft_fault_record* operand_fault_records;
    /* tcgen05 kernel shape: -1 automatic (CTA pairs, cta_group::2 on 256 x 256
     * tiles over two SMs, whenever eligible: N-major B, no operand faults, no
     * grid-barrier tail; else one CTA per 128 x 256 tile), 0 one CTA, 1 CTA
     * pairs. */
    int32_t cta_mode;
    /* FP32 handles (tcgen05 kind::tf32): 0 or 3 = 3xTF32 error compensation
     * (FP32-level products), 1 = a single TF32 pass. Ignored otherwise. */
    int32_t tf32_passes;
    /* [v2] Parity dump (BF16/FP16 handles): an M x N FP32 device buffer that
     * receives the saturated, post-injection FP32 accumulator — the matrix
     * online verification reads (EncodedProduct::c_accum, checksum.hpp:45).
     * NULL = none. FP32 / FP64 handles: C itself is the accumulator. */
    float* accum_out;
    /* [v2] Workspace contract: the workspace passed to vabft_fused_gemm
     * carries per-row counters between launches. The library resets them when
     * the workspace was last used by another handle, another shape, a wide
     * (FP32 / FP64) launch or a stage-masked launch; a caller whose workspace
     * bytes were written by anything else since (pooled or freshly allocated
     * memory at a reused address) sets workspace_fresh = 1. */
    int32_t workspace_fresh;
    int32_t reserved_v2;
    /* [v2] Row strides in elements of A (M x K) and C (M x N); 0 = dense.
     * BF16 / FP16 handles: multiples of 8 (16-byte rows); FP32 / FP64: dense
     * only. With vabft_bside_create_ld a slice B[:, n0:n1] of a wider weight
     * and the matching C[:, n0:n1] run without copies (SURVEY §8(e) N-split). */
    int64_t lda;
    int64_t ldc;
    /* [v3] threshold_method 3: row i is verified against t_in[i * ldt]
     * (device doubles, >= 0 — verify's T >= 0 contract, detect.cpp:24-27, is
     * the caller's; ldt 0 = 1). With vabft_blockwise_thresholds and a column
     * slice of the weight (vabft_bside_create_ld) each tile_n-column block of
     * C is verified against its block-wise threshold in the fused kernel. */
    const double* t_in;
    int64_t ldt;
} vabft_fused_opts;

/* Workspace bytes for vabft_fused_gemm at this shape. */
vabft_status vabft_fused_workspace_size(int64_t m, int64_t n, int64_t k, size_t* bytes);

/* The hot path: stats of A (row stats + A (B r) checksums + thresholds),
 * the GEMM with the ABFT epilogue (row partials of the FP32 accumulator or
 * the quantized output), and the verify tail. BF16/FP16: one persistent
 * tcgen05 kernel; FP32: tcgen05 kind::tf32 (3xTF32) + side-stream A pass +
 * tail kernel; FP64: SIMT DFMA + side-stream A pass + tail kernel. Writes C
 * (M x N, format of the B-side handle), thresholds T (M doubles, may be
 * NULL), verdicts and accumulates counts. No host synchronization. */
vabft_status vabft_fused_gemm(const vabft_fused_opts* opts, vabft_bside_t bside, int64_t m,
                              const void* A, void* C, double* T, vabft_verdicts verdicts,
                              int64_t* counts, void* workspace, size_t ws_bytes, void* stream);

/* Plain GEMM with the ABFT epilogue compiled out (the overhead baseline):
 * C = A B — BF16/FP16 on tcgen05 with FP32 accumulation, FP32 on tcgen05
 * with 3xTF32 compensation (operands split into temporaries), FP64 on the
 * SIMT DFMA kernel. */
vabft_status vabft_gemm_plain(int32_t format, int32_t b_kmajor, int64_t m, int64_t n, int64_t k,
                              const void* A, const void* B, void* C, void* stream);
/* Same with an explicit kernel shape (cta_mode as in vabft_fused_opts; the
 * plain GEMM's automatic choice is CTA pairs whenever eligible). */
vabft_status vabft_gemm_plain_mode(int32_t format, int32_t b_kmajor, int64_t m, int64_t n, int64_t k,
                                   const void* A, const void* B, void* C, int32_t cta_mode, void* stream);
/* 1 if vabft_fused_gemm with these options and shape runs the CTA-pair
 * kernel, 0 if the one-CTA kernel. */
int32_t vabft_fused_uses_cta_pairs(const vabft_fused_opts* opts, int64_t m, int64_t n, int64_t k);

#ifdef __cplusplus
}
#endif

#endif /* VABFT_C_H_ */
