/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the V-ABFT hot path.
 *
 * A plain-C restatement of the reference algorithm (arxiv/paper_2602_08043,
 * /root/reference/proj/src). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference arm may load it, and only as the
 * checker. Parity status: PINNED — tests/test_oracle_golden.py checks it
 * against the reference's own known-answer tests and against golden vectors
 * produced by the unmodified reference (oracle/_ref, tests/golden/).
 *
 * Matrices are row-major double arrays holding values on the format grid,
 * exactly like vabft::Matrix (proj/include/vabft/precision.hpp:94-131).
 * Return codes: 0 ok, 1 invalid_argument, 2 domain_error, 3 range_error,
 * 4 out_of_range, 5 logic_error.
 */
#ifndef VABFT_ORACLE_H_
#define VABFT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VO_BF16 = 0, VO_FP16 = 1, VO_FP32 = 2, VO_FP64 = 3 };
enum { VO_ACC_FP32_ROUND = 0, VO_ACC_SEQ = 1, VO_ACC_BLOCKED = 2, VO_ACC_PAIRWISE = 3 };
enum { VO_DIST_NORMAL = 0, VO_DIST_UNIFORM = 1, VO_DIST_TRUNCNORMAL = 2, VO_DIST_ABSNORMAL = 3 };

typedef struct vo_rng {
    uint64_t seed, stream, block_index;
    uint32_t buf[4];
    int pos;
} vo_rng;

const char* vo_last_error(void);

void vo_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void vo_rng_init(vo_rng* r, uint64_t seed, uint64_t stream);
uint32_t vo_next_u32(vo_rng* r);
uint64_t vo_next_u64(vo_rng* r);
double vo_next_double(vo_rng* r);
double vo_normal(vo_rng* r);
uint64_t vo_next_below(vo_rng* r, uint64_t n);
int vo_philox_draws(uint64_t seed, uint64_t stream, int kind, double arg, int64_t count,
                    double* out, uint64_t* out_u);
int vo_trial_inputs(int64_t m, int64_t k, int64_t n, int fmt, int dist_kind, double p0, double p1,
                    double lo, double hi, uint64_t seed, uint64_t stream, double* A, double* B);

int vo_quantize(double x, int fmt, int overflow_error, double* out);
int vo_gemm(int fmt, int accum_kind, int64_t block_len, int64_t m, int64_t k, int64_t n,
            const double* A, const double* B, double* C, double* C_accum);
int vo_encode_and_multiply(int fmt, int accum_kind, int64_t block_len, int mode, int64_t m,
                           int64_t k, int64_t n, const double* A, const double* B, double* C,
                           double* C_accum, double* rc1, double* rc2, double* cc1, double* cc2);
int vo_row_sums(int fmt, int mode, int accum_kind, int64_t block_len, int64_t m, int64_t n,
                const double* src, double* r1, double* r2);
int vo_row_stats(const double* v, int64_t n, double out[5]);
int vo_b_summary(int64_t k, int64_t n, const double* B, double summary[3]);
int vo_threshold_row(const double a_stats[4], const double b_summary[3], int64_t n, double e_max,
                     double c_sigma, double out[4]);
int vo_vabft_thresholds(int fmt, int64_t m, int64_t k, int64_t n, const double* A,
                        const double* B, double e_max, double c_sigma, double* T,
                        double* summary);
int vo_resolve_e_max(int fmt, int64_t dim, double* out);
int vo_aabft_sigma(int64_t n, int t, double y, double* out);
int vo_aabft_threshold(int fmt, int64_t m, int64_t k, int64_t n, const double* A, const double* B,
                       int mantissa_bits, double fixed_y, double conf, double* T, double* y_used,
                       int* degenerate);
int vo_localize(double d1, double d2, int64_t n_cols, int64_t* j, double* residual);
int vo_verify(int fmt, int mode, int accum_kind, int64_t block_len, int64_t m, int64_t n,
              const double* source, const double* rc1, const double* rc2, const double* T,
              double floor_scale, double* diff1, double* diff2, uint8_t* detected,
              int64_t* location, double* residual);
int vo_encode_bits(double v, int fmt, uint64_t* out);
int vo_decode_bits(uint64_t b, int fmt, double* out);
int vo_inject(int fmt, int src_fp32, int64_t m, int64_t n, double* X, int64_t pos_i, int64_t pos_j,
              int bit, int dir, uint64_t seed, uint64_t stream, int64_t* rec, double* vals);
int vo_campaign_trial(int64_t m, int64_t k, int64_t n, int fmt, int dist_kind, double p0,
                      double p1, double lo, double hi, int bit, int dir, uint64_t seed,
                      uint64_t trial, int mode, int method, double e_max, double c_sigma,
                      int64_t out[6]);

#ifdef __cplusplus
}
#endif

#endif
