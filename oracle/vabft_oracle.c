/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the V-ABFT hot path of
 * arxiv/paper_2602_08043 (reference sources under /root/reference/proj).
 * Used by tests/ and bench.py's cpu_baseline leg as the CHECKER; the product
 * (paper_2602_08043_b200) never loads it. Parity: pinned against the
 * reference's known-answer tests and golden vectors from the unmodified
 * reference (see vabft_oracle.h).
 *
 * Each function cites the reference lines it restates. Compiled with
 * -ffp-contract=off (proj/CMakeLists.txt:12-14): every float/double multiply
 * and add rounds separately.
 */
#include "vabft_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* vo_last_error(void) { return g_err; }

/* ------------------------------------------------------------ formats */
/* PrecisionSpec::bf16/fp16/fp32/fp64, min_normal_exponent, max_finite,
 * min_subnormal, bit_width — proj/src/precision.cpp:44-127 */
static int fmt_t(int f) { return f == VO_BF16 ? 8 : f == VO_FP16 ? 11 : f == VO_FP32 ? 24 : 53; }
static int fmt_emin(int f) { return f == VO_FP16 ? -14 : f == VO_FP64 ? -1022 : -126; }
static double fmt_max(int f) {
    switch (f) {
        case VO_BF16: return 0x1.FEp127;
        case VO_FP16: return 65504.0;
        case VO_FP32: return (double)3.40282346638528859812e+38F;
        default: return 1.7976931348623157e308;
    }
}
static double fmt_min_sub(int f) { return ldexp(1.0, fmt_emin(f) - fmt_t(f) + 1); }
static int fmt_bits(int f) { return f <= VO_FP16 ? 16 : f == VO_FP32 ? 32 : 64; }
static int fmt_ok(int f) { return f >= 0 && f <= 3; }
/* default accumulation kinds: 16-bit formats accumulate in FP32 and round
 * once; FP32/FP64 use the pairwise tree (precision.cpp:44-82) */
static int default_kind(int f) { return f <= VO_FP16 ? VO_ACC_FP32_ROUND : VO_ACC_PAIRWISE; }

static uint64_t dbits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static double bitsd(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }
static uint32_t fbits(float x) { uint32_t b; memcpy(&b, &x, 4); return b; }
static float bitsf(uint32_t b) { float x; memcpy(&x, &b, 4); return x; }

/* quantize — proj/src/precision.cpp:129-159. RNE on the FP64 pattern for
 * the normal range (add half-ulp-minus-one plus the kept lsb, truncate),
 * fixed-quantum nearbyint for the subnormal range, then the overflow policy. */
int vo_quantize(double x, int f, int overflow_error, double* out) {
    if (!isfinite(x)) return err(2, "quantize: non-finite input");
    if (f == VO_FP64 || x == 0.0) { *out = x; return 0; }
    const int t = fmt_t(f), emin = fmt_emin(f), drop = 53 - t;
    const uint64_t b = dbits(x);
    const int biased = (int)((b >> 52) & 0x7FF);
    double y;
    if (biased != 0 && biased - 1023 >= emin) {
        const uint64_t low = ((uint64_t)1 << drop) - 1;
        const uint64_t keep_lsb = (b >> drop) & 1u;
        y = bitsd((b + (low >> 1) + keep_lsb) & ~low);
    } else {
        const double q = fmt_min_sub(f);
        y = nearbyint(x / q) * q;
    }
    if (fabs(y) > fmt_max(f)) {
        if (overflow_error) return err(3, "quantize: overflow beyond max finite value");
        y = copysign(fmt_max(f), x);
    }
    *out = y;
    return 0;
}

static double q_or_die(double x, int f, int* rc) {
    double y = 0.0;
    int r = vo_quantize(x, f, 0, &y);
    if (r && !*rc) *rc = r;
    return y;
}

/* ---------------------------------------------------------- Philox RNG */
/* Philox4x32-10 — proj/src/rng.cpp:9-48 */
void vo_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t pa = (uint64_t)0xD2511F53u * c0;
        const uint64_t pb = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(pb >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)pb;
        const uint32_t n2 = (uint32_t)(pa >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)pa;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void vo_rng_init(vo_rng* r, uint64_t seed, uint64_t stream) {
    r->seed = seed; r->stream = stream; r->block_index = 0; r->pos = 4;
}

uint32_t vo_next_u32(vo_rng* r) {
    if (r->pos == 4) {
        const uint32_t ctr[4] = {(uint32_t)r->block_index, (uint32_t)(r->block_index >> 32),
                                 (uint32_t)r->stream, (uint32_t)(r->stream >> 32)};
        const uint32_t key[2] = {(uint32_t)r->seed, (uint32_t)(r->seed >> 32)};
        vo_philox_block(ctr, key, r->buf);
        r->block_index++;
        r->pos = 0;
    }
    return r->buf[r->pos++];
}

uint64_t vo_next_u64(vo_rng* r) {
    const uint64_t lo = vo_next_u32(r);
    const uint64_t hi = vo_next_u32(r);
    return (hi << 32) | lo;
}

double vo_next_double(vo_rng* r) { return (double)(vo_next_u64(r) >> 11) * 0x1.0p-53; }

/* Marsaglia-Tsang ziggurat, 128 layers — proj/src/rng.cpp:73-123 */
static struct { uint32_t kn[128]; double wn[128], fn[128]; int ready; } zig;

static void zig_init(void) {
    if (zig.ready) return;
    const double m1 = 2147483648.0, vn = 9.91256303526217e-3;
    double dn = 3.442619855899, tn = dn;
    const double q = vn / exp(-0.5 * dn * dn);
    zig.kn[0] = (uint32_t)((dn / q) * m1);
    zig.kn[1] = 0;
    zig.wn[0] = q / m1;
    zig.wn[127] = dn / m1;
    zig.fn[0] = 1.0;
    zig.fn[127] = exp(-0.5 * dn * dn);
    for (int i = 126; i >= 1; --i) {
        dn = sqrt(-2.0 * log(vn / dn + exp(-0.5 * dn * dn)));
        zig.kn[i + 1] = (uint32_t)((dn / tn) * m1);
        tn = dn;
        zig.fn[i] = exp(-0.5 * dn * dn);
        zig.wn[i] = dn / m1;
    }
    zig.ready = 1;
}

double vo_normal(vo_rng* r) {
    const double tail = 3.442619855899;
    zig_init();
    for (;;) {
        const int32_t hz = (int32_t)vo_next_u32(r);
        const int idx = hz & 127;
        const int64_t ahz = hz < 0 ? -(int64_t)hz : (int64_t)hz;
        if (ahz < (int64_t)zig.kn[idx]) return hz * zig.wn[idx];
        if (idx == 0) {
            for (;;) {
                const double u1 = (double)((vo_next_u64(r) >> 11) + 1) * 0x1.0p-53;
                const double u2 = (double)((vo_next_u64(r) >> 11) + 1) * 0x1.0p-53;
                const double x = -log(u1) / tail;
                const double y = -log(u2);
                if (y + y >= x * x) return hz > 0 ? tail + x : -(tail + x);
            }
        }
        const double x = hz * zig.wn[idx];
        if (zig.fn[idx] + vo_next_double(r) * (zig.fn[idx - 1] - zig.fn[idx]) < exp(-0.5 * x * x))
            return x;
    }
}

/* rejection-sampled unbiased integer — proj/src/rng.cpp:136-143 */
uint64_t vo_next_below(vo_rng* r, uint64_t n) {
    const uint64_t limit = n * (UINT64_MAX / n);
    for (;;) {
        const uint64_t v = vo_next_u64(r);
        if (v < limit) return v % n;
    }
}

int vo_philox_draws(uint64_t seed, uint64_t stream, int kind, double arg, int64_t count,
                    double* out, uint64_t* out_u) {
    vo_rng r;
    vo_rng_init(&r, seed, stream);
    for (int64_t i = 0; i < count; ++i) {
        switch (kind) {
            case 0: out_u[i] = vo_next_u32(&r); break;
            case 1: out_u[i] = vo_next_u64(&r); break;
            case 2: out[i] = vo_next_double(&r); break;
            case 3: out[i] = vo_normal(&r); break;
            default: out_u[i] = vo_next_below(&r, (uint64_t)arg); break;
        }
    }
    return 0;
}

/* Distribution::sample — proj/src/distribution.cpp:44-52 and the rng
 * helpers it calls (rng.cpp:57-59, 125-134) */
static double sample(vo_rng* r, int kind, double p0, double p1, double lo, double hi) {
    switch (kind) {
        case VO_DIST_NORMAL: return p0 + p1 * vo_normal(r);
        case VO_DIST_UNIFORM: return p0 + (p1 - p0) * vo_next_double(r);
        case VO_DIST_TRUNCNORMAL:
            for (;;) {
                const double z = p0 + p1 * vo_normal(r);
                if (z >= lo && z <= hi) return z;
            }
        default: return fabs(p0 + p1 * vo_normal(r));
    }
}

/* random_matrix — proj/src/distribution.cpp:95-101: row-major draws, each
 * quantized to the format */
static int random_matrix(vo_rng* r, int64_t rows, int64_t cols, int f, int kind, double p0,
                         double p1, double lo, double hi, double* out) {
    int rc = 0;
    for (int64_t i = 0; i < rows * cols; ++i) out[i] = q_or_die(sample(r, kind, p0, p1, lo, hi), f, &rc);
    return rc;
}

int vo_trial_inputs(int64_t m, int64_t k, int64_t n, int f, int dist_kind, double p0, double p1,
                    double lo, double hi, uint64_t seed, uint64_t stream, double* A, double* B) {
    vo_rng r;
    vo_rng_init(&r, seed, stream);
    int rc = random_matrix(&r, m, k, f, dist_kind, p0, p1, lo, hi, A);
    if (!rc && B) rc = random_matrix(&r, k, n, f, dist_kind, p0, p1, lo, hi, B);
    return rc;
}

/* ---------------------------------------------------------- reductions */
/* reduce_terms — proj/src/precision.cpp:344-381: sequential, blocked(bl)
 * or the balanced pairwise tree split at n/2 (n == 2 is a plain add). */
static float pairwise_f(const float* v, int64_t n) {
    if (n == 1) return v[0];
    if (n == 2) return v[0] + v[1];
    const int64_t h = n / 2;
    const float l = pairwise_f(v, h);
    const float rr = pairwise_f(v + h, n - h);
    return l + rr;
}
static double pairwise_d(const double* v, int64_t n) {
    if (n == 1) return v[0];
    if (n == 2) return v[0] + v[1];
    const int64_t h = n / 2;
    const double l = pairwise_d(v, h);
    const double rr = pairwise_d(v + h, n - h);
    return l + rr;
}
static float reduce_f(const float* v, int64_t n, int kind, int64_t bl) {
    if (n == 0) return 0.0f;
    if (kind == VO_ACC_PAIRWISE) return pairwise_f(v, n);
    if (kind == VO_ACC_BLOCKED) {
        if (bl <= 0) bl = 128;
        float tot = 0.0f, part = 0.0f;
        for (int64_t i = 0; i < n; ++i) {
            part += v[i];
            if ((i + 1) % bl == 0 || i + 1 == n) { tot += part; part = 0.0f; }
        }
        return tot;
    }
    float acc = 0.0f;
    for (int64_t i = 0; i < n; ++i) acc += v[i];
    return acc;
}
static double reduce_d(const double* v, int64_t n, int kind, int64_t bl) {
    if (n == 0) return 0.0;
    if (kind == VO_ACC_PAIRWISE) return pairwise_d(v, n);
    if (kind == VO_ACC_BLOCKED) {
        if (bl <= 0) bl = 128;
        double tot = 0.0, part = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            part += v[i];
            if ((i + 1) % bl == 0 || i + 1 == n) { tot += part; part = 0.0; }
        }
        return tot;
    }
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += v[i];
    return acc;
}

/* accumulates_in_float — proj/src/precision.cpp:203-206 */
static int in_float(int f, int kind) { return kind == VO_ACC_FP32_ROUND || f == VO_FP32; }

/* ---------------------------------------------------------------- GEMM */
/* Per output element: sequential / blocked / pairwise accumulation over k
 * in the working type — gemm_row_block and pairwise_block,
 * proj/src/precision.cpp:220-275 (the 128-column blocking there does not
 * change any element's arithmetic). */
static float dot_pairwise_f(const float* a, const float* b, int64_t n_cols, int64_t j,
                            int64_t k0, int64_t k1) {
    if (k1 - k0 == 1) return a[k0] * b[k0 * n_cols + j];
    const int64_t mid = k0 + (k1 - k0) / 2;
    const float l = dot_pairwise_f(a, b, n_cols, j, k0, mid);
    const float r = dot_pairwise_f(a, b, n_cols, j, mid, k1);
    return l + r;
}
static double dot_pairwise_d(const double* a, const double* b, int64_t n_cols, int64_t j,
                             int64_t k0, int64_t k1) {
    if (k1 - k0 == 1) return a[k0] * b[k0 * n_cols + j];
    const int64_t mid = k0 + (k1 - k0) / 2;
    const double l = dot_pairwise_d(a, b, n_cols, j, k0, mid);
    const double r = dot_pairwise_d(a, b, n_cols, j, mid, k1);
    return l + r;
}

/* gemm_emulated_with_accum / run_gemm — proj/src/precision.cpp:285-338 */
int vo_gemm(int f, int kind, int64_t bl, int64_t m, int64_t k, int64_t n, const double* A,
            const double* B, double* C, double* C_accum) {
    if (!fmt_ok(f)) return err(1, "bad format");
    if (kind < 0) kind = default_kind(f);
    if ((f == VO_BF16 || f == VO_FP16) && kind != VO_ACC_FP32_ROUND)
        return err(1, "gemm_emulated: 16-bit formats require fp32 accumulation");
    if (bl <= 0) bl = 128;
    const int flt = in_float(f, kind);
    const int acc_fmt = flt ? VO_FP32 : VO_FP64;
    const int needs_round = f != acc_fmt;
    int rc = 0;
    if (flt) {
        float* a = malloc(sizeof(float) * (size_t)(m * k));
        float* b = malloc(sizeof(float) * (size_t)(k * n));
        float* row = malloc(sizeof(float) * (size_t)n);
        float* part = malloc(sizeof(float) * (size_t)n);
        for (int64_t i = 0; i < m * k; ++i) a[i] = (float)A[i];
        for (int64_t i = 0; i < k * n; ++i) b[i] = (float)B[i];
        for (int64_t i = 0; i < m && !rc; ++i) {
            const float* ar = a + i * k;
            if (kind == VO_ACC_PAIRWISE) {
                for (int64_t j = 0; j < n; ++j) row[j] = dot_pairwise_f(ar, b, n, j, 0, k);
            } else if (kind == VO_ACC_BLOCKED) {
                for (int64_t j = 0; j < n; ++j) { row[j] = 0.0f; part[j] = 0.0f; }
                for (int64_t kk = 0; kk < k; ++kk) {
                    for (int64_t j = 0; j < n; ++j) part[j] += ar[kk] * b[kk * n + j];
                    if ((kk + 1) % bl == 0 || kk + 1 == k)
                        for (int64_t j = 0; j < n; ++j) { row[j] += part[j]; part[j] = 0.0f; }
                }
            } else {
                for (int64_t j = 0; j < n; ++j) row[j] = 0.0f;
                for (int64_t kk = 0; kk < k; ++kk) {
                    const float av = ar[kk];
                    const float* br = b + kk * n;
                    for (int64_t j = 0; j < n; ++j) row[j] += av * br[j];
                }
            }
            for (int64_t j = 0; j < n; ++j) {
                const double acc = (double)row[j];
                double cv, av;
                if (!isfinite(acc)) {
                    cv = av = copysign(fmt_max(f), acc);
                } else {
                    av = acc;
                    cv = needs_round ? q_or_die(acc, f, &rc) : acc;
                }
                if (C_accum) C_accum[i * n + j] = av;
                if (C) C[i * n + j] = cv;
            }
        }
        free(a); free(b); free(row); free(part);
    } else {
        double* row = malloc(sizeof(double) * (size_t)n);
        double* part = malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < m; ++i) {
            const double* ar = A + i * k;
            if (kind == VO_ACC_PAIRWISE) {
                for (int64_t j = 0; j < n; ++j) row[j] = dot_pairwise_d(ar, B, n, j, 0, k);
            } else if (kind == VO_ACC_BLOCKED) {
                for (int64_t j = 0; j < n; ++j) { row[j] = 0.0; part[j] = 0.0; }
                for (int64_t kk = 0; kk < k; ++kk) {
                    for (int64_t j = 0; j < n; ++j) part[j] += ar[kk] * B[kk * n + j];
                    if ((kk + 1) % bl == 0 || kk + 1 == k)
                        for (int64_t j = 0; j < n; ++j) { row[j] += part[j]; part[j] = 0.0; }
                }
            } else {
                for (int64_t j = 0; j < n; ++j) row[j] = 0.0;
                for (int64_t kk = 0; kk < k; ++kk)
                    for (int64_t j = 0; j < n; ++j) row[j] += ar[kk] * B[kk * n + j];
            }
            for (int64_t j = 0; j < n; ++j) {
                const double acc = row[j];
                const double v = isfinite(acc) ? acc : copysign(fmt_max(f), acc);
                if (C_accum) C_accum[i * n + j] = v;
                if (C) C[i * n + j] = v;
            }
        }
        free(row); free(part);
    }
    return rc;
}

/* ------------------------------------------------------------ checksums */
/* checksum_precision_for — proj/src/checksum.cpp:18-24: offline keeps the
 * input spec; online moves to FP32 (FP64 for FP64) keeping the strategy. */
static void cs_prec(int f, int mode, int kind, int* cs_fmt, int* cs_kind) {
    *cs_kind = kind;
    *cs_fmt = mode == 0 ? f : (f == VO_FP64 ? VO_FP64 : VO_FP32);
}

/* ChecksumVectors::make weight-range check — proj/src/checksum.cpp:26-34 */
static int weights_ok(int64_t n, int cs_fmt, int cs_kind) {
    if (n < 1) return err(1, "ChecksumVectors: length must be >= 1");
    const int t = in_float(cs_fmt, cs_kind) ? 24 : 53;
    if (n > ((int64_t)1 << t)) return err(1, "ChecksumVectors: weights exceed exact range");
    return 0;
}

/* ChecksumEngine::plain / position_weighted / contract and encode_impl —
 * proj/src/checksum.cpp:50-146. `lhs == NULL` gives plain/weighted sums. */
static void cs_reduce(int flt, int kind, int64_t bl, const double* mat, int64_t rows, int64_t cols,
                      int over_cols, const double* lhs, int weighted, double* out) {
    const int64_t out_len = over_cols ? rows : cols;
    const int64_t k_len = over_cols ? cols : rows;
    if (flt) {
        float* t = malloc(sizeof(float) * (size_t)k_len);
        for (int64_t i = 0; i < out_len; ++i) {
            for (int64_t q = 0; q < k_len; ++q) {
                const float mv = (float)(over_cols ? mat[i * cols + q] : mat[q * cols + i]);
                if (lhs) t[q] = (float)lhs[q] * mv;
                else t[q] = weighted ? (float)(q + 1) * mv : mv;
            }
            out[i] = (double)reduce_f(t, k_len, kind, bl);
        }
        free(t);
    } else {
        double* t = malloc(sizeof(double) * (size_t)k_len);
        for (int64_t i = 0; i < out_len; ++i) {
            for (int64_t q = 0; q < k_len; ++q) {
                const double mv = over_cols ? mat[i * cols + q] : mat[q * cols + i];
                if (lhs) t[q] = lhs[q] * mv;
                else t[q] = weighted ? (double)(q + 1) * mv : mv;
            }
            out[i] = reduce_d(t, k_len, kind, bl);
        }
        free(t);
    }
}

/* encode_and_multiply — proj/src/checksum.cpp:150-158 */
int vo_encode_and_multiply(int f, int kind, int64_t bl, int mode, int64_t m, int64_t k, int64_t n,
                           const double* A, const double* B, double* C, double* C_accum,
                           double* rc1, double* rc2, double* cc1, double* cc2) {
    if (kind < 0) kind = default_kind(f);
    int rc = vo_gemm(f, kind, bl, m, k, n, A, B, C, C_accum);
    if (rc) return rc;
    int csf, csk;
    cs_prec(f, mode, kind, &csf, &csk);
    if ((rc = weights_ok(n, csf, csk)) || (rc = weights_ok(m, csf, csk))) return rc;
    const int flt = in_float(csf, csk);
    const int round = mode == 0;
    double* br1 = malloc(sizeof(double) * (size_t)k);
    double* br2 = malloc(sizeof(double) * (size_t)k);
    double* ac1 = malloc(sizeof(double) * (size_t)k);
    double* ac2 = malloc(sizeof(double) * (size_t)k);
    double* t1 = malloc(sizeof(double) * (size_t)(m > n ? m : n));
    /* row checksums: B r first, then A (B r) */
    cs_reduce(flt, csk, bl, B, k, n, 1, NULL, 0, br1);
    cs_reduce(flt, csk, bl, B, k, n, 1, NULL, 1, br2);
    if (round) for (int64_t q = 0; q < k; ++q) { br1[q] = q_or_die(br1[q], f, &rc); br2[q] = q_or_die(br2[q], f, &rc); }
    if (rc1) { cs_reduce(flt, csk, bl, A, m, k, 1, br1, 0, rc1); if (round) for (int64_t i = 0; i < m; ++i) rc1[i] = q_or_die(rc1[i], f, &rc); }
    if (rc2) { cs_reduce(flt, csk, bl, A, m, k, 1, br2, 0, rc2); if (round) for (int64_t i = 0; i < m; ++i) rc2[i] = q_or_die(rc2[i], f, &rc); }
    /* column checksums: c A first, then (c A) B */
    cs_reduce(flt, csk, bl, A, m, k, 0, NULL, 0, ac1);
    cs_reduce(flt, csk, bl, A, m, k, 0, NULL, 1, ac2);
    if (round) for (int64_t q = 0; q < k; ++q) { ac1[q] = q_or_die(ac1[q], f, &rc); ac2[q] = q_or_die(ac2[q], f, &rc); }
    if (cc1) { cs_reduce(flt, csk, bl, B, k, n, 0, ac1, 0, cc1); if (round) for (int64_t j = 0; j < n; ++j) cc1[j] = q_or_die(cc1[j], f, &rc); }
    if (cc2) { cs_reduce(flt, csk, bl, B, k, n, 0, ac2, 0, cc2); if (round) for (int64_t j = 0; j < n; ++j) cc2[j] = q_or_die(cc2[j], f, &rc); }
    free(br1); free(br2); free(ac1); free(ac2); free(t1);
    return rc;
}

/* row_sums — proj/src/checksum.cpp:160-187 */
int vo_row_sums(int f, int mode, int kind, int64_t bl, int64_t m, int64_t n, const double* src,
                double* r1, double* r2) {
    int csf, csk;
    cs_prec(f, mode, kind >= 0 ? kind : default_kind(f), &csf, &csk);
    int rc = weights_ok(n, csf, csk);
    if (rc) return rc;
    const int flt = in_float(csf, csk);
    cs_reduce(flt, csk, bl, src, m, n, 1, NULL, 0, r1);
    cs_reduce(flt, csk, bl, src, m, n, 1, NULL, 1, r2);
    return 0;
}

/* ---------------------------------------------------------- statistics */
/* row_stats — proj/src/stats.cpp:9-32: Neumaier-compensated FP64 mean,
 * max, min; mean clamped into [min, max]; var_bound = (max-mean)(mean-min). */
int vo_row_stats(const double* v, int64_t n, double out[5]) {
    if (n < 1) return err(1, "row_stats: empty row");
    double sum = 0.0, comp = 0.0, mx = v[0], mn = v[0];
    for (int64_t i = 0; i < n; ++i) {
        const double x = v[i];
        if (!isfinite(x)) return err(2, "row_stats: non-finite value");
        const double t = sum + x;
        if (fabs(sum) >= fabs(x)) comp += (sum - t) + x;
        else comp += (x - t) + sum;
        sum = t;
        if (mx < x) mx = x;
        if (x < mn) mn = x;
    }
    double mean = (sum + comp) / (double)n;
    if (mean < mn) mean = mn;
    else if (mx < mean) mean = mx;
    const double vb = (mx - mean) * (mean - mn);
    out[0] = mean; out[1] = mx; out[2] = mn; out[3] = vb > 0.0 ? vb : 0.0; out[4] = (double)n;
    return 0;
}

/* precompute_b_stats + BStatsSummary::from — threshold_vabft.cpp:8-26 */
int vo_b_summary(int64_t k, int64_t n, const double* B, double s[3]) {
    if (k < 1) return err(1, "BStatsSummary: empty stats");
    s[0] = s[1] = s[2] = 0.0;
    for (int64_t q = 0; q < k; ++q) {
        double st[5];
        int rc = vo_row_stats(B + q * n, n, st);
        if (rc) return rc;
        if (st[3] < 0.0) return err(5, "BStatsSummary: negative variance bound");
        s[0] += fabs(st[0]);
        s[1] += st[0] * st[0];
        s[2] += st[3];
    }
    return 0;
}

/* threshold_row — proj/src/threshold_vabft.cpp:28-42, evaluated in the
 * written order (det, var23, var4, e_max * sum). */
int vo_threshold_row(const double a[4], const double b[3], int64_t n, double e_max,
                     double c_sigma, double out[4]) {
    if (n < 1) return err(1, "threshold_row: n must be >= 1");
    const double nn = (double)n, mu = a[0], sa = sqrt(a[3]);
    const double det = nn * fabs(mu) * b[0];
    const double var23 = c_sigma * sqrt(nn * mu * mu * b[2] + nn * nn * a[3] * b[1]);
    const double var4 = c_sigma * sqrt(nn) * sa * sqrt(b[2]);
    out[0] = det; out[1] = var23; out[2] = var4; out[3] = e_max * (det + var23 + var4);
    return 0;
}

/* vabft_thresholds — proj/src/threshold_vabft.cpp:54-61 (n = N) */
int vo_vabft_thresholds(int f, int64_t m, int64_t k, int64_t n, const double* A, const double* B,
                        double e_max, double c_sigma, double* T, double* summary) {
    (void)f;
    double s[3];
    int rc = vo_b_summary(k, n, B, s);
    if (rc) return rc;
    if (summary) memcpy(summary, s, sizeof s);
    for (int64_t i = 0; i < m; ++i) {
        double st[5], out[4];
        if ((rc = vo_row_stats(A + i * k, k, st))) return rc;
        if ((rc = vo_threshold_row(st, s, n, e_max, c_sigma, out))) return rc;
        T[i] = out[3];
    }
    return 0;
}

/* resolve_e_max with the format default EmaxModel — precision.cpp:39-82,
 * threshold_vabft.cpp:49-52 */
int vo_resolve_e_max(int f, int64_t dim, double* out) {
    if (dim < 1) return err(1, "resolve_e_max: dim must be >= 1");
    switch (f) {
        case VO_BF16: *out = 8e-3; break;
        case VO_FP16: *out = 1e-3; break;
        case VO_FP32: *out = 5.0e-9 * sqrt((double)dim) + 1.2e-7; break;
        default: *out = 1.0e-17 * sqrt((double)dim) + 2.5e-16; break;
    }
    return 0;
}

/* aabft_sigma — proj/src/threshold_aabft.cpp:31-36 */
int vo_aabft_sigma(int64_t n, int t, double y, double* out) {
    if (n < 1) return err(1, "aabft_sigma: n must be >= 1");
    const double nn = (double)n;
    const double poly = nn * (nn + 1.0) * (nn + 0.5) + 2.0 * nn;
    *out = sqrt(poly / 24.0) * ldexp(1.0, -t) * y;
    return 0;
}

/* aabft_threshold / aabft_computed_y / AabftParams::for_format —
 * proj/src/threshold_aabft.cpp:8-60. fixed_y NaN selects computed y;
 * mantissa_bits < 0 takes the format default (53/23/8/11). */
int vo_aabft_threshold(int f, int64_t m, int64_t k, int64_t n, const double* A, const double* B,
                       int t, double fixed_y, double conf, double* T, double* y_used,
                       int* degenerate) {
    if (t < 0) t = f == VO_FP64 ? 53 : f == VO_FP32 ? 23 : f == VO_BF16 ? 8 : 11;
    if (conf <= 0) conf = 3.0;
    double y = fixed_y;
    if (isnan(fixed_y)) {
        double max_a = 0.0, max_rs = 0.0;
        for (int64_t i = 0; i < m * k; ++i) { const double a = fabs(A[i]); if (max_a < a) max_a = a; }
        for (int64_t q = 0; q < k; ++q) {
            double s = 0.0;
            for (int64_t j = 0; j < n; ++j) s += B[q * n + j];
            if (max_rs < fabs(s)) max_rs = fabs(s);
        }
        y = max_a * max_rs;
    }
    double sig;
    int rc = vo_aabft_sigma(k, t, y, &sig);
    if (rc) return rc;
    for (int64_t i = 0; i < m; ++i) T[i] = conf * sig;
    *y_used = y;
    *degenerate = y == 0.0;
    return 0;
}

/* ---------------------------------------------------------------- verify */
/* localize — proj/src/detect.cpp:9-17. The int64 conversion of an
 * out-of-range `nearest` follows x86-64 cvttsd2si (INT64_MIN), which is
 * what the reference binary does. */
int vo_localize(double d1, double d2, int64_t n_cols, int64_t* j, double* residual) {
    if (d1 == 0.0 || !isfinite(d1) || !isfinite(d2)) return 0;
    const double pos = d2 / d1 - 1.0;
    if (!isfinite(pos)) return 0;
    const double nearest = nearbyint(pos);
    *residual = fabs(pos - nearest);
    int64_t q = (nearest >= 0x1.0p63 || nearest < -0x1.0p63) ? INT64_MIN : (int64_t)nearest;
    if (q < 0) q = 0;
    if (q > n_cols - 1) q = n_cols - 1;
    *j = q;
    return 1;
}

/* verify — proj/src/detect.cpp:19-55 */
int vo_verify(int f, int mode, int kind, int64_t bl, int64_t m, int64_t n, const double* source,
              const double* rc1, const double* rc2, const double* T, double floor_scale,
              double* diff1, double* diff2, uint8_t* detected, int64_t* location,
              double* residual) {
    for (int64_t i = 0; i < m; ++i)
        if (!(T[i] >= 0.0)) return err(1, "verify: thresholds must be >= 0");
    double* r1 = malloc(sizeof(double) * (size_t)m);
    double* r2 = malloc(sizeof(double) * (size_t)m);
    int rc = vo_row_sums(f, mode, kind, bl, m, n, source, r1, r2);
    if (rc) { free(r1); free(r2); return rc; }
    for (int64_t i = 0; i < m; ++i) {
        const double d1 = r1[i] - rc1[i], d2 = r2[i] - rc2[i];
        int det = 0;
        int64_t loc = -1;
        double res = 0.0;
        if (isnan(d1) || isnan(d2)) {
            det = 1;
        } else {
            det = fabs(d1) > T[i];
            if (det && fabs(d1) > floor_scale * T[i]) {
                int64_t j;
                double rr;
                if (vo_localize(d1, d2, n, &j, &rr)) { loc = j; res = rr; }
            }
        }
        if (diff1) diff1[i] = d1;
        if (diff2) diff2[i] = d2;
        if (detected) detected[i] = (uint8_t)det;
        if (location) location[i] = loc;
        if (residual) residual[i] = res;
    }
    free(r1); free(r2);
    return 0;
}

/* --------------------------------------------------------------- faults */
/* f16_encode / f16_decode — proj/src/faults.cpp:25-62 */
static uint16_t f16_encode(double v) {
    if (isnan(v)) {
        const uint64_t b = dbits(v);
        uint16_t m = (uint16_t)((b >> 42) & 0x3FF);
        if (m == 0) m = 0x200;
        return (uint16_t)(((b >> 48) & 0x8000) | 0x7C00 | m);
    }
    const uint16_t sign = signbit(v) ? 0x8000 : 0;
    if (isinf(v)) return sign | 0x7C00;
    const double a = fabs(v);
    if (a == 0.0) return sign;
    const int e = ilogb(a);
    if (e < -14) return (uint16_t)(sign | (uint16_t)llrint(ldexp(a, 24)));
    if (e > 15) return sign | 0x7C00;
    const uint16_t mant = (uint16_t)llrint((ldexp(a, -e) - 1.0) * 1024.0);
    return (uint16_t)(sign | (uint16_t)((e + 15) << 10) | mant);
}
static double f16_decode(uint16_t bits) {
    const int neg = (bits & 0x8000) != 0;
    const int e = (bits >> 10) & 0x1F;
    const uint16_t m = bits & 0x3FF;
    double v;
    if (e == 31) {
        if (m == 0) v = INFINITY;
        else return bitsd(0x7FF0000000000000ull | ((uint64_t)neg << 63) | ((uint64_t)m << 42));
    } else if (e == 0) {
        v = ldexp((double)m, -24);
    } else {
        v = ldexp(1.0 + (double)m / 1024.0, e - 15);
    }
    return neg ? -v : v;
}

/* encode_bits / decode_bits — proj/src/faults.cpp:66-87 (BF16 goes through
 * float, which quiets signalling NaNs — the reference's own behaviour) */
int vo_encode_bits(double v, int f, uint64_t* out) {
    switch (f) {
        case VO_BF16: *out = fbits((float)v) >> 16; return 0;
        case VO_FP16: *out = f16_encode(v); return 0;
        case VO_FP32: *out = fbits((float)v); return 0;
        case VO_FP64: *out = dbits(v); return 0;
    }
    return err(1, "encode_bits: bad format");
}
int vo_decode_bits(uint64_t b, int f, double* out) {
    switch (f) {
        case VO_BF16: *out = (double)bitsf((uint32_t)b << 16); return 0;
        case VO_FP16: *out = f16_decode((uint16_t)b); return 0;
        case VO_FP32: *out = (double)bitsf((uint32_t)b); return 0;
        case VO_FP64: *out = bitsd(b); return 0;
    }
    return err(1, "decode_bits: bad format");
}

static int eligible(uint64_t bits, int bit, int dir) {
    const uint64_t b = (bits >> bit) & 1u;
    if (dir == 1) return b == 0;
    if (dir == 2) return b == 1;
    return 1;
}

static int inject_rng(int f, int64_t m, int64_t n, double* X, int64_t pi0, int64_t pj0, int bit,
                      int dir, vo_rng* r, int64_t* rec, double* vals) {
    if (bit < 0 || bit >= fmt_bits(f)) return err(4, "inject: bit index outside the format's width");
    if (dir == 3) dir = (vo_next_u32(r) & 1) ? 1 : 2;
    rec[0] = -1; rec[1] = -1; rec[2] = 0; rec[3] = dir;
    vals[0] = vals[1] = 0.0;
    int64_t i = -1, j = -1;
    uint64_t bits;
    if (pi0 >= 0) {
        i = pi0; j = pj0;
        if (i >= m || j < 0 || j >= n) return err(4, "inject: position out of range");
        vo_encode_bits(X[i * n + j], f, &bits);
        if (!eligible(bits, bit, dir)) {
            rec[0] = i; rec[1] = j;
            vals[0] = vals[1] = X[i * n + j];
            return 0;
        }
    } else {
        const int64_t total = m * n;
        int found = 0;
        for (int probe = 0; probe < 128 && !found; ++probe) {
            const int64_t flat = (int64_t)vo_next_below(r, (uint64_t)total);
            vo_encode_bits(X[flat], f, &bits);
            if (eligible(bits, bit, dir)) { i = flat / n; j = flat % n; found = 1; }
        }
        if (!found) {
            int64_t cnt = 0;
            int64_t* el = malloc(sizeof(int64_t) * (size_t)total);
            for (int64_t flat = 0; flat < total; ++flat) {
                vo_encode_bits(X[flat], f, &bits);
                if (eligible(bits, bit, dir)) el[cnt++] = flat;
            }
            if (cnt == 0) { free(el); return 0; }
            const int64_t flat = el[vo_next_below(r, (uint64_t)cnt)];
            free(el);
            i = flat / n; j = flat % n;
        }
    }
    vo_encode_bits(X[i * n + j], f, &bits);
    double after;
    vo_decode_bits(bits ^ ((uint64_t)1 << bit), f, &after);
    vals[0] = X[i * n + j];
    X[i * n + j] = after;
    vals[1] = after;
    rec[0] = i; rec[1] = j; rec[2] = 1;
    return 0;
}

/* inject — proj/src/faults.cpp:104-168 */
int vo_inject(int f, int src_fp32, int64_t m, int64_t n, double* X, int64_t pos_i, int64_t pos_j,
              int bit, int dir, uint64_t seed, uint64_t stream, int64_t* rec, double* vals) {
    vo_rng r;
    vo_rng_init(&r, seed, stream);
    return inject_rng(src_fp32 ? VO_FP32 : f, m, n, X, pos_i, pos_j, bit, dir, &r, rec, vals);
}

/* One trial of injection_campaign — proj/src/faults.cpp:181-203.
 * out = {applied, detected, located, nonfinite, i, j}. method 0 V-ABFT,
 * 1 A-ABFT fixed y = 21, 2 A-ABFT computed y (harness.cpp:148-173). */
int vo_campaign_trial(int64_t m, int64_t k, int64_t n, int f, int dist_kind, double p0, double p1,
                      double lo, double hi, int bit, int dir, uint64_t seed, uint64_t trial,
                      int mode, int method, double e_max, double c_sigma, int64_t out[6]) {
    vo_rng r;
    vo_rng_init(&r, seed, trial);
    double* A = malloc(sizeof(double) * (size_t)(m * k));
    double* B = malloc(sizeof(double) * (size_t)(k * n));
    double* C = malloc(sizeof(double) * (size_t)(m * n));
    double* Ca = malloc(sizeof(double) * (size_t)(m * n));
    double* rc1 = malloc(sizeof(double) * (size_t)m);
    double* rc2 = malloc(sizeof(double) * (size_t)m);
    double* T = malloc(sizeof(double) * (size_t)m);
    double* d1 = malloc(sizeof(double) * (size_t)m);
    uint8_t* det = malloc((size_t)m);
    int64_t* loc = malloc(sizeof(int64_t) * (size_t)m);
    int rc = random_matrix(&r, m, k, f, dist_kind, p0, p1, lo, hi, A);
    if (!rc) rc = random_matrix(&r, k, n, f, dist_kind, p0, p1, lo, hi, B);
    if (!rc) rc = vo_encode_and_multiply(f, -1, 128, mode, m, k, n, A, B, C, Ca, rc1, rc2, NULL, NULL);
    if (!rc) {
        if (method == 0) {
            rc = vo_vabft_thresholds(f, m, k, n, A, B, e_max, c_sigma, T, NULL);
        } else {
            double y; int dg;
            rc = vo_aabft_threshold(f, m, k, n, A, B, -1, method == 1 ? 21.0 : NAN, 3.0, T, &y, &dg);
        }
    }
    for (int q = 0; q < 6; ++q) out[q] = 0;
    if (!rc) {
        const int online = mode == 1;
        double* target = online ? Ca : C;
        const int tf = online ? (f == VO_FP64 ? VO_FP64 : VO_FP32) : f;
        int64_t rec[4];
        double vals[2];
        rc = inject_rng(tf, m, n, target, -1, -1, bit, dir, &r, rec, vals);
        out[4] = rec[0];
        out[5] = rec[1];
        if (!rc && rec[2]) {
            rc = vo_verify(f, mode, -1, 128, m, n, target, rc1, rc2, T, 1e-3, d1, NULL, det, loc, NULL);
            if (!rc) {
                const int64_t i = rec[0];
                out[0] = 1;
                out[1] = det[i];
                out[2] = det[i] && loc[i] == rec[1];
                out[3] = !isfinite(vals[1]);
            }
        }
    }
    free(A); free(B); free(C); free(Ca); free(rc1); free(rc2); free(T); free(d1); free(det); free(loc);
    return rc;
}
