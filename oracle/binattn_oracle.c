/*
 * binattn_oracle.c -- CPU restatement of the BinaryAttention forward path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it; the product (paper_2603_09582_b200/) never does.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function below
 * against (i) the known-answer vectors of the reference's own test-suite
 * (proj/tests/test_bitops.cpp, test_attention.cpp, test_quantize.cpp) and
 * (ii) golden fixtures under tests/golden/ produced by the unmodified
 * reference compiled into oracle/_ref (see oracle/Makefile, oracle/gen_golden.py).
 *
 * Every function cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Plain C11, no dependencies beyond libm / pthreads.
 * Build: see oracle/Makefile (-O2 -ffp-contract=off -mpopcnt, the reference's
 * own flags, CMakeLists.txt:17-23, so fused/unfused stay bit-identical).
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BO_OK 0
#define BO_ESHAPE 1  /* reference: ShapeError      (errors.hpp:16) */
#define BO_EVALID 2  /* reference: ValidationError (errors.hpp:22) */
#define BO_ENOMEM 3

/* ------------------------------------------------------------------------ */
/* rng.hpp:9-65 -- splitmix64, make_rng (mt19937_64), uniform01, Box-Muller  */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t mt[312];
    int idx;
    double spare;
    int have_spare;
} bo_rng;

/* rng.hpp:17-23 */
static uint64_t bo_splitmix64(uint64_t *state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* std::mt19937_64 (ISO C++ [rand.eng.mers]; Matsumoto-Nishimura 2004). */
static void bo_mt_seed(bo_rng *r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
    r->spare = 0.0;
    r->have_spare = 0;
}

static uint64_t bo_mt_next(bo_rng *r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* rng.hpp:26-31 make_rng(seed, stream_id) */
void bo_rng_init(bo_rng *r, uint64_t seed, uint64_t stream_id) {
    uint64_t s = seed;
    uint64_t a = bo_splitmix64(&s);
    uint64_t mix = a ^ (stream_id * 0xda942042e4dd58b5ULL + 0x2545f4914f6cdd1dULL);
    bo_mt_seed(r, bo_splitmix64(&mix));
}

uint64_t bo_rng_u64(bo_rng *r) { return bo_mt_next(r); }

/* rng.hpp:34-36 uniform01 in (0,1] */
static double bo_uniform01(bo_rng *r) {
    return (double)((bo_mt_next(r) >> 11) + 1) * 0x1.0p-53;
}

/* rng.hpp:44-65 GaussianSource::operator() */
double bo_rng_gauss(bo_rng *r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = bo_uniform01(r);
    const double u2 = bo_uniform01(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(a);
    r->have_spare = 1;
    return rad * cos(a);
}

size_t bo_rng_sizeof(void) { return sizeof(bo_rng); }

/* tests/oracles.hpp:19-25 random_dense: a FRESH GaussianSource per matrix over a
 * shared rng word stream (the spare is dropped between matrices). */
void bo_random_dense(bo_rng *r, size_t count, double scale, double *out) {
    r->have_spare = 0;
    for (size_t i = 0; i < count; ++i) out[i] = scale * bo_rng_gauss(r);
    r->have_spare = 0;
}

/* ------------------------------------------------------------------------ */
/* bitops.cpp -- sign packing and XNOR-popcount                              */
/* ------------------------------------------------------------------------ */

size_t bo_words_needed(size_t d) { return (d + 63) / 64; } /* tensor.hpp:87-89 */

/* bitops.cpp:13-16 */
static uint64_t bo_tail_mask(size_t d) {
    const size_t rem = d % 64;
    return rem == 0 ? ~(uint64_t)0 : (((uint64_t)1 << rem) - 1);
}

/* bitops.cpp:37-49 pack_signs: bit c of row i = 1 iff m(i,c) >= 0.0 (so -0.0 -> 1),
 * LSB-first inside u64 words, pad bits zero. */
void bo_pack_signs(const double *m, size_t rows, size_t d, uint64_t *words) {
    const size_t wpr = bo_words_needed(d);
    memset(words, 0, rows * wpr * sizeof(uint64_t));
    for (size_t i = 0; i < rows; ++i) {
        uint64_t *out = words + i * wpr;
        for (size_t c = 0; c < d; ++c)
            if (m[i * d + c] >= 0.0) out[c / 64] |= (uint64_t)1 << (c % 64);
    }
}

/* bitops.cpp:24-33 agree_count */
static uint64_t bo_agree_count(const uint64_t *a, const uint64_t *b, size_t words, uint64_t tail) {
    uint64_t agree = 0;
    for (size_t w = 0; w + 1 < words; ++w) agree += (uint64_t)__builtin_popcountll(~(a[w] ^ b[w]));
    if (words > 0) agree += (uint64_t)__builtin_popcountll(~(a[words - 1] ^ b[words - 1]) & tail);
    return agree;
}

/* bitops.cpp:59-67 xnor_popcount_dot = 2*agree - d */
int64_t bo_xnor_popcount_dot(const uint64_t *a, const uint64_t *b, size_t d) {
    const uint64_t agree = bo_agree_count(a, b, bo_words_needed(d), bo_tail_mask(d));
    return 2 * (int64_t)agree - (int64_t)d;
}

/* bitops.cpp:75-88 hamming_distance */
uint64_t bo_hamming_distance(const uint64_t *a, const uint64_t *b, size_t d) {
    const size_t words = bo_words_needed(d);
    const uint64_t tail = bo_tail_mask(d);
    uint64_t diff = 0;
    for (size_t w = 0; w + 1 < words; ++w) diff += (uint64_t)__builtin_popcountll(a[w] ^ b[w]);
    if (words > 0) diff += (uint64_t)__builtin_popcountll((a[words - 1] ^ b[words - 1]) & tail);
    return diff;
}

/* bitops.cpp:96-131 binary_gemm: out(i,j) = xnor_popcount_dot(S row i, T row j) */
void bo_binary_gemm(const uint64_t *s, size_t n, const uint64_t *t, size_t m, size_t d, int32_t *out) {
    const size_t words = bo_words_needed(d);
    const uint64_t tail = bo_tail_mask(d);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < m; ++j)
            out[i * m + j] =
                (int32_t)(2 * (int64_t)bo_agree_count(s + i * words, t + j * words, words, tail) - (int64_t)d);
}

/* ------------------------------------------------------------------------ */
/* quantize.cpp                                                              */
/* ------------------------------------------------------------------------ */

/* quantize.cpp:16-23 binary_quantize: mu = (sequential sum of |x|) / size, + pack_signs */
int bo_binary_quantize(const double *m, size_t rows, size_t d, uint64_t *words, double *mu) {
    if (rows * d == 0) return BO_ESHAPE; /* quantize.cpp:17 */
    double sum_abs = 0.0;
    for (size_t i = 0; i < rows * d; ++i) sum_abs += fabs(m[i]);
    *mu = sum_abs / (double)(rows * d);
    bo_pack_signs(m, rows, d, words);
    return BO_OK;
}

/* quantize.hpp:43 round_half_away == std::round */
static double bo_round_half_away(double x) { return round(x); }

/* quantize.cpp:57-74 quantize_values: per-column scale = max|v|/127 (1 for a zero column) */
void bo_quantize_values(const double *v, size_t rows, size_t cols, int8_t *data, double *scales) {
    for (size_t c = 0; c < cols; ++c) {
        double amax = 0.0;
        for (size_t i = 0; i < rows; ++i) amax = fmax(amax, fabs(v[i * cols + c]));
        scales[c] = amax > 0.0 ? amax / 127.0 : 1.0;
    }
    for (size_t i = 0; i < rows; ++i)
        for (size_t c = 0; c < cols; ++c)
            data[i * cols + c] = (int8_t)bo_round_half_away(v[i * cols + c] / scales[c]);
}

/* quantize.cpp:35-48 quantize_coeffs: round(P*255) with clamp to [0,1] */
int bo_quantize_coeffs(const double *p, size_t count, uint8_t *q) {
    const double tol = 1e-9;
    for (size_t k = 0; k < count; ++k) {
        const double v = p[k];
        if (v < -tol || v > 1.0 + tol) return BO_EVALID; /* RangeError in the reference */
        const double clamped = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        q[k] = (uint8_t)bo_round_half_away(clamped * 255.0);
    }
    return BO_OK;
}

/* ------------------------------------------------------------------------ */
/* attention.cpp                                                             */
/* ------------------------------------------------------------------------ */

/* attention.cpp:65-76 Relative1dBias: b_ij = offsets[i - j + N - 1] */
void bo_materialize_bias_rel1d(const double *offsets, size_t n, double *table) {
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j)
            table[i * n + j] = offsets[(size_t)((ptrdiff_t)i - (ptrdiff_t)j + (ptrdiff_t)n - 1)];
}

/* attention.cpp:78-96 Relative2dBias: g = sqrt(N) grid, b_ij = row[dr+g-1] + col[dc+g-1] */
int bo_materialize_bias_rel2d(const double *row_off, const double *col_off, size_t n, double *table) {
    size_t g = (size_t)lround(sqrt((double)n));
    if (g * g != n) return BO_ESHAPE;
    for (size_t i = 0; i < n; ++i) {
        const ptrdiff_t ri = (ptrdiff_t)(i / g), ci = (ptrdiff_t)(i % g);
        for (size_t j = 0; j < n; ++j) {
            const ptrdiff_t rj = (ptrdiff_t)(j / g), cj = (ptrdiff_t)(j % g);
            table[i * n + j] = row_off[(size_t)(ri - rj + (ptrdiff_t)g - 1)] + col_off[(size_t)(ci - cj + (ptrdiff_t)g - 1)];
        }
    }
    return BO_OK;
}

/* attention.cpp:34-36 binary_score: mu_prod * double(dot) / tau + bias, in that order, unfused */
static double bo_binary_score(int64_t dot, double mu_prod, double tau, double bias) {
    return mu_prod * (double)dot / tau + bias;
}

/* attention.cpp:17-29 check_shapes (shape part is implied by the flat arguments) */
static int bo_check_cfg(size_t n, size_t d, double tau, size_t br, size_t bc) {
    if (n == 0 || d == 0) return BO_ESHAPE;
    if (!(tau > 0.0)) return BO_EVALID;
    if (br < 1 || br > n || bc < 1 || bc > n) return BO_EVALID;
    return BO_OK;
}

/* fidelity.cpp:12-24 check_row_stochastic: weights >= -1e-6, every row sums to 1 within 1e-6 */
static int bo_check_row_stochastic(const double *p, size_t rows, size_t cols) {
    for (size_t i = 0; i < rows; ++i) {
        double sum = 0.0;
        for (size_t j = 0; j < cols; ++j) {
            const double v = p[i * cols + j];
            if (v < -1e-6) return BO_EVALID;
            sum += v;
        }
        if (fabs(sum - 1.0) > 1e-6) return BO_EVALID;
    }
    return BO_OK;
}

/* fidelity.cpp:26-36 topk_indices: the k largest entries, ties broken toward the lower index (selection form) */
static void bo_topk(const double *row, size_t n, size_t k, char *used, size_t *out) {
    memset(used, 0, n);
    for (size_t t = 0; t < k; ++t) {
        size_t best = n;
        for (size_t j = 0; j < n; ++j) {
            if (used[j]) continue;
            if (best == n || row[j] > row[best]) best = j;
        }
        used[best] = 1;
        out[t] = best;
    }
}

/* fidelity.cpp:40-85 attention_fidelity: out = {cos_sim, relative_l1, rmse, precision_at_k} */
int bo_attention_fidelity(const double *p_ref, const double *p_other, size_t rows, size_t cols, size_t k, double *out) {
    if (rows == 0 || cols == 0) return BO_ESHAPE;
    if (k == 0) return BO_EVALID;
    int rc = bo_check_row_stochastic(p_ref, rows, cols);
    if (rc) return rc;
    rc = bo_check_row_stochastic(p_other, rows, cols);
    if (rc) return rc;
    const size_t count = rows * cols;
    double dot = 0.0, na = 0.0, nb = 0.0, l1_diff = 0.0, l1_ref = 0.0, sq = 0.0;
    for (size_t t = 0; t < count; ++t) {
        const double a = p_ref[t], b = p_other[t];
        dot += a * b;
        na += a * a;
        nb += b * b;
        l1_diff += fabs(a - b);
        l1_ref += fabs(a);
        sq += (a - b) * (a - b);
    }
    out[0] = dot / (sqrt(na) * sqrt(nb));
    out[1] = l1_diff / l1_ref;
    out[2] = sqrt(sq / (double)count);
    const size_t keff = k < cols ? k : cols;
    char *used = (char *)malloc(cols), *in_a = (char *)malloc(cols);
    size_t *ta = (size_t *)malloc(keff * sizeof(size_t)), *tb = (size_t *)malloc(keff * sizeof(size_t));
    if (!used || !in_a || !ta || !tb) {
        free(used); free(in_a); free(ta); free(tb);
        return BO_ENOMEM;
    }
    double prec = 0.0;
    for (size_t i = 0; i < rows; ++i) {
        bo_topk(p_ref + i * cols, cols, keff, used, ta);
        bo_topk(p_other + i * cols, cols, keff, used, tb);
        memset(in_a, 0, cols);
        for (size_t t = 0; t < keff; ++t) in_a[ta[t]] = 1;
        size_t hits = 0;
        for (size_t t = 0; t < keff; ++t) hits += (size_t)in_a[tb[t]];
        prec += (double)hits / (double)keff;
    }
    out[3] = prec / (double)rows;
    free(used); free(in_a); free(ta); free(tb);
    return BO_OK;
}

/* attention.cpp:99-147 reference_attention (fp64 dense softmax attention) */
int bo_reference_attention(const double *q, const double *k, const double *v, size_t n, size_t d, double tau,
                           const double *bias /* n*n or NULL */, double *y, double *m, double *l,
                           double *probs /* n*n or NULL */) {
    int rc = bo_check_cfg(n, d, tau, 1, 1);
    if (rc) return rc;
    double *srow = (double *)malloc(n * sizeof(double));
    if (!srow) return BO_ENOMEM;
    memset(y, 0, n * d * sizeof(double));
    for (size_t i = 0; i < n; ++i) {
        for (size_t j = 0; j < n; ++j) {
            double dot = 0.0;
            for (size_t c = 0; c < d; ++c) dot += q[i * d + c] * k[j * d + c];
            srow[j] = dot / tau + (bias ? bias[i * n + j] : 0.0);
        }
        double mi = -INFINITY;
        for (size_t j = 0; j < n; ++j) mi = fmax(mi, srow[j]);
        double li = 0.0;
        for (size_t j = 0; j < n; ++j) {
            srow[j] = exp(srow[j] - mi);
            li += srow[j];
        }
        for (size_t j = 0; j < n; ++j) srow[j] /= li;
        for (size_t j = 0; j < n; ++j) {
            const double p = srow[j];
            for (size_t c = 0; c < d; ++c) y[i * d + c] += p * v[j * d + c];
        }
        if (m) m[i] = mi;
        if (l) l[i] = li;
        if (probs) memcpy(probs + i * n, srow, n * sizeof(double));
    }
    free(srow);
    return BO_OK;
}

/* attention.cpp:149-248 binary_attention_unfused */
int bo_binary_attention_unfused(const double *q, const double *k, const double *v, size_t n, size_t d, double tau,
                                int quantize_pv, const double *bias, double *y, double *m, double *l,
                                double *probs /* n*n or NULL */) {
    int rc = bo_check_cfg(n, d, tau, 1, 1);
    if (rc) return rc;
    const size_t wpr = bo_words_needed(d);
    uint64_t *qb = (uint64_t *)malloc(n * wpr * 8), *kb = (uint64_t *)malloc(n * wpr * 8);
    int32_t *g = (int32_t *)malloc(n * n * sizeof(int32_t));
    double *s = (double *)malloc(n * n * sizeof(double));
    if (!qb || !kb || !g || !s) return BO_ENOMEM;
    double mu_q, mu_k;
    bo_binary_quantize(q, n, d, qb, &mu_q);
    bo_binary_quantize(k, n, d, kb, &mu_k);
    const double mu_prod = mu_q * mu_k;
    bo_binary_gemm(qb, n, kb, n, d, g);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j)
            s[i * n + j] = bo_binary_score(g[i * n + j], mu_prod, tau, bias ? bias[i * n + j] : 0.0);
    for (size_t i = 0; i < n; ++i) { /* attention.cpp:173-186 */
        double *row = s + i * n;
        double mi = -INFINITY;
        for (size_t j = 0; j < n; ++j) mi = fmax(mi, row[j]);
        double li = 0.0;
        for (size_t j = 0; j < n; ++j) {
            row[j] = exp(row[j] - mi);
            li += row[j];
        }
        m[i] = mi;
        l[i] = li;
    }
    memset(y, 0, n * d * sizeof(double));
    if (!quantize_pv) { /* attention.cpp:193-214: divide AFTER accumulation */
        for (size_t i = 0; i < n; ++i) {
            const double *row = s + i * n;
            double *yrow = y + i * d;
            for (size_t j = 0; j < n; ++j) {
                const double p = row[j];
                for (size_t c = 0; c < d; ++c) yrow[c] += p * v[j * d + c];
            }
            for (size_t c = 0; c < d; ++c) yrow[c] /= l[i];
        }
        if (probs)
            for (size_t i = 0; i < n; ++i)
                for (size_t j = 0; j < n; ++j) probs[i * n + j] = s[i * n + j] / l[i];
    } else { /* attention.cpp:215-245 */
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < n; ++j) s[i * n + j] /= l[i];
        uint8_t *pq = (uint8_t *)malloc(n * n);
        int8_t *vq = (int8_t *)malloc(n * d);
        double *scales = (double *)malloc(d * sizeof(double));
        int32_t *acc = (int32_t *)malloc(d * sizeof(int32_t));
        if (!pq || !vq || !scales || !acc) return BO_ENOMEM;
        rc = bo_quantize_coeffs(s, n * n, pq);
        bo_quantize_values(v, n, d, vq, scales);
        for (size_t i = 0; i < n && !rc; ++i) {
            memset(acc, 0, d * sizeof(int32_t));
            for (size_t j = 0; j < n; ++j) {
                const int32_t p8 = pq[i * n + j];
                for (size_t c = 0; c < d; ++c) acc[c] += p8 * (int32_t)vq[j * d + c];
            }
            for (size_t c = 0; c < d; ++c) y[i * d + c] = (double)acc[c] * scales[c] / 255.0;
        }
        if (probs) memcpy(probs, s, n * n * sizeof(double));
        free(pq); free(vq); free(scales); free(acc);
    }
    free(qb); free(kb); free(g); free(s);
    return rc;
}

/* attention.cpp:250-382 binary_attention_fused (Algorithm 1: tiled online softmax).
 * br/bc are the reference's block_rows/block_cols. */
int bo_binary_attention_fused(const double *q, const double *k, const double *v, size_t n, size_t d, double tau,
                              size_t br_max, size_t bv, int quantize_pv, const double *bias, double *y, double *m,
                              double *l) {
    int rc = bo_check_cfg(n, d, tau, br_max, bv);
    if (rc) return rc;
    const size_t t_r = (n + br_max - 1) / br_max;
    const size_t t_v = (n + bv - 1) / bv;
    const size_t wpr = bo_words_needed(d);
    uint64_t *qb = (uint64_t *)malloc(n * wpr * 8), *kb = (uint64_t *)malloc(n * wpr * 8);
    double *sblk = (double *)malloc(br_max * bv * sizeof(double));
    double *o = (double *)malloc(br_max * d * sizeof(double));
    int32_t *acc = (int32_t *)malloc(d * sizeof(int32_t));
    int8_t *vq = NULL;
    double *vscale = NULL;
    if (!qb || !kb || !sblk || !o || !acc) return BO_ENOMEM;
    double mu_q, mu_k;
    bo_binary_quantize(q, n, d, qb, &mu_q); /* :262 */
    bo_binary_quantize(k, n, d, kb, &mu_k); /* :263 */
    const double mu_prod = mu_q * mu_k;     /* :264 */
    if (quantize_pv) {                      /* :266 */
        vq = (int8_t *)malloc(n * d);
        vscale = (double *)malloc(d * sizeof(double));
        if (!vq || !vscale) return BO_ENOMEM;
        bo_quantize_values(v, n, d, vq, vscale);
    }
    for (size_t i = 0; i < n; ++i) { m[i] = -INFINITY; l[i] = 0.0; } /* :270 */

    for (size_t ib = 0; ib < t_r; ++ib) { /* :278 */
        const size_t r0 = ib * br_max;
        const size_t r1 = n < r0 + br_max ? n : r0 + br_max;
        const size_t br = r1 - r0;
        memset(o, 0, br * d * sizeof(double));
        for (size_t jb = 0; jb < t_v; ++jb) { /* :284 */
            const size_t c0 = jb * bv;
            const size_t c1 = n < c0 + bv ? n : c0 + bv;
            const size_t bc = c1 - c0;
            for (size_t r = 0; r < br; ++r) { /* :289-298 scores */
                double *out_row = sblk + r * bc;
                for (size_t j = 0; j < bc; ++j) {
                    const int64_t dot = bo_xnor_popcount_dot(qb + (r0 + r) * wpr, kb + (c0 + j) * wpr, d);
                    out_row[j] = bo_binary_score(dot, mu_prod, tau, bias ? bias[(r0 + r) * n + c0 + j] : 0.0);
                }
            }
            for (size_t r = 0; r < br; ++r) { /* :306-344 online-softmax update */
                double *row = sblk + r * bc;
                double bm = -INFINITY;
                for (size_t j = 0; j < bc; ++j) bm = fmax(bm, row[j]);
                const double m_old = m[r0 + r];
                const double m_new = fmax(m_old, bm);
                const double rescale = exp(m_old - m_new);
                double rs = 0.0;
                for (size_t j = 0; j < bc; ++j) {
                    row[j] = exp(row[j] - m_new);
                    rs += row[j];
                }
                l[r0 + r] = rescale * l[r0 + r] + rs;
                m[r0 + r] = m_new;
                double *orow = o + r * d;
                if (rescale != 1.0)
                    for (size_t c = 0; c < d; ++c) orow[c] *= rescale;
                if (!quantize_pv) { /* :326-331 */
                    for (size_t j = 0; j < bc; ++j) {
                        const double p = row[j];
                        const double *vj = v + (c0 + j) * d;
                        for (size_t c = 0; c < d; ++c) orow[c] += p * vj[c];
                    }
                } else { /* :332-343 */
                    memset(acc, 0, d * sizeof(int32_t));
                    for (size_t j = 0; j < bc; ++j) {
                        const int32_t p8 = (int32_t)bo_round_half_away(row[j] * 255.0);
                        const int8_t *vj = vq + (c0 + j) * d;
                        for (size_t c = 0; c < d; ++c) acc[c] += p8 * (int32_t)vj[c];
                    }
                    for (size_t c = 0; c < d; ++c) orow[c] += (double)acc[c];
                }
            }
        }
        for (size_t r = 0; r < br; ++r) { /* :354-364 epilogue */
            const double *orow = o + r * d;
            double *yrow = y + (r0 + r) * d;
            const double li = l[r0 + r];
            if (!quantize_pv)
                for (size_t c = 0; c < d; ++c) yrow[c] = orow[c] / li;
            else
                for (size_t c = 0; c < d; ++c) yrow[c] = orow[c] / li / 255.0 * vscale[c];
        }
    }
    free(qb); free(kb); free(sblk); free(o); free(acc); free(vq); free(vscale);
    return BO_OK;
}

/* ------------------------------------------------------------------------ */
/* Batched driver: heads are independent calls, spread over    */
/* host threads.  Used only for the CPU baseline timing in bench.py.         */
/* ------------------------------------------------------------------------ */

typedef struct {
    const double *q, *k, *v, *bias;
    double *y;
    size_t n, d, heads, bias_heads, br, bc;
    double tau;
    int quantize_pv;
    size_t begin, end;
    int rc;
} bo_job;

static void *bo_worker(void *arg) {
    bo_job *j = (bo_job *)arg;
    double *m = (double *)malloc(j->n * sizeof(double)), *l = (double *)malloc(j->n * sizeof(double));
    for (size_t h = j->begin; h < j->end; ++h) {
        const double *b = j->bias ? j->bias + (h % j->bias_heads) * j->n * j->n : NULL;
        int rc = bo_binary_attention_fused(j->q + h * j->n * j->d, j->k + h * j->n * j->d, j->v + h * j->n * j->d,
                                           j->n, j->d, j->tau, j->br, j->bc, j->quantize_pv, b,
                                           j->y + h * j->n * j->d, m, l);
        if (rc) j->rc = rc;
    }
    free(m); free(l);
    return NULL;
}

/* q,k,v,y: [heads, n, d]; bias: [bias_heads, n, n] or NULL (head h uses table h % bias_heads). */
int bo_binary_attention_fused_heads(const double *q, const double *k, const double *v, size_t heads, size_t n,
                                    size_t d, double tau, size_t br, size_t bc, int quantize_pv, const double *bias,
                                    size_t bias_heads, double *y, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if ((size_t)nthreads > heads) nthreads = (int)heads;
    if (heads == 0) return BO_OK;
    pthread_t *tid = (pthread_t *)malloc((size_t)nthreads * sizeof(pthread_t));
    bo_job *jobs = (bo_job *)malloc((size_t)nthreads * sizeof(bo_job));
    const size_t chunk = (heads + (size_t)nthreads - 1) / (size_t)nthreads;
    int rc = BO_OK;
    for (int t = 0; t < nthreads; ++t) {
        bo_job jb = {q, k, v, bias, y, n, d, heads, bias_heads ? bias_heads : 1, br, bc, tau, quantize_pv,
                     (size_t)t * chunk, 0, BO_OK};
        jb.end = jb.begin + chunk < heads ? jb.begin + chunk : heads;
        if (jb.begin > heads) jb.begin = heads;
        jobs[t] = jb;
        pthread_create(&tid[t], NULL, bo_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(tid[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    free(tid); free(jobs);
    return rc;
}
