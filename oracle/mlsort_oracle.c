/*
 * mlsort_oracle.c -- CPU ORACLE for Machine Learning Sort (Zhao & Luo, arXiv 1805.04272).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this code.  The product path
 * (paper_1805_04272_b200/) never includes, links or calls it, and it shares no
 * code, header, table or constant with the product.
 *
 * Plain, slow, obviously-correct fp64 implementation of the inference-and-
 * placement phase, written step by step in the paper's order
 * (SURVEY.md §8(c) "Oracle algorithm"):
 *
 *   1 validate      reject NaN/+-Inf, lowest index          (reading A11)
 *   2 predict       Eq. 3, y = sum_j w2_j f0(beta_j(w1_j x^ - b_j)),
 *                   f0 = logistic, x^ = 2(x-lo)/(hi-lo) - 1  (§2 Eq. 3 l.73-76;
 *                                                             readings A2, A3, A5)
 *   3 bucket        r = round(y * B), half away from zero, clamp [0, B-1]
 *                   (§2 l.65 "r_j = round(y_j N/N0)"; readings A4, A6, A7, A8)
 *   4 tails         count x < lo and x > hi (diagnostic)    (§3 l.121; A13, A26)
 *   5 place         keys into buckets in input order         (§2 l.86)
 *   6 fix-up        per-bucket stable insertion sort         (§2 l.86 "only the
 *                                                             numbers inside each bucket need
 *                                                             to be sorted"; A12)
 *   7 concatenate   buckets 0..B-1 (implicit in the layout)
 *   8 verify/repair adjacent-pair check; on violation a stable insertion sort of the
 *                   whole array (reading A14)
 *   9 emit          keys, permutation, y, b, counts, tails, repairs
 *
 * Keys are handled as IEEE doubles (f32 keys widen exactly) and ordered by IEEE-754
 * totalOrder through order-preserving unsigned bits, ties by input index (A9, A10).
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (no fast-math, no
 * FMA contraction, so every product and sum is rounded as written).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_NONFINITE 5
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_NOMEM 12

/* ---- IEEE totalOrder key (reading A10): negative -> flip all bits, else flip sign. */
static uint64_t order_bits(double x) {
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

/* (key, idx) strictly precedes (key', idx') */
static int precedes(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

/* ---- Step 1: validate.  Returns the lowest index of a NaN or +-Inf key, or -1. */
int64_t oracle_validate(const double* x, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return (int64_t)i;
    return -1;
}

/* ---- Step 2: Eq. 3 forward pass for one key, double precision, neuron order j = 0..m-1.
 * x^ = 2 (x - lo) / (hi - lo) - 1 (reading A3); f0(t) = 1 / (1 + exp(-t)) (reading A2).
 * exp(-t) overflowing to +inf gives the exact limit 0 for that term. */
double oracle_gvm_forward(int m, const double* w1, const double* w2, const double* b,
                          const double* beta, double lo, double hi, double x) {
    double xh = 2.0 * (x - lo) / (hi - lo) - 1.0;
    double y = 0.0;
    for (int j = 0; j < m; ++j) {
        double t = beta[j] * (w1[j] * xh - b[j]);
        double f0 = 1.0 / (1.0 + exp(-t));
        y = y + w2[j] * f0;
    }
    return y;
}

void oracle_predict(int m, const double* w1, const double* w2, const double* b,
                    const double* beta, double lo, double hi,
                    const double* x, uint64_t n, double* y) {
    for (uint64_t i = 0; i < n; ++i)
        y[i] = oracle_gvm_forward(m, w1, w2, b, beta, lo, hi, x[i]);
}

/* ---- Step 3: r = round(y * B) half away from zero, clamped to [0, B-1]
 * (S:232, S:297-S:298). */
uint64_t oracle_bucket_of(double y, uint64_t B) {
    double v = y * (double)B;
    double r = (v >= 0.0) ? floor(v + 0.5) : -floor(-v + 0.5);
    if (!(r > 0.0)) return 0;                       /* also catches r <= 0 */
    if (r >= (double)(B - 1)) return B - 1;
    return (uint64_t)r;
}

void oracle_bucket(const double* y, uint64_t n, uint64_t B, uint32_t* bucket) {
    for (uint64_t i = 0; i < n; ++i) bucket[i] = (uint32_t)oracle_bucket_of(y[i], B);
}

/* ---- Step 8 helper: stable insertion sort of (key, idx) pairs by (order_bits, idx).
 * Returns the number of element moves (inversions resolved). */
static uint64_t insertion_sort(double* k, uint32_t* idx, uint64_t n) {
    uint64_t moves = 0;
    for (uint64_t i = 1; i < n; ++i) {
        double kv = k[i];
        uint32_t iv = idx[i];
        uint64_t ov = order_bits(kv);
        uint64_t j = i;
        while (j > 0 && precedes(ov, iv, order_bits(k[j - 1]), idx[j - 1])) {
            k[j] = k[j - 1];
            idx[j] = idx[j - 1];
            --j;
            ++moves;
        }
        k[j] = kv;
        idx[j] = iv;
    }
    return moves;
}

/* ---- Steps 5-7: place keys into B buckets (given their bucket ids) in input order, then
 * sort each bucket by stable insertion sort.  `counts` (B entries) is written if non-NULL.
 * This is the textbook bucket sort the paper reduces to. */
int oracle_place_fixup(const double* x, const uint32_t* bucket, uint64_t n, uint64_t B,
                       double* out_keys, uint32_t* out_idx, uint32_t* counts_out,
                       uint64_t* fixup_moves) {
    uint64_t* start = (uint64_t*)calloc(B + 1, sizeof(uint64_t));
    if (!start) return ORACLE_ERR_NOMEM;
    for (uint64_t i = 0; i < n; ++i) start[bucket[i] + 1]++;          /* counts */
    if (counts_out)
        for (uint64_t c = 0; c < B; ++c) counts_out[c] = (uint32_t)start[c + 1];
    for (uint64_t c = 0; c < B; ++c) start[c + 1] += start[c];        /* exclusive scan */
    uint64_t* fill = (uint64_t*)malloc(B * sizeof(uint64_t));
    if (!fill) { free(start); return ORACLE_ERR_NOMEM; }
    memcpy(fill, start, B * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {                                /* place, input order */
        uint64_t p = fill[bucket[i]]++;
        out_keys[p] = x[i];
        out_idx[p] = (uint32_t)i;
    }
    free(fill);
    uint64_t moves = 0;
    for (uint64_t c = 0; c < B; ++c) {                                /* per-bucket fix-up */
        uint64_t s = start[c], e = start[c + 1];
        if (e - s > 1) moves += insertion_sort(out_keys + s, out_idx + s, e - s);
    }
    free(start);
    if (fixup_moves) *fixup_moves = moves;
    return ORACLE_OK;
}

/* ---- Step 8: verify; on violation repair with a whole-array stable insertion sort.
 * stable != 0: (key, idx) must be strictly increasing; else keys non-decreasing.
 * Returns the number of adjacent violations found before the repair. */
uint64_t oracle_verify_repair(double* keys, uint32_t* idx, uint64_t n, int stable) {
    uint64_t bad = 0;
    for (uint64_t i = 1; i < n; ++i) {
        uint64_t a = order_bits(keys[i - 1]), b = order_bits(keys[i]);
        if (stable ? !precedes(a, idx[i - 1], b, idx[i]) : (a > b)) ++bad;
    }
    if (bad) insertion_sort(keys, idx, n);
    return bad;
}

/* ---- Step 4: tail diagnostic (strict inequalities, reading A26). */
void oracle_tails(const double* x, uint64_t n, double lo, double hi,
                  uint64_t* below, uint64_t* above) {
    uint64_t a = 0, b = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (x[i] < lo) ++a;
        if (x[i] > hi) ++b;
    }
    *below = a;
    *above = b;
}

/* ---- Full pipeline, steps 1-9.  Outputs out_keys[n], out_idx[n] (gather form: out_idx[i]
 * is the input index of the i-th output), optional y[n], bucket[n], counts[B].
 * info[0]=bad_index (or -1), info[1]=repairs, info[2]=tail_lo, info[3]=tail_hi,
 * info[4]=fix-up moves, info[5]=max bucket size.  Returns 0 or ORACLE_ERR_NONFINITE. */
int oracle_ml_sort(const double* x, uint64_t n, int m, const double* w1, const double* w2,
                   const double* b, const double* beta, double lo, double hi, uint64_t B,
                   int stable, double* out_keys, uint32_t* out_idx, double* y_out,
                   uint32_t* bucket_out, uint32_t* counts_out, int64_t* info) {
    for (int i = 0; i < 6; ++i) info[i] = 0;
    int64_t badi = oracle_validate(x, n);                              /* step 1 */
    info[0] = badi;
    if (badi >= 0) return ORACLE_ERR_NONFINITE;
    if (n == 0) return ORACLE_OK;
    if (B == 0) B = n;
    uint32_t* bucket = bucket_out ? bucket_out : (uint32_t*)malloc(n * sizeof(uint32_t));
    if (!bucket) return ORACLE_ERR_NOMEM;
    for (uint64_t i = 0; i < n; ++i) {                                 /* steps 2-3 */
        double yi = oracle_gvm_forward(m, w1, w2, b, beta, lo, hi, x[i]);
        if (y_out) y_out[i] = yi;
        bucket[i] = (uint32_t)oracle_bucket_of(yi, B);
    }
    uint64_t tl, th;
    oracle_tails(x, n, lo, hi, &tl, &th);                              /* step 4 */
    info[2] = (int64_t)tl;
    info[3] = (int64_t)th;
    uint32_t* counts = counts_out ? counts_out : (uint32_t*)malloc(B * sizeof(uint32_t));
    if (!counts) { if (!bucket_out) free(bucket); return ORACLE_ERR_NOMEM; }
    uint64_t moves = 0;                                                /* steps 5-7 */
    int rc = oracle_place_fixup(x, bucket, n, B, out_keys, out_idx, counts, &moves);
    if (rc == ORACLE_OK) {
        uint32_t mx = 0;
        for (uint64_t c = 0; c < B; ++c) if (counts[c] > mx) mx = counts[c];
        info[4] = (int64_t)moves;
        info[5] = (int64_t)mx;
        info[1] = (int64_t)oracle_verify_repair(out_keys, out_idx, n, stable);   /* step 8 */
    }
    if (!counts_out) free(counts);
    if (!bucket_out) free(bucket);
    return rc;
}

/* ---- Eq. 5: p(q) = C(N,q) (1/N)^q (1 - 1/N)^(N-q), generalised to
 * B buckets as Binomial(N, 1/B) (reading A8).  Evaluated in log space. */
double oracle_expected_occupancy(uint64_t N, uint64_t B, uint64_t q) {
    if (q > N) return 0.0;
    double n = (double)N, p = 1.0 / (double)B, k = (double)q;
    if (B == 1) return q == N ? 1.0 : 0.0;
    double lg = lgamma(n + 1.0) - lgamma(k + 1.0) - lgamma(n - k + 1.0);
    return exp(lg + k * log(p) + (n - k) * log1p(-p));
}

/* ---- Occupancy histogram: hist[q] = #buckets holding exactly q keys, q < qmax;
 * hist[qmax] = #buckets holding >= qmax keys. */
void oracle_occupancy_histogram(const uint32_t* counts, uint64_t B, uint32_t qmax,
                                uint64_t* hist) {
    for (uint32_t q = 0; q <= qmax; ++q) hist[q] = 0;
    for (uint64_t c = 0; c < B; ++c) hist[counts[c] < qmax ? counts[c] : qmax]++;
}
