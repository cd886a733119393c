/* cfg5.c — TEST INFRASTRUCTURE ONLY: CPU restatements for BASELINE config 5
 * (the support-count kernel microbenchmark: 50M x 512 i.i.d. Bernoulli(0.05)
 * bits, 100k candidates with k ~ U{2..6}).
 *
 *  - orc_bernoulli_rows / orc_bernoulli_cols restate the device generator
 *    (paper_1812_10959_b200/csrc/probe.cu, bernoulli_rows_kernel): bit
 *    (row r, item i) is set iff a 32-bit half of
 *        mix64(key ^ r*0xD1B54A32D192ED03 + (i>>1)*0x9E3779B97F4A7C15)
 *    (high half for even i, low half for odd i) is below floor(p * 2^32),
 *    key = mix64(seed ^ 0x62657266).  The column form holds item i's bits
 *    of 64 consecutive rows per word.
 *  - orc_count_cols is the reference's support count (_count_block,
 *    engine.py:43-58: rows r in [0, n) with (T_r & I) == I) for many
 *    candidates, computed column-wise: popcount of the AND of the
 *    candidate's item columns, blocked over row words so the columns of a
 *    block stay in cache.  Same arithmetic as dic_oracle.c's row form
 *    (tests cross-check the two on small n).
 *
 * Only tests/ and the golden-fixture scripts use these.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static uint32_t threshold(double p) {
    double t = p * 4294967296.0;
    return t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
}

/* rows [r0, r0 + nrows) as uint64 [nrows][W] (LSW first) */
void orc_bernoulli_rows(int64_t r0, int64_t nrows, int m, double p, uint64_t seed, uint64_t* rows) {
    const int W = (m + 63) / 64;
    const uint32_t th = threshold(p);
    const uint64_t key = mix64(seed ^ 0x62657266ull);
    for (int64_t j = 0; j < nrows; ++j) {
        const uint64_t base = key ^ ((uint64_t)(r0 + j) * 0xD1B54A32D192ED03ull);
        for (int w = 0; w < W; ++w) {
            uint64_t word = 0;
            for (int b = 0; b < 64; b += 2) {
                const int item = w * 64 + b;
                const uint64_t h = mix64(base + (uint64_t)(item >> 1) * 0x9E3779B97F4A7C15ull);
                if (item < m && (uint32_t)(h >> 32) < th) word |= 1ull << b;
                if (item + 1 < m && (uint32_t)h < th) word |= 1ull << (b + 1);
            }
            rows[j * W + w] = word;
        }
    }
}

typedef struct {
    int64_t n, nw, w0, w1;
    int m;
    uint32_t th;
    uint64_t key;
    uint64_t* cols;
} ColJob;

static void* cols_worker(void* arg) {
    ColJob* J = (ColJob*)arg;
    uint64_t acc[1024];
    for (int64_t w = J->w0; w < J->w1; ++w) {
        memset(acc, 0, sizeof(uint64_t) * (size_t)J->m);
        for (int b = 0; b < 64; ++b) {
            const int64_t r = w * 64 + b;
            if (r >= J->n) break;
            const uint64_t base = J->key ^ ((uint64_t)r * 0xD1B54A32D192ED03ull);
            for (int i = 0; i < J->m; i += 2) {
                const uint64_t h = mix64(base + (uint64_t)(i >> 1) * 0x9E3779B97F4A7C15ull);
                if ((uint32_t)(h >> 32) < J->th) acc[i] |= 1ull << b;
                if (i + 1 < J->m && (uint32_t)h < J->th) acc[i + 1] |= 1ull << b;
            }
        }
        for (int i = 0; i < J->m; ++i) J->cols[(int64_t)i * J->nw + w] = acc[i];
    }
    return NULL;
}

/* all n rows as columns uint64 [m][ceil(n/64)]; m <= 1024 */
int orc_bernoulli_cols(int64_t n, int m, double p, uint64_t seed, uint64_t* cols, int threads) {
    if (m < 1 || m > 1024 || n < 1) return -1;
    const int64_t nw = (n + 63) / 64;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    ColJob jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (ColJob){n, nw, nw * t / threads, nw * (t + 1) / threads, m, threshold(p),
                           mix64(seed ^ 0x62657266ull), cols};
        pthread_create(&th[t], NULL, cols_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    return 0;
}

typedef struct {
    const uint64_t* cols;
    int64_t nw, w0, w1;
    const uint16_t* items;
    const int32_t* ks;
    int64_t C;
    int kmax;
    int64_t* out; /* [C] partial counts of this worker */
} CountJob;

#define BLOCK_WORDS 2048

static void* count_worker(void* arg) {
    CountJob* J = (CountJob*)arg;
    for (int64_t b0 = J->w0; b0 < J->w1; b0 += BLOCK_WORDS) {
        const int64_t b1 = b0 + BLOCK_WORDS < J->w1 ? b0 + BLOCK_WORDS : J->w1;
        const int64_t len = b1 - b0;
        for (int64_t c = 0; c < J->C; ++c) {
            const int k = J->ks[c];
            const uint16_t* it = J->items + c * J->kmax;
            const uint64_t* p[8];
            for (int j = 0; j < k && j < 8; ++j) p[j] = J->cols + (int64_t)it[j] * J->nw + b0;
            int64_t s = 0;
            if (k == 1) {
                for (int64_t w = 0; w < len; ++w) s += __builtin_popcountll(p[0][w]);
            } else if (k == 2) {
                for (int64_t w = 0; w < len; ++w) s += __builtin_popcountll(p[0][w] & p[1][w]);
            } else if (k == 3) {
                for (int64_t w = 0; w < len; ++w) s += __builtin_popcountll(p[0][w] & p[1][w] & p[2][w]);
            } else {
                for (int64_t w = 0; w < len; ++w) {
                    uint64_t x = p[0][w] & p[1][w] & p[2][w] & p[3][w];
                    for (int j = 4; j < k; ++j) x &= J->cols[(int64_t)it[j] * J->nw + b0 + w];
                    s += __builtin_popcountll(x);
                }
            }
            J->out[c] += s;
        }
    }
    return NULL;
}

/* out[c] = number of rows holding every item of candidate c (items[c][0..k)) */
int orc_count_cols(const uint64_t* cols, int64_t nw, const uint16_t* items, const int32_t* ks, int64_t C, int kmax,
                   int64_t* out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    CountJob jobs[256];
    int64_t* part = (int64_t*)calloc((size_t)threads * (size_t)(C > 0 ? C : 1), sizeof(int64_t));
    if (!part) return -1;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (CountJob){cols, nw, nw * t / threads, nw * (t + 1) / threads, items, ks, C, kmax, part + t * C};
        pthread_create(&th[t], NULL, count_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    for (int64_t c = 0; c < C; ++c) {
        int64_t s = 0;
        for (int t = 0; t < threads; ++t) s += part[t * C + c];
        out[c] = s;
    }
    free(part);
    return 0;
}
