/*
 * dic_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C CPU restatement of the
 * reference `dicmine` DIC engine, generalised from one uint64 word to W words
 * per mask exactly as SURVEY.md §8(c) route 2 does (the reference's own
 * logic is width-agnostic over Python ints).  Only tests/, the smoke() check
 * and bench.py's cpu_baseline / --impl reference leg may load this; the
 * product path (paper_1812_10959_b200) never does.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, run where /root/reference exists) — see
 * tests/test_oracle_golden.py.
 *
 * Function-by-function citations (paths under /root/reference/pkg/src/dicmine):
 *   orc_count_block   _count_block          engine.py:43-58   (and _count_block_python :61-67)
 *   orc_count_many    _count_partitioned_by_itemset engine.py:226-245 (threads own
 *                     disjoint candidate slices)
 *   orc_item_support  first_pass counting   engine.py:132-154
 *   orc_mine          _run                  engine.py:398-458 with
 *                       first_pass          engine.py:105-173
 *                       count_support_interval engine.py:176-223
 *                       prune               engine.py:273-317
 *                       make_candidates     engine.py:320-369 (+ immediate_subsets bitops.py:63-69)
 *                       check_full_pass     engine.py:372-390
 *                     catalog semantics     itemsets.py:88-136
 *                     chunk_bounds          params.py:67-75
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ count */

/* rows [n][W]; mask has W words; only its non-zero words constrain */
int64_t orc_count_block(const uint64_t* rows, int W, int64_t first, int64_t last, const uint64_t* mask) {
    int nz[4096];
    int nnz = 0;
    for (int w = 0; w < W && nnz < 4096; ++w)
        if (mask[w]) nz[nnz++] = w;
    int64_t total = 0;
    for (int64_t j = first; j <= last; ++j) {
        const uint64_t* t = rows + j * (int64_t)W;
        int ok = 1;
        for (int q = 0; q < nnz; ++q) {
            uint64_t m = mask[nz[q]];
            if ((t[nz[q]] & m) != m) { ok = 0; break; }
        }
        total += ok;
    }
    return total;
}

typedef struct {
    const uint64_t* rows;
    int W;
    int64_t first, last;
    const uint64_t* masks;
    int64_t c0, c1;
    int64_t* out;
} count_job;

static void* count_worker(void* arg) {
    count_job* j = (count_job*)arg;
    for (int64_t c = j->c0; c < j->c1; ++c)
        j->out[c] += orc_count_block(j->rows, j->W, j->first, j->last, j->masks + c * (int64_t)j->W);
    return NULL;
}

/* out[c] += count of masks[c] over [first, last]; threads own disjoint
 * candidate slices (the reference's itemset-partitioned mode). */
void orc_count_many(const uint64_t* rows, int W, int64_t first, int64_t last, const uint64_t* masks, int64_t C,
                    int64_t* out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (C < threads) threads = (int)(C > 0 ? C : 1);
    pthread_t th[256];
    count_job jobs[256];
    int64_t step = (C + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (count_job){rows, W, first, last, masks, t * step, (t + 1) * step < C ? (t + 1) * step : C, out};
        if (jobs[t].c0 > jobs[t].c1) jobs[t].c0 = jobs[t].c1;
        if (t > 0) pthread_create(&th[t], NULL, count_worker, &jobs[t]);
    }
    count_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
}

void orc_item_support(const uint64_t* rows, int64_t n, int W, int m, int64_t* counts) {
    for (int i = 0; i < m; ++i) counts[i] = 0;
    for (int64_t j = 0; j < n; ++j) {
        const uint64_t* t = rows + j * (int64_t)W;
        for (int w = 0; w < W; ++w) {
            uint64_t x = t[w];
            while (x) {
                int b = __builtin_ctzll(x);
                x &= x - 1;
                int it = w * 64 + b;
                if (it < m) counts[it]++;
            }
        }
    }
}

/* --------------------------------------------------------------- catalog */

enum { DC = 0, DB = 1, SC = 2, SB = 3, NILS = 4 };
static int is_box(int s) { return s == DB || s == SB; }
static int is_dashed(int s) { return s == DC || s == DB; }

typedef struct {
    int W;
    int64_t n, cap;
    uint64_t* mask;      /* [cap][W] */
    int32_t* size;
    int64_t* support;
    int64_t* intervals;
    uint8_t* shape;
    /* known: open addressing mask -> record */
    int64_t* ht;
    int64_t hcap;
} catalog;

static uint64_t mix(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static uint64_t hash_mask(const uint64_t* m, int W) {
    uint64_t h = 0x1234567ull;
    for (int w = 0; w < W; ++w) h = mix(h ^ (m[w] + 0x9E3779B97F4A7C15ull * (uint64_t)(w + 1)));
    return h;
}

static int64_t cat_find(const catalog* c, const uint64_t* m) {
    uint64_t s = hash_mask(m, c->W) & (uint64_t)(c->hcap - 1);
    for (;;) {
        int64_t e = c->ht[s];
        if (e < 0) return -1;
        if (memcmp(c->mask + e * c->W, m, (size_t)c->W * 8) == 0) return e;
        s = (s + 1) & (uint64_t)(c->hcap - 1);
    }
}

static void cat_index(catalog* c, int64_t r) {
    uint64_t s = hash_mask(c->mask + r * c->W, c->W) & (uint64_t)(c->hcap - 1);
    while (c->ht[s] >= 0) s = (s + 1) & (uint64_t)(c->hcap - 1);
    c->ht[s] = r;
}

static int cat_reserve(catalog* c, int64_t need) {
    if (need > c->cap) {
        int64_t nc = c->cap ? c->cap : 1024;
        while (nc < need) nc *= 2;
        c->mask = realloc(c->mask, (size_t)nc * c->W * 8);
        c->size = realloc(c->size, (size_t)nc * 4);
        c->support = realloc(c->support, (size_t)nc * 8);
        c->intervals = realloc(c->intervals, (size_t)nc * 8);
        c->shape = realloc(c->shape, (size_t)nc);
        if (!c->mask || !c->size || !c->support || !c->intervals || !c->shape) return -1;
        c->cap = nc;
    }
    if (need * 2 > c->hcap) {
        int64_t nh = c->hcap ? c->hcap : 2048;
        while (nh < need * 2) nh *= 2;
        free(c->ht);
        c->ht = malloc((size_t)nh * 8);
        if (!c->ht) return -1;
        for (int64_t i = 0; i < nh; ++i) c->ht[i] = -1;
        c->hcap = nh;
        for (int64_t r = 0; r < c->n; ++r) cat_index(c, r);
    }
    return 0;
}

/* CountedItemset.fresh + known[mask] = item (itemsets.py:80-85, 116-123) */
static int64_t cat_add(catalog* c, const uint64_t* m) {
    if (cat_reserve(c, c->n + 1)) return -1;
    int64_t r = c->n++;
    memcpy(c->mask + r * c->W, m, (size_t)c->W * 8);
    int sz = 0;
    for (int w = 0; w < c->W; ++w) sz += __builtin_popcountll(m[w]);
    c->size[r] = sz;
    c->support[r] = 0;
    c->intervals[r] = 0;
    c->shape[r] = DC;
    cat_index(c, r);
    return r;
}

typedef struct {
    int64_t* v;
    int64_t n, cap;
} ivec;

static int iv_push(ivec* a, int64_t x) {
    if (a->n == a->cap) {
        int64_t nc = a->cap ? a->cap * 2 : 256;
        int64_t* p = realloc(a->v, (size_t)nc * 8);
        if (!p) return -1;
        a->v = p;
        a->cap = nc;
    }
    a->v[a->n++] = x;
    return 0;
}

/* MSW-first numeric compare of two W-word masks (Python-int order). */
static int cmp_mask(const uint64_t* a, const uint64_t* b, int W) {
    for (int w = W - 1; w >= 0; --w)
        if (a[w] != b[w]) return a[w] < b[w] ? -1 : 1;
    return 0;
}

static const catalog* g_sort_cat;
static int cmp_rec(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    const catalog* c = g_sort_cat;
    if (c->size[a] != c->size[b]) return c->size[a] < c->size[b] ? -1 : 1;
    return cmp_mask(c->mask + a * c->W, c->mask + b * c->W, c->W);
}

typedef struct {
    int64_t scanned;
    int64_t peak_dashed, candidates_generated, candidates_pruned, interval_counts;
    int64_t stops;
} orc_stats;

typedef struct {
    catalog cat;
    int64_t* frequent;  /* record ids, sorted */
    int64_t nfreq;
} orc_result;

/*
 * The whole run.  need = ceil(minsup * n) computed by the caller exactly as
 * params.py:17-19 does; interval = M; stop_max = ceil(n / M) (params.py:57).
 * max_stops < 0 = run to completion; otherwise stop after that many
 * checkpoints (bounded CPU-baseline samples).  Returns a handle, NULL on OOM.
 */
void* orc_mine(const uint64_t* rows, int64_t n, int W, int m, int64_t need, int64_t interval, int prune_bound,
               int threads, int64_t max_stops, orc_stats* st) {
    orc_result* res = calloc(1, sizeof(orc_result));
    if (!res) return NULL;
    catalog* c = &res->cat;
    c->W = W;
    memset(st, 0, sizeof(*st));
    const int64_t stop_max = (n + interval - 1) / interval;
    ivec dashed = {0}, solid = {0}, promoted = {0}, level1 = {0};
    uint64_t* tmp = calloc((size_t)W, 8);
    uint64_t* sub = calloc((size_t)W, 8);
    int64_t* counts = malloc((size_t)(m > 0 ? m : 1) * 8);
    /* ---- first_pass (engine.py:105-173) */
    orc_item_support(rows, n, W, m, counts);
    for (int i = 0; i < m; ++i) {
        memset(tmp, 0, (size_t)W * 8);
        tmp[i >> 6] = 1ull << (i & 63);
        int64_t r = cat_add(c, tmp); /* register (singles are not in dashed) */
        c->support[r] = counts[i];
        c->intervals[r] = stop_max;
        c->shape[r] = counts[i] >= need ? SB : SC;
        iv_push(&solid, r);
        if (c->shape[r] == SB) iv_push(&level1, i);
    }
    for (int64_t a = 0; a < level1.n; ++a)
        for (int64_t b = a + 1; b < level1.n; ++b) {
            memset(tmp, 0, (size_t)W * 8);
            tmp[level1.v[a] >> 6] |= 1ull << (level1.v[a] & 63);
            tmp[level1.v[b] >> 6] |= 1ull << (level1.v[b] & 63);
            iv_push(&dashed, cat_add(c, tmp));
        }
    st->candidates_generated += dashed.n;
    if (dashed.n > st->peak_dashed) st->peak_dashed = dashed.n;
    st->scanned += n;

    uint64_t* cmasks = NULL;
    int64_t* cinc = NULL;
    int64_t ccap = 0;
    int64_t stop = 0;
    while (dashed.n > 0 && (max_stops < 0 || st->stops < max_stops)) {
        ++stop;
        if (stop > stop_max) stop = 1;
        int64_t first = (stop - 1) * interval;
        int64_t last = (stop * interval < n ? stop * interval : n) - 1;
        st->interval_counts += dashed.n;
        /* ---- count_support_interval */
        if (dashed.n > ccap) {
            ccap = dashed.n * 2;
            cmasks = realloc(cmasks, (size_t)ccap * W * 8);
            cinc = realloc(cinc, (size_t)ccap * 8);
        }
        for (int64_t q = 0; q < dashed.n; ++q) {
            memcpy(cmasks + q * W, c->mask + dashed.v[q] * W, (size_t)W * 8);
            cinc[q] = 0;
        }
        orc_count_many(rows, W, first, last, cmasks, dashed.n, cinc, threads);
        for (int64_t q = 0; q < dashed.n; ++q) {
            c->support[dashed.v[q]] += cinc[q];
            c->intervals[dashed.v[q]] += 1;
        }
        st->scanned += last - first + 1;
        /* ---- prune */
        promoted.n = 0;
        for (int64_t q = 0; q < dashed.n; ++q) {
            int64_t r = dashed.v[q];
            if (c->shape[r] != DC) continue;
            if (c->support[r] >= need) {
                c->shape[r] = DB;
                iv_push(&promoted, r);
            } else if (prune_bound && c->intervals[r] < stop_max) {
                int64_t remaining = stop_max - c->intervals[r];
                int64_t ceiling = c->support[r] + interval * remaining;
                if (ceiling < need) {
                    c->shape[r] = NILS;
                    st->candidates_pruned++;
                    const uint64_t* im = c->mask + r * W;
                    for (int64_t o = 0; o < dashed.n; ++o) {
                        int64_t ro = dashed.v[o];
                        if (c->shape[ro] != DC) continue;
                        const uint64_t* om = c->mask + ro * W;
                        int sup = 1;
                        for (int w = 0; w < W; ++w)
                            if ((im[w] & om[w]) != im[w]) { sup = 0; break; }
                        if (sup) {
                            c->shape[ro] = NILS;
                            st->candidates_pruned++;
                        }
                    }
                }
            }
        }
        {
            int64_t k = 0;
            for (int64_t q = 0; q < dashed.n; ++q)
                if (is_dashed(c->shape[dashed.v[q]])) dashed.v[k++] = dashed.v[q];
            dashed.n = k;
        }
        /* ---- make_candidates(frontier = promoted, level1) */
        int64_t inserted = 0;
        for (int64_t f = 0; f < promoted.n; ++f) {
            int64_t src = promoted.v[f];
            if (!is_box(c->shape[src])) continue;
            for (int64_t l = 0; l < level1.n; ++l) {
                int it = (int)level1.v[l];
                /* c->mask may move in cat_add: re-read src each time */
                memcpy(tmp, c->mask + src * W, (size_t)W * 8);
                if ((tmp[it >> 6] >> (it & 63)) & 1ull) continue; /* cand == base */
                tmp[it >> 6] |= 1ull << (it & 63);
                if (cat_find(c, tmp) >= 0) continue;
                int ok = 1;
                for (int w = 0; w < W && ok; ++w) {
                    uint64_t x = tmp[w];
                    while (x && ok) {
                        int b = __builtin_ctzll(x);
                        x &= x - 1;
                        memcpy(sub, tmp, (size_t)W * 8);
                        sub[w] ^= 1ull << b;
                        int64_t e = cat_find(c, sub);
                        if (e < 0 || !is_box(c->shape[e])) ok = 0;
                    }
                }
                if (ok) {
                    iv_push(&dashed, cat_add(c, tmp));
                    inserted++;
                }
            }
        }
        st->candidates_generated += inserted;
        if (dashed.n > st->peak_dashed) st->peak_dashed = dashed.n;
        /* ---- check_full_pass */
        {
            int64_t k = 0;
            for (int64_t q = 0; q < dashed.n; ++q) {
                int64_t r = dashed.v[q];
                if (is_dashed(c->shape[r]) && c->intervals[r] == stop_max) {
                    c->shape[r] = c->support[r] >= need ? SB : SC;
                    iv_push(&solid, r);
                } else {
                    dashed.v[k++] = r;
                }
            }
            dashed.n = k;
        }
        st->stops++;
    }
    /* ---- frequent = SOLID_BOX sorted by (size, mask) */
    int64_t nf = 0;
    for (int64_t q = 0; q < solid.n; ++q)
        if (c->shape[solid.v[q]] == SB) nf++;
    res->frequent = malloc((size_t)(nf > 0 ? nf : 1) * 8);
    nf = 0;
    for (int64_t q = 0; q < solid.n; ++q)
        if (c->shape[solid.v[q]] == SB) res->frequent[nf++] = solid.v[q];
    res->nfreq = nf;
    g_sort_cat = c;
    qsort(res->frequent, (size_t)nf, sizeof(int64_t), cmp_rec);
    free(tmp); free(sub); free(counts); free(cmasks); free(cinc);
    free(dashed.v); free(solid.v); free(promoted.v); free(level1.v);
    return res;
}

int64_t orc_result_count(void* h) { return ((orc_result*)h)->nfreq; }

void orc_result_get(void* h, uint64_t* masks, int32_t* sizes, int64_t* supports) {
    orc_result* r = (orc_result*)h;
    const catalog* c = &r->cat;
    for (int64_t i = 0; i < r->nfreq; ++i) {
        int64_t id = r->frequent[i];
        memcpy(masks + i * c->W, c->mask + id * c->W, (size_t)c->W * 8);
        sizes[i] = c->size[id];
        supports[i] = c->support[id];
    }
}

void orc_result_free(void* h) {
    orc_result* r = (orc_result*)h;
    if (!r) return;
    catalog* c = &r->cat;
    free(c->mask); free(c->size); free(c->support); free(c->intervals); free(c->shape); free(c->ht);
    free(r->frequent);
    free(r);
}
