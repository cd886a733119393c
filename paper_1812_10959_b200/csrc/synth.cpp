// synth.cpp — seeded synthetic transaction generators for BASELINE.json's
// configs (host, multithreaded).  This is input tooling, not the hot path:
// the reference's own generator (datasets.py:75-142) is single-word and does
// not produce the configs' Zipf / Quest / Beta shapes, so these are new,
// written from the config text (see DESIGN.md §Inputs for the exact rules).
//
// Determinism: every row draws from its own counter-based stream
// (SplitMix64 keyed by seed, a per-generator tag and the GLOBAL row index),
// and shared structure (Quest patterns, Beta probabilities, planted groups)
// from a stream keyed by the seed alone.  Output is therefore identical for
// any thread count and for any split of the rows into ranges — which is what
// lets each rank of a sharded run generate only its own slices.
#include "csr.hpp"
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/dic_b200.h"

namespace {

inline uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct Rng {
    uint64_t s;
    explicit Rng(uint64_t key) : s(key) {}
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ull;
        return mix64(s);
    }
    // uniform in (0, 1)
    double uni() { return ((double)(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
};

Rng stream(uint64_t seed, uint64_t tag, int64_t row) {
    return Rng(mix64(mix64(seed ^ tag) + (uint64_t)(row + 1) * 0xD1B54A32D192ED03ull));
}

int poisson(Rng& r, double lam) {
    // inversion by sequential search; fine for the configs' means (<= 20)
    double u = r.uni();
    double p = exp(-lam), F = p;
    int k = 0;
    while (u > F && k < 100000) {
        ++k;
        p *= lam / k;
        F += p;
        if (p == 0.0) break;
    }
    return k;
}

double normal(Rng& r) {
    double u1 = r.uni(), u2 = r.uni();
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

// k distinct uniform items of [0, m), ascending (rejection; k << m here)
void distinct_items(Rng& r, int m, int k, std::vector<int32_t>& out) {
    out.clear();
    k = std::min(k, m);
    if (2 * k > m) {  // dense request: partial Fisher-Yates
        std::vector<int32_t> all(m);
        for (int i = 0; i < m; ++i) all[i] = i;
        for (int i = 0; i < k; ++i) {
            int j = i + (int)(r.next() % (uint64_t)(m - i));
            std::swap(all[i], all[j]);
            out.push_back(all[i]);
        }
    } else {
        while ((int)out.size() < k) {
            int32_t x = (int32_t)(r.next() % (uint64_t)m);
            if (std::find(out.begin(), out.end(), x) == out.end()) out.push_back(x);
        }
    }
    std::sort(out.begin(), out.end());
}

struct Ranges {
    std::vector<int64_t> begin, len, local0;  // local0 = first local row of range
    int64_t total = 0;
};

}  // namespace


namespace {

// Run gen(row, rng-free row generator) for every local row with `threads`
// workers; each worker fills private buffers then they are stitched in order.
template <class RowGen>
int run_rows(const Ranges& rg, int threads, RowGen gen, dic_csr** out) {
    const int64_t n = rg.total;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, std::max<int64_t>(1, n / 4096)));
    std::vector<std::vector<int32_t>> idx(threads);
    std::vector<std::vector<int64_t>> len(threads);
    auto work = [&](int t) {
        int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
        std::vector<int32_t> row;
        len[t].reserve(hi - lo);
        // locate range of lo
        size_t ri = 0;
        while (ri + 1 < rg.begin.size() && rg.local0[ri + 1] <= lo) ++ri;
        for (int64_t l = lo; l < hi; ++l) {
            while (ri + 1 < rg.begin.size() && rg.local0[ri + 1] <= l) ++ri;
            int64_t grow = rg.begin[ri] + (l - rg.local0[ri]);
            row.clear();
            gen(grow, row);
            len[t].push_back((int64_t)row.size());
            idx[t].insert(idx[t].end(), row.begin(), row.end());
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    dic_csr* c = new dic_csr();
    c->n = n;
    c->indptr.resize(n + 1);
    size_t nnz = 0;
    for (int t = 0; t < threads; ++t) nnz += idx[t].size();
    c->indices.reserve(nnz);
    int64_t r = 0;
    c->indptr[0] = 0;
    for (int t = 0; t < threads; ++t) {
        for (int64_t L : len[t]) {
            c->indptr[r + 1] = c->indptr[r] + L;
            ++r;
        }
        c->indices.insert(c->indices.end(), idx[t].begin(), idx[t].end());
    }
    *out = c;
    return DIC_OK;
}

int make_ranges(const int64_t* rb, const int64_t* rl, int nr, Ranges& rg) {
    if (nr < 0 || (nr > 0 && (!rb || !rl))) return DIC_EINVAL;
    int64_t acc = 0;
    for (int i = 0; i < nr; ++i) {
        if (rb[i] < 0 || rl[i] < 0) return DIC_EINVAL;
        if (rl[i] == 0) continue;
        rg.begin.push_back(rb[i]);
        rg.len.push_back(rl[i]);
        rg.local0.push_back(acc);
        acc += rl[i];
    }
    rg.total = acc;
    if (rg.begin.empty()) {  // keep the search loops well-defined
        rg.begin.push_back(0);
        rg.len.push_back(0);
        rg.local0.push_back(0);
    }
    return DIC_OK;
}

}  // namespace

extern "C" {

int dic_csr_info(const dic_csr* c, int64_t* n, int64_t* nnz) {
    if (!c) return DIC_EINVAL;
    if (n) *n = c->n;
    if (nnz) *nnz = (int64_t)c->indices.size();
    return DIC_OK;
}

int dic_csr_export(const dic_csr* c, int64_t* indptr, int32_t* indices) {
    if (!c || !indptr || (!indices && !c->indices.empty())) return DIC_EINVAL;
    memcpy(indptr, c->indptr.data(), c->indptr.size() * sizeof(int64_t));
    if (!c->indices.empty()) memcpy(indices, c->indices.data(), c->indices.size() * sizeof(int32_t));
    return DIC_OK;
}

void dic_csr_free(dic_csr* c) { delete c; }

// cfg1: L ~ Poisson(mean_len) clipped to [1, m]; L distinct items weighted
// by Zipf(s) over ids (w_i = (i+1)^-s), successive sampling without
// replacement via Gumbel-top-L.
int dic_synth_zipf(const int64_t* range_begin, const int64_t* range_len, int nranges, int32_t m, double s,
                   double mean_len, uint64_t seed, int threads, dic_csr** out) {
    if (!out || m < 1 || mean_len <= 0) return DIC_EINVAL;
    Ranges rg;
    if (make_ranges(range_begin, range_len, nranges, rg)) return DIC_EINVAL;
    std::vector<double> logw(m);
    for (int i = 0; i < m; ++i) logw[i] = -s * log((double)(i + 1));
    return run_rows(rg, threads, [&](int64_t row, std::vector<int32_t>& items) {
        Rng r = stream(seed, 0x7A697066ull, row);
        int L = std::min(std::max(poisson(r, mean_len), 1), m);
        std::vector<std::pair<double, int32_t>> keys(m);
        for (int i = 0; i < m; ++i) keys[i] = {logw[i] - log(-log(r.uni())), i};
        std::partial_sort(keys.begin(), keys.begin() + L, keys.end(),
                          [](const auto& a, const auto& b) { return a.first > b.first; });
        for (int i = 0; i < L; ++i) items.push_back(keys[i].second);
        std::sort(items.begin(), items.end());
    }, out);
}

// cfg2/cfg4: Quest-style.  n_patterns patterns, length ~ Poisson(pattern_len)
// clipped to [1, m], items uniform without replacement, weights ~ Exp(1)
// (normalised), corruption c ~ N(0.5, 0.1) clipped to [0, 1].  A transaction
// draws L ~ Poisson(mean_len) clipped to [1, m], then repeatedly picks a
// pattern by weight and adds each of its items independently with
// probability 1 - c, stopping as soon as |T| = L (the last pattern is
// truncated) or after 8L + 64 draws.
int dic_synth_quest(const int64_t* range_begin, const int64_t* range_len, int nranges, int32_t m,
                    int32_t n_patterns, double pattern_len, double mean_len, uint64_t seed, int threads,
                    dic_csr** out) {
    if (!out || m < 1 || n_patterns < 1 || mean_len <= 0 || pattern_len <= 0) return DIC_EINVAL;
    Ranges rg;
    if (make_ranges(range_begin, range_len, nranges, rg)) return DIC_EINVAL;
    Rng g(mix64(seed ^ 0x7175657374ull));
    std::vector<int64_t> pstart(n_patterns + 1, 0);
    std::vector<int32_t> pitems;
    std::vector<double> cum(n_patterns), corr(n_patterns);
    std::vector<int32_t> tmp;
    double tot = 0;
    for (int p = 0; p < n_patterns; ++p) {
        int len = std::min(std::max(poisson(g, pattern_len), 1), m);
        distinct_items(g, m, len, tmp);
        pitems.insert(pitems.end(), tmp.begin(), tmp.end());
        pstart[p + 1] = (int64_t)pitems.size();
        tot += -log(g.uni());
        cum[p] = tot;
        double c = 0.5 + 0.1 * normal(g);
        corr[p] = std::min(1.0, std::max(0.0, c));
    }
    for (int p = 0; p < n_patterns; ++p) cum[p] /= tot;
    cum[n_patterns - 1] = 1.0;
    return run_rows(rg, threads, [&](int64_t row, std::vector<int32_t>& items) {
        Rng r = stream(seed, 0x74786e73ull, row);
        int L = std::min(std::max(poisson(r, mean_len), 1), m);
        int draws = 8 * L + 64;
        while ((int)items.size() < L && draws-- > 0) {
            double u = r.uni();
            int p = (int)(std::lower_bound(cum.begin(), cum.end(), u) - cum.begin());
            if (p >= n_patterns) p = n_patterns - 1;
            double c = corr[p];
            for (int64_t q = pstart[p]; q < pstart[p + 1] && (int)items.size() < L; ++q) {
                if (r.uni() < c) continue;  // dropped by corruption
                int32_t it = pitems[q];
                if (std::find(items.begin(), items.end(), it) == items.end()) items.push_back(it);
            }
        }
        std::sort(items.begin(), items.end());
    }, out);
}

// cfg3: item j present independently with p_j ~ Beta(2, 5) (the 2nd
// smallest of 6 uniforms), then `groups` planted groups of `group_size`
// distinct items, each OR-ed into a row independently with probability
// group_p.
int dic_synth_dense(const int64_t* range_begin, const int64_t* range_len, int nranges, int32_t m,
                    int32_t groups, int32_t group_size, double group_p, uint64_t seed, int threads,
                    dic_csr** out) {
    if (!out || m < 1 || groups < 0 || group_size < 1 || group_size > m) return DIC_EINVAL;
    Ranges rg;
    if (make_ranges(range_begin, range_len, nranges, rg)) return DIC_EINVAL;
    Rng g(mix64(seed ^ 0x64656e7365ull));
    std::vector<double> pj(m);
    for (int j = 0; j < m; ++j) {
        double u[6];
        for (double& x : u) x = g.uni();
        std::sort(u, u + 6);
        pj[j] = u[1];
    }
    std::vector<std::vector<int32_t>> grp(groups);
    for (int q = 0; q < groups; ++q) distinct_items(g, m, group_size, grp[q]);
    return run_rows(rg, threads, [&](int64_t row, std::vector<int32_t>& items) {
        Rng r = stream(seed, 0x726f7773ull, row);
        std::vector<uint8_t> on(m, 0);
        for (int j = 0; j < m; ++j) on[j] = r.uni() < pj[j];
        for (int q = 0; q < groups; ++q)
            if (r.uni() < group_p)
                for (int32_t it : grp[q]) on[it] = 1;
        for (int j = 0; j < m; ++j)
            if (on[j]) items.push_back(j);
    }, out);
}

// cfg5 candidates: k ~ U{kmin..kmax}, items uniform without replacement.
int dic_synth_candidates(int64_t C, int32_t m, int32_t kmin, int32_t kmax, uint64_t seed, int32_t* cand_k,
                         uint16_t* cand_items) {
    if (C < 0 || m < 1 || m > 65535 || kmin < 1 || kmax < kmin || kmax > m || !cand_k || !cand_items)
        return DIC_EINVAL;
    std::vector<int32_t> tmp;
    for (int64_t c = 0; c < C; ++c) {
        Rng r = stream(seed, 0x63616e64ull, c);
        int k = kmin + (int)(r.next() % (uint64_t)(kmax - kmin + 1));
        distinct_items(r, m, k, tmp);
        cand_k[c] = k;
        for (int j = 0; j < kmax; ++j) cand_items[c * kmax + j] = j < k ? (uint16_t)tmp[j] : (uint16_t)0xFFFF;
    }
    return DIC_OK;
}

}  // extern "C"
