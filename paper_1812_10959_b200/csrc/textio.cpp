// textio.cpp — the transaction text format (datasets.py:150-201): one
// transaction per line, whitespace-separated integer item ids, '#' comment
// lines and blank lines skipped, duplicates collapse (counted by the GPU
// encoder), a bad token raises ParseError / ItemOutOfRange naming its line.
//
// Host-side input tooling in front of the encoder: a multithreaded parser
// from a byte buffer to CSR, and the canonical writer (ascending ids, one
// line per row).  Semantics follow the reference's Python loop exactly for
// ASCII input: lines end at "\n", "\r\n" or "\r" (universal newlines);
// tokens are separated by the characters str.split() treats as whitespace
// (space, \t, \v, \f, \x1c-\x1f); a token is an int() literal: an optional
// sign, then digits with single underscores between them.  A buffer holding
// any byte >= 0x80 is reported back (kind 3) so the caller can take the
// Unicode-aware path.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dic_b200.h"
#include "csr.hpp"

namespace {

inline bool is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f); }
inline bool is_eol(unsigned char c) { return c == '\n' || c == '\r'; }

// int() of an ASCII token: 0 = ok (*big set when |value| >= 2^62), 1 = not an integer
int parse_int(const unsigned char* p, const unsigned char* q, int64_t* v, bool* big) {
    bool neg = false;
    if (p < q && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p == q || *p < '0' || *p > '9') return 1;
    int64_t x = 0;
    *big = false;
    bool prev_digit = false;
    for (; p < q; ++p) {
        const unsigned char c = *p;
        if (c >= '0' && c <= '9') {
            if (x > ((int64_t)1 << 58)) *big = true;
            else x = x * 10 + (c - '0');
            prev_digit = true;
        } else if (c == '_') {
            if (!prev_digit || p + 1 == q || p[1] < '0' || p[1] > '9') return 1;
            prev_digit = false;
        } else {
            return 1;
        }
    }
    *v = neg ? -x : x;
    return 0;
}

struct Chunk {
    std::vector<int64_t> lens;
    std::vector<int32_t> ids;
    int64_t lines = 0;
    int kind = 0;  // dic_parse_status.kind
    int64_t err_line = 0, err_off = 0, err_len = 0;
};

void parse_range(const unsigned char* buf, int64_t b, int64_t e, int32_t max_item, Chunk& c) {
    for (int64_t i = b; i < e && !c.kind;) {
        int64_t j = i;
        while (j < e && !is_eol(buf[j])) {
            if (buf[j] >= 0x80) {
                c.kind = 3;
                c.err_line = c.lines;
                return;
            }
            ++j;
        }
        // the line is [i, j)
        int64_t k = i;
        while (k < j && is_ws(buf[k])) ++k;
        if (k < j && buf[k] != '#') {
            int64_t count = 0;
            while (k < j) {
                int64_t t = k;
                while (t < j && !is_ws(buf[t])) ++t;
                int64_t v = 0;
                bool big = false;
                if (parse_int(buf + k, buf + t, &v, &big)) {
                    c.kind = 1;
                } else if (big || v < 0 || v >= max_item) {
                    c.kind = 2;
                }
                if (c.kind) {
                    c.err_line = c.lines;
                    c.err_off = k;
                    c.err_len = t - k;
                    return;
                }
                c.ids.push_back((int32_t)v);
                ++count;
                k = t;
                while (k < j && is_ws(buf[k])) ++k;
            }
            c.lens.push_back(count);
        }
        ++c.lines;
        if (j < e) j += (buf[j] == '\r' && j + 1 < e && buf[j + 1] == '\n') ? 2 : 1;
        i = j;
    }
}

// first position >= s that starts a line (just past a terminator), or len
int64_t line_start_after(const unsigned char* buf, int64_t len, int64_t s) {
    if (s <= 0) return 0;
    int64_t k = s;
    while (k < len && !is_eol(buf[k])) ++k;
    if (k >= len) return len;
    if (buf[k] == '\n' && k > 0 && buf[k - 1] == '\r' && k == s) return k + 1;  // s sat inside "\r\n"
    return (buf[k] == '\r' && k + 1 < len && buf[k + 1] == '\n') ? k + 2 : k + 1;
}

}  // namespace

extern "C" int dic_parse_transactions(const char* text, int64_t len, int32_t max_item, int32_t threads,
                                      dic_csr** out, dic_parse_status* st) {
    if (!out || !st || len < 0 || (len > 0 && !text) || max_item < 1) return DIC_EINVAL;
    *out = nullptr;
    memset(st, 0, sizeof(*st));
    const unsigned char* buf = reinterpret_cast<const unsigned char*>(text);
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, len / (1 << 20) + 1));
    std::vector<int64_t> cut(threads + 1);
    cut[0] = 0;
    for (int t = 1; t < threads; ++t) cut[t] = std::max(cut[t - 1], line_start_after(buf, len, len * t / threads));
    cut[threads] = len;
    std::vector<Chunk> ch(threads);
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back([&, t] { parse_range(buf, cut[t], cut[t + 1], max_item, ch[t]); });
    parse_range(buf, cut[0], cut[1], max_item, ch[0]);
    for (auto& th : pool) th.join();
    int64_t line0 = 0;
    for (int t = 0; t < threads; ++t) {
        if (ch[t].kind) {
            st->kind = ch[t].kind;
            st->line = line0 + ch[t].err_line + 1;  // 1-based, blank and comment lines included
            st->offset = ch[t].err_off;
            st->length = ch[t].err_len;
            return DIC_EDATA;
        }
        line0 += ch[t].lines;
    }
    dic_csr* c = new dic_csr();
    int64_t n = 0, nnz = 0;
    for (const Chunk& k : ch) {
        n += (int64_t)k.lens.size();
        nnz += (int64_t)k.ids.size();
    }
    c->n = n;
    c->indptr.resize(n + 1);
    c->indices.reserve(nnz);
    int64_t r = 0;
    c->indptr[0] = 0;
    for (const Chunk& k : ch) {
        for (int64_t L : k.lens) {
            c->indptr[r + 1] = c->indptr[r] + L;
            ++r;
        }
        c->indices.insert(c->indices.end(), k.ids.begin(), k.ids.end());
    }
    st->line = line0;
    *out = c;
    return DIC_OK;
}

// The canonical text form of rows [n][W] (save_transactions,
// datasets.py:196-209): ascending ids joined by single spaces, "\n" after
// every row (an empty row gives an empty line).
extern "C" int dic_format_transactions(const uint64_t* rows, int64_t n, int32_t W, int32_t threads, char** out,
                                       int64_t* len) {
    if (!rows || !out || !len || n < 0 || W < 1) return DIC_EINVAL;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n / 4096 + 1));
    std::vector<std::string> parts(threads);
    auto work = [&](int t) {
        std::string& s = parts[t];
        char tmp[8];
        for (int64_t r = n * t / threads; r < n * (t + 1) / threads; ++r) {
            bool first = true;
            for (int w = 0; w < W; ++w) {
                uint64_t x = rows[r * W + w];
                while (x) {
                    const int b = __builtin_ctzll(x);
                    x &= x - 1;
                    unsigned v = (unsigned)(w * 64 + b);
                    int k = 0;
                    do {
                        tmp[k++] = (char)('0' + v % 10);
                        v /= 10;
                    } while (v);
                    if (!first) s.push_back(' ');
                    first = false;
                    while (k) s.push_back(tmp[--k]);
                }
            }
            s.push_back('\n');
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    int64_t total = 0;
    for (const auto& p : parts) total += (int64_t)p.size();
    char* b = static_cast<char*>(malloc((size_t)std::max<int64_t>(total, 1)));
    if (!b) return DIC_ENOMEM;
    int64_t off = 0;
    for (const auto& p : parts) {
        memcpy(b + off, p.data(), p.size());
        off += (int64_t)p.size();
    }
    *out = b;
    *len = total;
    return DIC_OK;
}

extern "C" void dic_free_buffer(char* p) { free(p); }
