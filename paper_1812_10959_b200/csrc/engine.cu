// engine.cu — the device-resident DIC checkpoint state machine.
//
// Reference: _run (engine.py:398-458) drives, per stop,
//   count_support_interval (:176-223) -> prune (:273-317) ->
//   make_candidates (:320-369) -> peak_dashed (:440) -> check_full_pass (:372-390)
// over an ItemsetCatalog of Python objects (itemsets.py:88-136).  Here the
// catalog lives on the device:
//
//   records   every itemset ever created (= the reference's `known` dict,
//             itemsets.py:97-99): mask[W], Zobrist hash, size, support,
//             intervals_counted, shape.  Append-only; record id = index.
//   ht        open-addressing hash index mask -> record id (linear probing,
//             load <= 1/2), keyed by the Zobrist hash XOR_{p in mask} z(p)
//             so subset / superset hashes are one XOR away.
//   buckets   the dashed vector split by itemset size k: record ids plus
//             the k ascending item ids of each candidate (the count kernel's
//             input).  Order-preserving compaction mirrors compact_dashed
//             (itemsets.py:130-132).
//   frontier  record ids promoted to DASHED_BOX at this stop (prune's return).
//
// Pipelined stops.  Every kernel of a stop reads its sizes from device
// memory (bucket fill, delta offsets, frontier size), so the host enqueues
// stop s without knowing the outcome of stop s-1: it processes the status of
// stop s-D (copied into a pinned ring) while the GPU runs stops s-D+1..s.
// Capacities are checked on the device; a stop whose candidate step would
// overflow sets an abort flag that turns every later kernel into a no-op,
// and the host (at the poll of that stop) grows the arrays, replays the
// candidate step and re-issues the aborted stops.  Slots that leave the
// dashed vector stay in their bucket as dead entries (skipped by the apply
// kernel) until the host schedules that bucket's compaction.
//
// Phase fusion (exactness argued in DESIGN.md §4): check_full_pass runs in
// the same kernel as prune because finalisation never changes box-ness
// (DASHED_BOX->SOLID_BOX, DASHED_CIRCLE->SOLID_CIRCLE) and freshly inserted
// candidates have intervals_counted == 0 < stop_max, so make_candidates sees
// the same admissions and check_full_pass the same records either way.
// prune's superset-NIL loop (:311-315) is provably dead in the engine (a
// dashed circle's proper subsets are boxes, and boxes never revert), so the
// engine omits it; the API-level prune on host catalogs keeps it.
#include "common.cuh"

#include <map>
#include <nccl.h>
#include <nccl_device.h>  // NCCL >= 2.28 device API: symmetric windows, LSA barriers

#include <algorithm>
#include <chrono>
#include <deque>
#include <mutex>
#include <numeric>
#include <vector>

namespace dic {

constexpr int kFusedCtas = 256;     // CTAs (and LSA barriers) of the fused per-stop reduction
constexpr int kFusedMaxPeers = 72;  // LSA team size it supports (one NVLink domain)

int count_dev_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last, int kuse,
                     uint16_t* const* items_tab, const unsigned long long* bn, const int64_t* doff,
                     unsigned long long* delta, const unsigned long long* abort_flag, int64_t tri_len,
                     cudaStream_t s, const int64_t* chunk_ring, const unsigned long long* seq, int ring,
                     int batch = 1, int64_t batch_stride = 0);
int item_support_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                        unsigned long long* counts, cudaStream_t s);
int count_pairs_dev_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                           unsigned long long* tri, const unsigned long long* bn2, int64_t tri_len,
                           const unsigned long long* abort_flag, cudaStream_t s, const int64_t* chunk_ring,
                           const unsigned long long* seq, int ring, unsigned long long* sched);
int tids_select_launch(const uint32_t* src, int64_t n, int m, const int32_t* items, int L, uint32_t* dst,
                       cudaStream_t s);

enum : uint8_t { DASHED_CIRCLE = 0, DASHED_BOX = 1, SOLID_CIRCLE = 2, SOLID_BOX = 3, NIL = 4 };

__host__ __device__ inline bool is_box(uint8_t s) { return s == DASHED_BOX || s == SOLID_BOX; }
__host__ __device__ inline bool is_dashed(uint8_t s) { return s == DASHED_CIRCLE || s == DASHED_BOX; }

__host__ __device__ inline uint64_t zob(uint32_t item) {
    return mix64(0x5A0B1157ull + (uint64_t)item * 0x9E3779B97F4A7C15ull);
}

// Hash-index entries, one 64-bit word each, so a probe reads one word and only
// a tag match touches a record:
//   record     bit 63 = 0 | 31-bit tag (bits 32.. of the mask's hash) | record id
//   temporary  bit 63 = 1 | joined item l (16) | source record (31) | 16 tag bits
//              a join of the current stop, cand = source's itemset + {l}, not
//              yet a record (checkpoint kernel); self-describing, so a thread
//              that meets it needs nothing but the records of earlier stops
//   empty      all ones (no temporary entry looks like it: record ids stay
//              far below 2^31 - 1)
typedef unsigned long long hent_t;
constexpr hent_t kEmptyEnt = ~0ull;
__host__ __device__ __forceinline__ uint32_t htag(uint64_t h) { return (uint32_t)(h >> 32) & 0x7FFFFFFFu; }
__host__ __device__ __forceinline__ hent_t hent(uint64_t h, int32_t id) {
    return ((hent_t)htag(h) << 32) | (uint32_t)id;
}
__host__ __device__ __forceinline__ int32_t hent_id(hent_t x) { return (int32_t)(uint32_t)x; }
__host__ __device__ __forceinline__ uint32_t hent_tag(hent_t x) { return (uint32_t)(x >> 32); }
__host__ __device__ __forceinline__ bool hent_temp(hent_t x) { return (x >> 63) != 0; }  // (after the empty test)
__host__ __device__ __forceinline__ hent_t hent_join(uint64_t h, int32_t src, int l) {
    return (1ull << 63) | ((hent_t)(uint32_t)l << 47) | ((hent_t)(uint32_t)src << 16) | ((h >> 32) & 0xFFFFull);
}
__host__ __device__ __forceinline__ int32_t hent_join_src(hent_t x) { return (int32_t)((x >> 16) & 0x7FFFFFFFull); }
__host__ __device__ __forceinline__ int hent_join_item(hent_t x) { return (int)((x >> 47) & 0xFFFFull); }

// Status words (device, one contiguous u64 array).
enum : int {
    S_NFRONT = 0,    // promoted DASHED_CIRCLE -> DASHED_BOX
    S_NPRUNED = 1,   // DASHED_CIRCLE -> NIL by the bound
    S_NFINAL = 2,    // dashed -> solid
    S_SURV = 3,      // live dashed entries after prune (before finalisation)
    S_NADM = 4,      // admissible joins (before dedup)
    S_NINS = 5,      // distinct new candidates committed
    S_OVERFLOW = 6,  // this stop's candidate step did not fit (not applied)
    S_NREC = 7,      // records (persistent)
    S_ABORT = 8,     // persistent: set with OVERFLOW, cleared by the host's replay
    S_SCRATCH = 9,   // scratch word (result collection)
    S_DONE = 10,     // (unused)
    S_SEQ = 11,      // persistent: stops completed (the status kernel advances it)
    S_HEAD = 12
};
constexpr int kDoffMax = 256;  // delta offsets kept for sizes < 256
constexpr int kRing = 16;      // status ring slots (> max stops in flight)
// followed by: removed[KS] (dead slots this stop), adm[KS] (admitted joins by
// size), bn[KS] (bucket fill, persistent), cflag[KS] (compact bucket k at the
// next stop), KS = m + 2.  The first S_HEAD + 3*KS words are the status
// snapshot copied to the host ring.

struct Records {
    unsigned long long* mask = nullptr;  // [cap][W]
    uint64_t* hash = nullptr;
    int64_t* support = nullptr;
    int64_t* intervals = nullptr;
    int32_t* size = nullptr;
    uint8_t* shape = nullptr;
    uint16_t* items = nullptr;  // [cap][8] ascending item ids of itemsets of <= 8 items (zero padded)
    int64_t cap = 0;
};

// L2 load (words other CTAs update during a kernel: the L1 copy may be stale)
__device__ __forceinline__ unsigned long long ldv(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Mask view: words of src with bit `add` set and bit `drop` cleared (-1 = none).
struct MaskView {
    const unsigned long long* src;
    int add, drop;
    __device__ __forceinline__ unsigned long long word(int w) const {
        unsigned long long x = src[w];
        if (add >= 0 && w == (add >> 6)) x |= 1ull << (add & 63);
        if (drop >= 0 && w == (drop >> 6)) x &= ~(1ull << (drop & 63));
        return x;
    }
};

__device__ __forceinline__ bool mask_eq(const unsigned long long* a, const MaskView& v, int W) {
    for (int w = 0; w < W; ++w)
        if (a[w] != v.word(w)) return false;
    return true;
}

__device__ __forceinline__ int32_t ht_lookup(const hent_t* __restrict__ ht, uint64_t hmask, const Records& R,
                                             int W, uint64_t h, const MaskView& v) {
    uint64_t slot = mix64(h) & hmask;
    const uint32_t tag = htag(h);
    while (true) {
        const hent_t x = ht[slot];
        const int32_t e = hent_id(x);
        if (x == kEmptyEnt) return -1;
        // (a temporary entry — an unpublished join of this stop, never a record — has bit 63 set: no tag match)
        if (hent_tag(x) == tag && mask_eq(R.mask + (int64_t)e * W, v, W)) return e;
        slot = (slot + 1) & hmask;
    }
}

// Lookup of the set its[0..k) + {add} - {drop} (add/drop = -1: none) of
// `size` items.  A tag match is confirmed without reading the whole W-word
// mask: a record of the same size holding every item of the set IS the set.
// The per-item bit loads are independent, so a confirmation costs one memory
// latency instead of W dependent word compares.
__device__ __forceinline__ int32_t ht_find_items(const hent_t* __restrict__ ht, uint64_t hmask, const Records& R,
                                                 int W, uint64_t h, const int* its, int k, int add, int drop,
                                                 int size) {
    uint64_t slot = mix64(h) & hmask;
    const uint32_t tag = htag(h);
    while (true) {
        const hent_t x = ht[slot];
        const int32_t e = hent_id(x);
        if (x == kEmptyEnt) return -1;
        if (hent_tag(x) == tag && R.size[e] == size) {
            const unsigned long long* rm = R.mask + (int64_t)e * W;
            bool ok = add < 0 || ((rm[add >> 6] >> (add & 63)) & 1ull);
            for (int q = 0; q < k; ++q) {
                const int it = its[q];
                if (it != drop) ok &= ((rm[it >> 6] >> (it & 63)) & 1ull) != 0;
            }
            if (ok) return e;
        }
        slot = (slot + 1) & hmask;
    }
}

// ---------------------------------------------------------------------------
// seeding / rehash
// ---------------------------------------------------------------------------
__global__ void ht_clear_kernel(hent_t* ht, int64_t cap) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
        ht[i] = kEmptyEnt;
}

// Insert records [0, *nrec) — the device count, so a rebuild enqueued behind
// in-flight stops sees their records too.
__global__ void ht_insert_records_kernel(hent_t* ht, uint64_t hmask, Records R, const unsigned long long* nrec) {
    const int64_t n = (int64_t)*nrec;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = R.hash[r];
        uint64_t slot = mix64(h) & hmask;
        while (atomicCAS(ht + slot, kEmptyEnt, hent(h, (int32_t)r)) != kEmptyEnt) slot = (slot + 1) & hmask;
    }
}

// Singletons: record i = item i (first_pass, engine.py:125-163).
__global__ void seed_singletons_kernel(Records R, int W, int m, const int64_t* __restrict__ counts, int64_t need,
                                       int64_t stop_max) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    for (int w = 0; w < W; ++w) R.mask[(int64_t)i * W + w] = (w == (i >> 6)) ? (1ull << (i & 63)) : 0ull;
    R.hash[i] = zob((uint32_t)i);
    for (int q = 0; q < 8; ++q) R.items[(int64_t)i * 8 + q] = q == 0 ? (uint16_t)i : (uint16_t)0;
    R.size[i] = 1;
    R.support[i] = counts[i];
    R.intervals[i] = stop_max;
    R.shape[i] = counts[i] >= need ? SOLID_BOX : SOLID_CIRCLE;
}

// Every pair (level1[a], level1[b]), a < b, in the reference's nested-loop
// order (engine.py:165-168): pair index p enumerates a-major.
__global__ void seed_pairs_kernel(Records R, int W, const int32_t* __restrict__ level1, int64_t L,
                                  const int64_t* __restrict__ row_start, int64_t npairs, int64_t rec0,
                                  int32_t* __restrict__ b_rec, uint16_t* __restrict__ b_items) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npairs) return;
    int64_t lo = 0, hi = L - 2;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (row_start[mid] <= p) lo = mid; else hi = mid - 1;
    }
    int64_t a = lo, b = a + 1 + (p - row_start[a]);
    int ia = level1[a], ib = level1[b];
    int64_t r = rec0 + p;
    for (int w = 0; w < W; ++w) {
        unsigned long long x = 0;
        if (w == (ia >> 6)) x |= 1ull << (ia & 63);
        if (w == (ib >> 6)) x |= 1ull << (ib & 63);
        R.mask[r * W + w] = x;
    }
    R.hash[r] = zob(ia) ^ zob(ib);
    *reinterpret_cast<uint4*>(R.items + r * 8) = make_uint4((uint32_t)ia | ((uint32_t)ib << 16), 0u, 0u, 0u);
    R.size[r] = 2;
    R.support[r] = 0;
    R.intervals[r] = 0;
    R.shape[r] = DASHED_CIRCLE;
    b_rec[p] = (int32_t)r;
    b_items[2 * p] = (uint16_t)ia;
    b_items[2 * p + 1] = (uint16_t)ib;
}

// ---------------------------------------------------------------------------
// per stop: ONE persistent cooperative kernel runs the whole checkpoint half
// ---------------------------------------------------------------------------
// count_support_interval's "support += delta" and everything _run does after
// it at a stop (engine.py:430-441: prune, make_candidates, peak_dashed,
// check_full_pass) as the phases of one kernel, one CTA per SM, separated by
// grid-wide barriers instead of kernel boundaries:
//
//   P1  apply      support += delta, intervals += 1, prune, check_full_pass,
//                  keep flags, frontier (every CTA, grid-stride over the slots)
//   --- barrier ---
//   P2  compaction of the buckets the last status flagged (CTA k = bucket k)
//       evaluation of the frontier x level1 joins (every CTA, after its bucket)
//   --- barrier ---  (nothing promoted: straight to the status)
//   P3  all-or-nothing capacity check (every CTA, same inputs, same verdict),
//       dedup: one owner per distinct admitted mask
//   --- barrier ---
//   P4  canonical commit: one warp per new candidate ranks it and writes it
//   last CTA out   bucket sizes after the commit, the stop's status snapshot
//
// Five kernel launches per stop became one: what is left of a phase is its
// dependent-load chain (a few microseconds) plus ~1 us per barrier.  The
// overflow replay (dic_engine_poll) runs the same kernel from P2's join
// evaluation on (replay = 1).
struct PairArgs {  // the dense pair triangle (tri == nullptr: none)
    unsigned long long* tri;
    const int32_t* rank;
    int64_t L, tri_len;
    int64_t rec0;  // record id of seeded pair 0: pair p = record rec0 + p = triangle slot p
};

__device__ __forceinline__ int64_t tri_pos(int64_t a, int64_t b, int64_t L) {
    return a * L - a * (a + 1) / 2 + (b - a - 1);
}

struct JoinRec;

constexpr int kCkptThreads = 1024;    // one CTA per SM
constexpr int kCompactItems = 16384;  // staged item ids per compaction chunk (32 KB)

// Buffers written by one phase and read by a later one are reached through
// plain (not __restrict__ const) pointers: loads must stay coherent across the
// grid barriers, which the non-coherent read-only path is not.
struct CkptArgs {
    int32_t* const* rec_tab;      // per-size bucket tables
    uint16_t* const* items_tab;
    const int64_t* bcap;
    int64_t* doff;                // per-size delta offsets (rewritten by the status)
    unsigned long long* delta;
    Records R;
    int64_t need, interval, stop_max;
    int32_t* frontier;
    int32_t* keep;
    unsigned long long* stat;
    PairArgs pa;
    const int32_t* level1;
    hent_t* ht;
    uint64_t hmask;
    JoinRec* joins;               // this stop's admitted joins (eval -> commit)
    int64_t tmp_cap, rec_cap, hcap;
    unsigned long long* ring;     // host-mapped status ring
    int64_t ring_words;
    unsigned long long* sync;     // [0] grid-barrier arrivals, [1] CTAs out (both zero between launches),
                                  // [2] CTA 0's verdict of a small stop, tagged with the stop's sequence number,
                                  // [4 + 1024 p + g] kept entries of CTA g in a grid compaction round of parity p
    int32_t W, KS, kuse_issue, kuse, bound, replay;
};

struct CkptSmem {
    int64_t doff[kDoffMax + 1];         // apply: bucket offsets; commit: start[]
    int64_t bn0[kDoffMax];              // commit: bucket fill before the commit
    int32_t* rec[kDoffMax];             // apply: bucket record tables
    unsigned long long rem[kDoffMax];   // apply: dead slots per bucket (this CTA)
    unsigned long long cnt[3];          // apply: pruned, finalized, survivors (this CTA)
    uint16_t items[kCompactItems];      // compaction staging
    int32_t pos[kCkptThreads];
    int32_t wsum[32];
    int32_t ctotal;
    int64_t nrec0;
    int flag;
};

#ifdef DIC_LAB_TIMING
// lab build: per-stop phase stamps of CTA 0 (globaltimer ns), slot S_SEQ % 512
__device__ unsigned long long g_lab_commit[512][12];
#define CKPT_STAMP(i)                                                                        \
    do {                                                                                     \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                                           \
            unsigned long long _t;                                                           \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                           \
            g_lab_commit[a.stat[S_SEQ] % 512][i] = _t;                                       \
        }                                                                                    \
    } while (0)
#else
#define CKPT_STAMP(i) \
    do {              \
    } while (0)
#endif

// Grid-wide barrier of the co-resident CTAs of a cooperative launch: arrival
// counter in global memory, target = arrivals expected so far.  Thread 0
// publishes the CTA's writes (fence), arrives, spins, then fences again before
// releasing the CTA, so every write before the barrier is visible to every
// thread after it.
__device__ __forceinline__ void grid_barrier(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// P1.  support += delta, intervals += 1 (count_support_interval), then prune
// (engine.py:292-310) and check_full_pass (:380-388) over every bucket slot.
// Slots already dead (left the dashed vector at an earlier stop, compaction
// pending) are only marked not-kept.  keep[g] = still dashed.  A thread takes
// four slots at a time and issues each level of their dependent loads
// (record id -> record fields and count) together.
__device__ __forceinline__ void apply_phase(const CkptArgs& a, CkptSmem& sm, int cta, int nctas,
                                            unsigned long long* delta) {
    unsigned long long* stat = a.stat;
    const int kuse = a.kuse_issue;
    const Records& R = a.R;
    for (int i = threadIdx.x; i <= kuse; i += blockDim.x) sm.doff[i] = a.doff[i];
    for (int i = threadIdx.x; i < kuse; i += blockDim.x) {
        sm.rem[i] = 0;
        sm.rec[i] = a.rec_tab[i];
    }
    if (threadIdx.x < 3) sm.cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t total = sm.doff[kuse];
    // pair counts come from the triangle while the pair bucket is dense
    const bool dense = a.pa.tri != nullptr && 2 * (int64_t)stat[S_HEAD + 2 * a.KS + 2] >= a.pa.tri_len;
    unsigned n_pr = 0, n_fi = 0, n_su = 0;
    constexpr int B = 4;
    const int64_t nth = (int64_t)nctas * blockDim.x;
    const int64_t tid = (int64_t)cta * blockDim.x + threadIdx.x;
    const int64_t iters = (total + nth * B - 1) / (nth * B);  // uniform trip count for the warp votes
    const int64_t wtid = tid & ~(int64_t)31;  // the warp's first slot of a round
    for (int64_t it = 0; it < iters; ++it) {
        // a warp with no slot left is done (slots only grow with it and i):
        // few live slots then cost a few warps' time, not the whole CTA's
        if (it * B * nth + wtid >= total) break;
        int64_t g[B], c[B];
        int bk[B];
        int32_t r[B];
        bool wlive[B];  // warp-uniform: some lane of the warp holds a slot
#pragma unroll
        for (int i = 0; i < B; ++i) {
            g[i] = (it * B + i) * nth + tid;
            wlive[i] = (it * B + i) * nth + wtid < total;
            bk[i] = 0;
            c[i] = 0;
            r[i] = -1;
            if (g[i] < total) {
                int b = 0;
                while (b + 1 < kuse && g[i] >= sm.doff[b + 1]) ++b;
                bk[i] = b;
                c[i] = g[i] - sm.doff[b];
                r[i] = sm.rec[b][c[i]];
            }
        }
        uint8_t sh[B];
        int64_t sup[B], iv[B], dg[B], tp[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
            sh[i] = NIL;
            sup[i] = iv[i] = dg[i] = 0;
            tp[i] = -1;
            if (r[i] >= 0) {
                sh[i] = R.shape[r[i]];
                sup[i] = R.support[r[i]];
                iv[i] = R.intervals[r[i]];
                if (!(bk[i] == 2 && dense)) {
                    // (dense pairs are counted into the triangle: their delta slots stay zero)
                    dg[i] = (int64_t)delta[g[i]];
                } else {
                    // until the bucket is first compacted, slot c still holds the
                    // seeded pair c (record rec0 + c, triangle slot c): no item /
                    // rank lookups on the dependent-load chain
                    int64_t p = c[i];
                    if ((int64_t)r[i] != a.pa.rec0 + c[i]) {
                        const uint16_t* its = a.items_tab[2] + 2 * c[i];
                        p = tri_pos(a.pa.rank[its[0]], a.pa.rank[its[1]], a.pa.L);
                    }
                    tp[i] = p;
                    dg[i] = (int64_t)a.pa.tri[p];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < B; ++i) {
            if (!wlive[i]) continue;
            bool gone = false;
            if (r[i] >= 0) {
                // the count buffers are zero again for the next stop's count
                if (dg[i]) {
                    if (tp[i] >= 0) a.pa.tri[tp[i]] = 0;
                    else delta[g[i]] = 0;
                }
                uint8_t s = sh[i];
                bool kept = false;
                if (is_dashed(s)) {
                    const int64_t sp = sup[i] + dg[i];
                    const int64_t v = iv[i] + 1;
                    if (dg[i]) R.support[r[i]] = sp;
                    R.intervals[r[i]] = v;
                    if (s == DASHED_CIRCLE) {
                        if (sp >= a.need) {
                            s = DASHED_BOX;
                            // order among promoted records is irrelevant to results and stats
                            a.frontier[atomicAdd(&stat[S_NFRONT], 1ull)] = r[i];
                        } else if (a.bound && v < a.stop_max && sp + a.interval * (a.stop_max - v) < a.need) {
                            s = NIL;
                            ++n_pr;
                        }
                    }
                    if (is_dashed(s)) {
                        ++n_su;
                        if (v == a.stop_max) {
                            s = sp >= a.need ? SOLID_BOX : SOLID_CIRCLE;
                            ++n_fi;
                        }
                    }
                    if (s != sh[i]) R.shape[r[i]] = s;
                    kept = is_dashed(s);
                }
                a.keep[g[i]] = kept ? 1 : 0;
                gone = !kept;
            }
            // removed[k], aggregated over the lanes of the same bucket (shared atomics)
            const unsigned gm = __ballot_sync(0xFFFFFFFFu, gone);
            if (gone) {
                const unsigned same = __match_any_sync(gm, bk[i]);
                if ((threadIdx.x & 31) == __ffs(same) - 1)
                    atomicAdd(&sm.rem[bk[i]], (unsigned long long)__popc(same));
            }
        }
    }
    // per-CTA tallies: one global atomic per CTA and counter (a per-warp atomic
    // on the same status word serialises at the L2 slice)
    n_pr = __reduce_add_sync(0xFFFFFFFFu, n_pr);
    n_fi = __reduce_add_sync(0xFFFFFFFFu, n_fi);
    n_su = __reduce_add_sync(0xFFFFFFFFu, n_su);
    if ((threadIdx.x & 31) == 0) {
        if (n_pr) atomicAdd(&sm.cnt[0], (unsigned long long)n_pr);
        if (n_fi) atomicAdd(&sm.cnt[1], (unsigned long long)n_fi);
        if (n_su) atomicAdd(&sm.cnt[2], (unsigned long long)n_su);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (sm.cnt[0]) atomicAdd(&stat[S_NPRUNED], sm.cnt[0]);
        if (sm.cnt[1]) atomicAdd(&stat[S_NFINAL], sm.cnt[1]);
        if (sm.cnt[2]) atomicAdd(&stat[S_SURV], sm.cnt[2]);
    }
    for (int i = threadIdx.x; i < kuse; i += blockDim.x)
        if (sm.rem[i]) atomicAdd(&stat[S_HEAD + i], sm.rem[i]);
}

// P2a.  Order-preserving in-place compaction (compact_dashed,
// itemsets.py:130-132) of bucket k by one CTA: chunks of E slots are scanned
// (keep flags of this stop's apply), staged in shared memory and written back
// to their compacted positions, which never pass the chunk being read.
// bn[k] = kept, removed[k] = cflag[k] = 0.
__device__ __forceinline__ void compact_bucket(const CkptArgs& a, CkptSmem& sm, int k) {
    unsigned long long* stat = a.stat;
    unsigned long long* bn = stat + S_HEAD + 2 * a.KS;
    const int64_t n = (int64_t)bn[k];
    const int32_t* keep = a.keep + a.doff[k];
    int32_t* rec = a.rec_tab[k];
    uint16_t* items = a.items_tab[k];
    const int E = min(kCkptThreads, kCompactItems / k);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t out = 0;
    for (int64_t base = 0; base < n; base += E) {
        const int cnt = (int)min((int64_t)E, n - base);
        const int e = threadIdx.x;
        const bool valid = e < cnt;
        const int kp = valid ? keep[base + e] : 0;
        const int32_t r = valid ? rec[base + e] : 0;
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, kp);
        if (lane == 0) sm.wsum[wid] = __popc(bal);
        for (int j = threadIdx.x; j < cnt * k; j += kCkptThreads) sm.items[j] = items[base * k + j];
        __syncthreads();
        if (wid == 0) {
            const int v = sm.wsum[lane];
            int x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            sm.wsum[lane] = x - v;  // exclusive
            if (lane == 31) sm.ctotal = x;
        }
        __syncthreads();
        const int pos = sm.wsum[wid] + __popc(bal & ((1u << lane) - 1u));
        sm.pos[e] = kp ? pos : -1;
        const int total = sm.ctotal;
        __syncthreads();
        if (kp) rec[out + pos] = r;
        for (int j = threadIdx.x; j < cnt * k; j += kCkptThreads) {
            const int cc = j / k;
            const int p = sm.pos[cc];
            if (p >= 0) items[(out + p) * k + (j - cc * k)] = sm.items[j];
        }
        __syncthreads();
        out += total;
    }
    if (threadIdx.x == 0) {
        bn[k] = (unsigned long long)out;
        stat[S_HEAD + k] = 0;  // removed: none left
        stat[S_HEAD + 3 * a.KS + k] = 0;  // cflag
    }
}

// P2a, large buckets: the same compaction by the whole grid (the pair bucket
// leaves its dense phase with ~500k slots to drop: 860 us on one CTA).  A
// round covers G x S slots: CTA g stages the kept entries of its S slots in
// shared memory and publishes their number; after a grid barrier every CTA
// knows its output offset (the kept entries of the rounds before, plus those
// of the CTAs below it) and writes its staged entries there.  In place and
// safe: a round's writes end at or before the next round's first slot, and
// every slot a write can reach was staged before the barrier.
constexpr int64_t kCoopCompact = 16384;  // bucket fill above which the grid compacts together
constexpr int kStageBytes = 96 * 1024;   // dynamic shared memory of the checkpoint kernel

__device__ __forceinline__ void coop_compact(const CkptArgs& a, CkptSmem& sm, uint8_t* stage, int k, int64_t n,
                                             unsigned long long& nbar) {
    unsigned long long* stat = a.stat;
    const int64_t G = gridDim.x;
    const int64_t smax = (kStageBytes / (4 + 2 * k)) & ~(int64_t)(kCkptThreads - 1);
    const int64_t S = min((((n + G - 1) / G) + kCkptThreads - 1) & ~(int64_t)(kCkptThreads - 1), smax);
    int32_t* srec = reinterpret_cast<int32_t*>(stage);
    uint16_t* sit = reinterpret_cast<uint16_t*>(stage + S * 4);
    const int32_t* keep = a.keep + a.doff[k];
    int32_t* rec = a.rec_tab[k];
    uint16_t* items = a.items_tab[k];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t carry = 0;
    for (int64_t base = 0, round = 0; base < n; base += G * S, ++round) {
        const int64_t lo = min(n, base + (int64_t)blockIdx.x * S), hi = min(n, lo + S);
        int cnt = 0;
        for (int64_t c0 = lo; c0 < hi; c0 += kCkptThreads) {
            const int64_t c = c0 + threadIdx.x;
            const bool valid = c < hi;
            const int kp = valid ? keep[c] : 0;
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, kp);
            if (lane == 0) sm.wsum[wid] = __popc(bal);
            __syncthreads();
            if (wid == 0) {
                const int v = sm.wsum[lane];
                int x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                    if (lane >= o) x += y;
                }
                sm.wsum[lane] = x - v;  // exclusive
                if (lane == 31) sm.ctotal = x;
            }
            __syncthreads();
            if (kp) {
                const int p = cnt + sm.wsum[wid] + __popc(bal & ((1u << lane) - 1u));
                srec[p] = rec[c];
                for (int q = 0; q < k; ++q) sit[(int64_t)p * k + q] = items[c * k + q];
            }
            cnt += sm.ctotal;
            __syncthreads();
        }
        unsigned long long* ccnt = a.sync + 4 + (round & 1) * 1024;
        if (threadIdx.x == 0) {
            ccnt[blockIdx.x] = (unsigned long long)cnt;
            sm.nrec0 = 0;  // (kept entries of the CTAs below this one)
            sm.flag = 0;   // (kept entries of the round)
        }
        grid_barrier(a.sync, (unsigned long long)G * ++nbar);
        if (threadIdx.x < G) {
            const int c = (int)ldv(ccnt + threadIdx.x);
            if (c) {
                atomicAdd(&sm.flag, c);
                if ((int)threadIdx.x < (int)blockIdx.x) atomicAdd(reinterpret_cast<unsigned long long*>(&sm.nrec0),
                                                                  (unsigned long long)c);
            }
        }
        __syncthreads();
        const int64_t off = carry + sm.nrec0;
        for (int i = threadIdx.x; i < cnt; i += kCkptThreads) rec[off + i] = srec[i];
        for (int j = threadIdx.x; j < cnt * k; j += kCkptThreads) items[off * k + j] = sit[j];
        carry += sm.flag;
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        stat[S_HEAD + 2 * a.KS + k] = (unsigned long long)carry;  // bn[k]
        stat[S_HEAD + k] = 0;                                     // removed: none left
        stat[S_HEAD + 3 * a.KS + k] = 0;                          // cflag
    }
}

// P2b.  make_candidates (engine.py:320-369): evaluation of the
// (frontier f, level1 item j) joins, and — in the same pass — the claim of
// every admitted join in the hash index.
//
// Admission needs cand not in known and every immediate subset known with a
// box shape; the subset equal to src is a box by construction (it was just
// promoted) and is skipped.  The subset test rejects almost every join (its
// first subset is rarely a box yet), so it runs first; the admitted set is the
// same in either order.
//
// A join that passes walks cand's probe chain once: an existing record with
// cand's mask -> already known, drop; a temporary entry with cand's mask ->
// another source produced the same candidate at this stop, drop (all
// duplicates carry the same mask, so which join wins does not matter); an
// empty slot -> CAS a temporary entry into it: the winner owns the candidate
// and takes a join record.  No record is published before the commit, so a
// non-temporary entry always names a record of an earlier stop, and a subset
// lookup that meets a temporary entry just keeps probing (a fresh candidate is
// no box: the join fails either way, as in the reference, where it is a
// DASHED_CIRCLE).  The all-or-nothing capacity check follows the phase; if it
// fails the host rebuilds the index from the records (dropping the temporary
// entries) and replays.
struct JoinRec {
    unsigned long long hi, lo;  // sort key (size, first seven ids, 16 bits each)
    uint64_t hash;
    int64_t slot;  // hash slot the owner claimed
    int32_t src;   // source record: the candidate is src's itemset + {l}
    uint16_t l, size;
};

__device__ __forceinline__ bool views_same(const MaskView& x, const MaskView& y, int W) {
    unsigned long long d = 0;
    for (int w = 0; w < W; ++w) d |= x.word(w) ^ y.word(w);  // no early exit: the loads go out together
    return d == 0;
}

__device__ __forceinline__ void key_take(int w, unsigned long long x, int& j, unsigned long long& hi,
                                         unsigned long long& lo) {
    while (x && j < 7) {
        const unsigned long long it = (unsigned long long)(w * 64 + __ffsll((long long)x) - 1);
        x &= x - 1;
        if (j < 3) hi |= it << (32 - 16 * j);
        else lo |= it << (48 - 16 * (j - 3));
        ++j;
    }
}

// Claim cand = src + {l} (hash hc, sz items, sort key (hi, lo)) in the index,
// or find it there.  Temporary entries of this stop's other joins are compared
// by mask (both are views of records of earlier stops).
__device__ __noinline__ void claim_join(const CkptArgs& a, int32_t src, int l, uint64_t hc, int sz,
                                        unsigned long long hi, unsigned long long lo, const int* its, int k) {
    unsigned long long* stat = a.stat;
    const Records& R = a.R;
    const int W = a.W;
    const uint32_t tag = htag(hc);
    const MaskView cand{R.mask + (int64_t)src * W, l, -1};
#ifdef DIC_LAB_TIMING
    struct LabT {
        unsigned long long t0, seq;
        __device__ LabT(unsigned long long s) : seq(s) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0)); }
        __device__ ~LabT() {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            atomicMax(&g_lab_commit[seq % 512][8], t1 - t0);
            atomicAdd(&g_lab_commit[seq % 512][10], 1ull);
        }
    } lab_t(stat[S_SEQ]);
#endif
    uint64_t slot = mix64(hc) & a.hmask;
    hent_t x = ldv(a.ht + slot);
    while (true) {
        if (x == kEmptyEnt) {
            x = atomicCAS(a.ht + slot, kEmptyEnt, hent_join(hc, src, l));
            if (x == kEmptyEnt) {  // owner: the stop's next join record
                const int64_t t = (int64_t)atomicAdd(&stat[S_NADM], 1ull);
                atomicAdd(&stat[S_NINS], 1ull);
                atomicAdd(&stat[S_HEAD + a.KS + sz], 1ull);  // adm[sz]
                if (t < a.tmp_cap) {                          // (else: the capacity check sees NADM)
                    JoinRec* j = a.joins + t;
                    j->hi = hi;
                    j->lo = lo;
                    j->hash = hc;
                    j->slot = (int64_t)slot;
                    j->src = src;
                    j->l = (uint16_t)l;
                    j->size = (uint16_t)sz;
                }
                return;
            }
            // another thread took the slot first: examine its entry
        }
        bool same = false;
        if (hent_temp(x)) {
            if ((x & 0xFFFFull) == ((hc >> 32) & 0xFFFFull))
                same = views_same(MaskView{R.mask + (int64_t)hent_join_src(x) * W, hent_join_item(x), -1}, cand, W);
        } else if (hent_tag(x) == tag) {
            const int32_t e = hent_id(x);
            if (its) {
                // a record of the same size holding every item of cand IS cand
                same = R.size[e] == sz;
                if (same) {
                    const unsigned long long* rm = R.mask + (int64_t)e * W;
                    bool ok = ((rm[l >> 6] >> (l & 63)) & 1ull) != 0;
                    for (int q = 0; q < k; ++q) ok &= ((rm[its[q] >> 6] >> (its[q] & 63)) & 1ull) != 0;
                    same = ok;
                }
            } else {
                same = mask_eq(R.mask + (int64_t)e * W, cand, W);
            }
        }
        if (same) return;  // known, or another join's candidate
        slot = (slot + 1) & a.hmask;
        x = ldv(a.ht + slot);
    }
}

__device__ __forceinline__ void eval_phase(const CkptArgs& a, int64_t nfront, int cta, int nctas) {
    const Records& R = a.R;
    const int W = a.W;
    const int64_t L = a.pa.L;
    const hent_t* ht = a.ht;
    const uint64_t hmask = a.hmask;
    const int32_t* prank = a.pa.rank;
    const int64_t prec0 = a.pa.rec0;
    const int64_t total = nfront * L;
    for (int64_t t = (int64_t)cta * blockDim.x + threadIdx.x; t < total; t += (int64_t)nctas * blockDim.x) {
        const int64_t f = t / L, j = t - f * L;
        const int32_t src = a.frontier[f];
        const int l = a.level1[j];
        // everything the join needs of src in one round of loads (its item
        // list is only meaningful for ks <= 8, but always addressable)
        const int ks = R.size[src];
        const uint4 iv = *reinterpret_cast<const uint4*>(R.items + (int64_t)src * 8);
        const uint64_t hsrc = R.hash[src];
        if (ks <= 7) {
            // item-list path: src's ascending ids came in one 16-byte load
            int its[8] = {(int)(iv.x & 0xFFFFu), (int)(iv.x >> 16), (int)(iv.y & 0xFFFFu), (int)(iv.y >> 16),
                          (int)(iv.z & 0xFFFFu), (int)(iv.z >> 16), (int)(iv.w & 0xFFFFu), (int)(iv.w >> 16)};
            bool in = false;
#pragma unroll
            for (int q = 0; q < 7; ++q) in |= q < ks && its[q] == l;
            if (in) continue;  // cand == base
            bool ok = true;
            if (ks == 2 && prank) {
                // a pair source (the pair wave's joins): its immediate subsets
                // {a, l} and {b, l} are seeded pairs of frequent items, whose
                // record ids follow from the items' level1 ranks (record
                // prec0 + triangle slot, seed_pairs_kernel): one load each
                // instead of a hash probe chain.  l = level1[j] has rank j.
                const int64_t ra = prank[its[0]], rb = prank[its[1]];
                const int64_t pa = ra < j ? tri_pos(ra, j, L) : tri_pos(j, ra, L);
                const int64_t pb = rb < j ? tri_pos(rb, j, L) : tri_pos(j, rb, L);
                const uint8_t sb = R.shape[prec0 + pb], sa = R.shape[prec0 + pa];  // (both loads at once)
                ok = is_box(sb) & is_box(sa);
            }
            if (!ok) continue;
            const uint64_t hc = hsrc ^ zob((uint32_t)l);
            if (!(ks == 2 && prank)) {
                if (ks <= 4) {
                    // the (up to four) subset probes side by side: their index
                    // slots in one round of loads, the records they name in a
                    // second, instead of a chain of 4 dependent loads per subset
                    int32_t eq[4];
                    unsigned slow = 0;  // probes that met a collision: sequential path below
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        eq[q] = -1;
                        if (q < ks) {
                            const uint64_t hq = hc ^ zob((uint32_t)its[q]);
                            const hent_t x = ht[mix64(hq) & hmask];
                            const int32_t e = hent_id(x);
                            if (x == kEmptyEnt) ok = false;  // not known
                            else if (hent_tag(x) == htag(hq)) eq[q] = e;
                            else slow |= 1u << q;
                        }
                    }
                    if (!ok) continue;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (q < ks && eq[q] >= 0) {
                            const unsigned long long* rm = R.mask + (int64_t)eq[q] * W;
                            bool match = R.size[eq[q]] == ks;
                            match &= ((rm[l >> 6] >> (l & 63)) & 1ull) != 0;
#pragma unroll
                            for (int p = 0; p < 4; ++p)
                                if (p < ks && p != q) match &= ((rm[its[p] >> 6] >> (its[p] & 63)) & 1ull) != 0;
                            const bool box = is_box(R.shape[eq[q]]);
                            if (!match) slow |= 1u << q;
                            else ok &= box;
                        }
                    }
                    for (int q = 0; q < ks && ok; ++q) {
                        if (!((slow >> q) & 1u)) continue;
                        const int d = its[q];
                        const int32_t e = ht_find_items(ht, hmask, R, W, hc ^ zob((uint32_t)d), its, ks, l, d, ks);
                        ok = e >= 0 && is_box(R.shape[e]);
                    }
                } else {
                    for (int q = 0; q < ks && ok; ++q) {
                        const int d = its[q];
                        const int32_t e = ht_find_items(ht, hmask, R, W, hc ^ zob((uint32_t)d), its, ks, l, d, ks);
                        ok = e >= 0 && is_box(R.shape[e]);
                    }
                }
                if (!ok) continue;
            }
            // sort key from the merged ascending list
            int p = 0;
#pragma unroll
            for (int q = 0; q < 7; ++q) p += (q < ks && its[q] < l) ? 1 : 0;
            unsigned long long hi = (unsigned long long)(uint32_t)(ks + 1) << 48, lo = 0;
#pragma unroll
            for (int q = 0; q < 7; ++q) {
                if (q <= ks) {
                    const unsigned long long it = (unsigned long long)(q < p ? its[q] : (q == p ? l : its[q > 0 ? q - 1 : 0]));
                    if (q < 3) hi |= it << (32 - 16 * q);
                    else lo |= it << (48 - 16 * (q - 3));
                }
            }
            claim_join(a, src, l, hc, ks + 1, hi, lo, its, ks);
        } else {
            // large itemsets: masks all the way
            const unsigned long long* sm = R.mask + (int64_t)src * W;
            if ((sm[l >> 6] >> (l & 63)) & 1ull) continue;  // cand == base
            const uint64_t hc = hsrc ^ zob((uint32_t)l);
            const MaskView cand{sm, l, -1};
            bool ok = true;
            for (int w = 0; w < W && ok; ++w) {
                unsigned long long x = cand.word(w);
                while (x) {
                    const int bit = w * 64 + __ffsll((long long)x) - 1;
                    x &= x - 1;
                    if (bit == l) continue;
                    const MaskView sub{sm, l, bit};
                    const int32_t e = ht_lookup(ht, hmask, R, W, hc ^ zob((uint32_t)bit), sub);
                    if (e < 0 || !is_box(R.shape[e])) {
                        ok = false;
                        break;
                    }
                }
            }
            if (!ok) continue;
            unsigned long long hi = (unsigned long long)(uint32_t)(ks + 1) << 48, lo = 0;
            int q = 0;
            for (int w = 0; w < W && q < 7; ++w) key_take(w, cand.word(w), q, hi, lo);
            claim_join(a, src, l, hc, ks + 1, hi, lo, nullptr, 0);
        }
    }
}

// All-or-nothing capacity check of the candidate step: the joins, the records
// and hash load after them, every bucket's room.  Every CTA evaluates it on
// the same (stable) inputs; CTA 0 records the verdict.  An overflow also
// raises the abort flag so every later stop is skipped until the host's replay.
__device__ __forceinline__ bool capacity_over(const CkptArgs& a, CkptSmem& sm) {
    unsigned long long* stat = a.stat;
    const int KS = a.KS;
    if (threadIdx.x == 0) {
        const unsigned long long na = ldv(stat + S_NADM), nr = ldv(stat + S_NREC);
        sm.flag = (int64_t)na > a.tmp_cap || (int64_t)(nr + na) > a.rec_cap || (int64_t)(nr + na) * 2 > a.hcap;
    }
    __syncthreads();
    const unsigned long long* adm = stat + S_HEAD + KS;
    const unsigned long long* bn = stat + S_HEAD + 2 * KS;
    // a stop's joins are one item larger than a live itemset, i.e. <= kuse items
    const int lim = min(KS, a.kuse + 1);
    for (int k = threadIdx.x; k < lim; k += blockDim.x) {
        const unsigned long long ak = ldv(adm + k);
        if (ak && (int64_t)(ldv(bn + k) + ak) > a.bcap[k]) sm.flag = 1;
    }
    __syncthreads();
    const bool over = sm.flag != 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        stat[S_OVERFLOW] = over ? 1ull : 0ull;
        if (over) stat[S_ABORT] = 1ull;
    }
    return over;
}

// P3.  Candidate commit with a CANONICAL result: the record ids and bucket
// positions of a stop's new candidates depend only on the SET of candidates,
// never on thread timing.  Sharded engines reduce their counts slot by slot,
// so every rank must lay its buckets out identically (the reference reduces
// per record, engine.py:268-270); with atomics deciding the order, ranks
// would add up counts of different itemsets.
//
// The owning joins are ranked by (size, item ids ascending) — the order of
// make_candidates' lexicographic joins, which also makes candidates sharing a
// prefix contiguous for the count kernel — and the one of rank i gets record
// id nrec + i and position bn[size] + (its rank within its size); then the
// record, bucket entry and hash entry are written by its warp.  A rank is a
// count of smaller keys, one warp per candidate (N^2 / 32 warp steps spread
// over the GPU: a few microseconds for the hundreds of joins a stop commits;
// no sort, no serial phase).  Equal keys (size >= 8 sharing seven ids) fall
// back to the masks, where the lexicographically smaller item list is the one
// holding the lowest bit in which the two masks differ.
__device__ __noinline__ bool join_less_slow(const CkptArgs& a, const JoinRec& x, const JoinRec& y) {
    const MaskView vx{a.R.mask + (int64_t)x.src * a.W, (int)x.l, -1};
    const MaskView vy{a.R.mask + (int64_t)y.src * a.W, (int)y.l, -1};
    for (int w = 0; w < a.W; ++w) {
        const unsigned long long xw = vx.word(w), d = xw ^ vy.word(w);
        if (d) return (xw & (d & (~d + 1))) != 0;
    }
    return false;  // equal masks: impossible among owners
}

__device__ __forceinline__ void commit_phase(const CkptArgs& a, CkptSmem& sm, int64_t na, int cta, int nctas) {
    unsigned long long* stat = a.stat;
    const Records& R = a.R;
    const int W = a.W;
    unsigned long long* bn = stat + S_HEAD + 2 * a.KS;
    const int top = a.kuse < kDoffMax ? a.kuse : kDoffMax;  // sizes that can hold candidates
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t* start = sm.doff;
    // start[k] = new candidates of sizes < k: warp 0 scans 32 sizes per step
    if (wid == 0) {
        int64_t carry = 0;
        for (int k0 = 0; k0 < top; k0 += 32) {
            const int k = k0 + lane;
            const int64_t v = k < top ? (int64_t)ldv(stat + S_HEAD + a.KS + k) : 0;  // adm[k]
            int64_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            if (k < top) {
                start[k] = carry + x - v;
                sm.bn0[k] = (int64_t)ldv(bn + k);
            }
            carry += __shfl_sync(0xFFFFFFFFu, x, 31);
        }
        if (lane == 0) sm.nrec0 = (int64_t)ldv(stat + S_NREC);
    }
    __syncthreads();
    // one warp per join: an owner's rank is the number of owners with smaller keys
    constexpr int kWarps = kCkptThreads / 32;
    const int64_t warps = (int64_t)nctas * kWarps;
    // consecutive joins go to different CTAs (every SM takes part even when
    // the stop commits only a few)
    for (int64_t e = (int64_t)wid * nctas + cta; e < na; e += warps) {
        const JoinRec je = a.joins[e];
        // what the commit needs of the source record and the bucket tables,
        // loaded before the ranking rounds instead of after them
        const int sz = je.size;
        const unsigned long long* smk = R.mask + (int64_t)je.src * W;
        unsigned long long mw = lane < W ? smk[lane] : 0ull;  // (masks of up to 32 words: one load per lane)
        const int mine = (sz <= 8 && lane < sz - 1) ? (int)R.items[(int64_t)je.src * 8 + lane] : 0x10000;
        int32_t* const brec = a.rec_tab[sz];
        uint16_t* const bits = a.items_tab[sz];
        unsigned cnt = 0;
        for (int64_t j0 = lane; j0 < na; j0 += 128) {
            // four keys per lane and round: their loads go out together
            unsigned long long hj[4], lj[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t j = j0 + 32 * u;
                hj[u] = j < na ? a.joins[j].hi : ~0ull;
                lj[u] = j < na ? a.joins[j].lo : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t j = j0 + 32 * u;
                bool less = hj[u] != je.hi ? hj[u] < je.hi : lj[u] < je.lo;  // (the ~0 filler is never smaller)
                if (hj[u] == je.hi && lj[u] == je.lo && j != e && j < na) less = join_less_slow(a, a.joins[j], je);
                cnt += less ? 1u : 0u;
            }
        }
        cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
        // record nrec0 + rank at bucket slot bn0[sz] + rank - start[sz]; its
        // record id replaces the temporary entry in the hash slot it claimed
        const int64_t r = sm.nrec0 + cnt;
        const int64_t pos = sm.bn0[sz] + ((int64_t)cnt - start[sz]);
        if (lane < W) {
            if (lane == (je.l >> 6)) mw |= 1ull << (je.l & 63);
            R.mask[r * W + lane] = mw;
        }
        for (int w = 32 + lane; w < W; w += 32) {
            unsigned long long x = smk[w];
            if (w == (je.l >> 6)) x |= 1ull << (je.l & 63);
            R.mask[r * W + w] = x;
        }
        uint16_t* bit = bits + pos * sz;
        if (sz <= 8) {
            // the ascending ids: src's list with l merged in; lane q holds item q
            const int p = __popc(__ballot_sync(0xFFFFFFFFu, mine < (int)je.l));
            const int up = __shfl_up_sync(0xFFFFFFFFu, mine, 1);
            const int it = lane < p ? mine : (lane == p ? (int)je.l : up);
            if (lane < sz) bit[lane] = (uint16_t)it;
            if (lane < 8) R.items[r * 8 + lane] = lane < sz ? (uint16_t)it : (uint16_t)0;
        } else if (lane == 0) {
            int q = 0;
            for (int w = 0; w < W; ++w) {
                unsigned long long x = smk[w];
                if (w == (je.l >> 6)) x |= 1ull << (je.l & 63);
                while (x) {
                    bit[q++] = (uint16_t)(w * 64 + __ffsll((long long)x) - 1);
                    x &= x - 1;
                }
            }
        }
        if (lane == 0) {
            R.hash[r] = je.hash;
            R.size[r] = sz;
            R.support[r] = 0;
            R.intervals[r] = 0;
            R.shape[r] = DASHED_CIRCLE;
            brec[pos] = (int32_t)r;
            a.ht[je.slot] = hent(je.hash, (int32_t)r);
        }
    }
}

// The stop's status into its (host-mapped, pinned) ring slot S_SEQ % kRing:
// head words, then removed[k], adm[k], bn[k] for k < kuse.  Then, unless the
// stop overflowed (the replay needs its counters; later stops are no-ops and
// rewrite the same slot), advance S_SEQ, flag the buckets to compact at the
// next stop (dead slots >= a quarter), reset the per-stop counters and
// compute the next stop's delta offsets from the bucket fill.
// ring == nullptr: reset only (engine seeding).
// Run by ONE warp (the caller's warp 0; the other warps skip it): every size's
// three words are loaded in one round (from L2: atomics of this launch updated
// them there) and stay in registers through the ring write, the flags and the
// offset scan — no CTA barrier, one chain of loads (2.9 -> ~1 us per stop).
__device__ void status_body(unsigned long long* stat, int KS, int kuse, unsigned long long* ring,
                            int64_t ring_words, int64_t* doff) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const unsigned long long seq = ldv(stat + S_SEQ), aborted = ldv(stat + S_ABORT);
    unsigned long long* slot = ring ? ring + (int64_t)(seq % kRing) * ring_words : nullptr;
    if (slot && lane < S_HEAD) slot[lane] = ldv(stat + lane);
    // sizes < lim can hold anything non-zero (a stop's joins are one item larger
    // than its largest live itemset, which is < kuse); offsets are kept for
    // sizes <= top (a later stop may use a larger kuse: all equal the total)
    const int top = KS < kDoffMax ? KS : kDoffMax;
    const int use = min(top, kuse);
    const int lim = min(min(KS, kDoffMax), kuse + 1);
    int64_t carry = 0;
    for (int k0 = 0; k0 < lim; k0 += 32) {
        const int k = k0 + lane;
        unsigned long long rem = 0, adm = 0, fill = 0;
        if (k < lim) {
            rem = ldv(stat + S_HEAD + k);
            adm = ldv(stat + S_HEAD + KS + k);
            fill = ldv(stat + S_HEAD + 2 * KS + k);
        }
        if (slot && k < kuse) {
            slot[S_HEAD + 3 * k] = rem;
            slot[S_HEAD + 3 * k + 1] = adm;
            slot[S_HEAD + 3 * k + 2] = fill;
        }
        if (aborted) continue;  // (warp-uniform)
        if (k < lim) {
            stat[S_HEAD + 3 * KS + k] = (rem > 0 && (rem * 4 >= fill || rem == fill)) ? 1ull : 0ull;  // cflag
            if (rem) stat[S_HEAD + k] = 0;       // removed
            if (adm) stat[S_HEAD + KS + k] = 0;  // adm
        }
        // delta offsets: exclusive prefix of the bucket fills
        const int64_t v = k < use ? (int64_t)fill : 0;
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (k < use) doff[k] = carry + x - v;
        carry += __shfl_sync(0xFFFFFFFFu, x, 31);
    }
    if (aborted) return;
    for (int k = use + lane; k <= top; k += 32) doff[k] = carry;
    if (lane < S_NREC) stat[lane] = 0;
    if (ring && lane == 0) stat[S_SEQ] = seq + 1;
}

// ring == nullptr: reset only (engine seeding)
__global__ void status_kernel(unsigned long long* __restrict__ stat, int KS, int kuse,
                              unsigned long long* __restrict__ ring, int64_t ring_words, int64_t* __restrict__ doff) {
    status_body(stat, KS, kuse, ring, ring_words, doff);
}

// Stops with few live slots (the long tail of a run: tens to a few thousand
// dashed itemsets) are run by CTA 0 alone, with CTA-level barriers: a
// grid-wide barrier costs ~1.5 us, more than such a phase's whole work.  The
// other CTAs wait for CTA 0's verdict after the apply — "done without you"
// or, when the stop promoted enough itemsets for the joins to need the grid,
// "join in" — published as a word tagged with the stop's sequence number.
constexpr int64_t kSmallSlots = 2048;  // <= 2 slots per thread of one CTA
constexpr int64_t kSoloJoins = 2048;   // <= 2 joins per thread of one CTA

__global__ void __launch_bounds__(kCkptThreads, 1) checkpoint_kernel(const __grid_constant__ CkptArgs a) {
    __shared__ CkptSmem sm;
    extern __shared__ __align__(16) uint8_t dyn_smem[];  // kStageBytes: coop_compact's staging
    unsigned long long* stat = a.stat;
    // a stop skipped by the overflow recovery: only its (unchanged) status
    if (stat[S_ABORT]) {
        if (blockIdx.x == 0) status_body(stat, a.KS, a.kuse, a.ring, a.ring_words, a.doff);
        return;
    }
    const unsigned long long G = gridDim.x;
    const unsigned long long tag = (stat[S_SEQ] + 1) << 2;
    unsigned long long nbar = 0;
    const bool small = !a.replay && G > 1 && a.doff[a.kuse_issue] <= kSmallSlots;
    bool solo = false;
    CKPT_STAMP(0);
    if (!a.replay) {
        if (!small) {
            apply_phase(a, sm, blockIdx.x, gridDim.x, a.delta);
            grid_barrier(a.sync, G * ++nbar);
        } else if (blockIdx.x == 0) {
            apply_phase(a, sm, 0, 1, a.delta);
            __syncthreads();
        }
    }
    CKPT_STAMP(1);
    if (small) {
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0) {
                sm.flag = (int64_t)ldv(stat + S_NFRONT) * a.pa.L <= kSoloJoins;
                // "join in" is a release (the apply's writes before the verdict);
                // "done without you" carries no data
                const unsigned long long v = tag | (sm.flag ? 1ull : 2ull);
                if (sm.flag) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a.sync + 2), "l"(v) : "memory");
                else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.sync + 2), "l"(v) : "memory");
            }
            __syncthreads();
            solo = sm.flag != 0;
        } else {
            if (threadIdx.x == 0) {
                unsigned long long v;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.sync + 2) : "memory");
                } while ((v & ~3ull) != tag);
                sm.flag = (v & 3ull) == 1ull;
            }
            __syncthreads();
            if (sm.flag) return;  // CTA 0 finishes the stop alone
        }
    }
    const int cta = solo ? 0 : (int)blockIdx.x, nctas = solo ? 1 : (int)gridDim.x;
    // The frontier size and the flagged buckets' fills in ONE round of loads (a
    // loop of dependent-latency loads otherwise), before any compaction of this
    // launch changes the fills: large buckets are compacted by the whole grid
    // (every CTA must take the same decisions), the others by one CTA each.
    const int kc = a.replay ? 0 : min(a.kuse_issue, a.KS);
    __syncthreads();
    if ((int)threadIdx.x < kc) {
        const unsigned long long* cflag = stat + S_HEAD + 3 * a.KS;
        const unsigned long long* bn = stat + S_HEAD + 2 * a.KS;
        // flag and fill loaded side by side
        const unsigned long long fl = cflag[threadIdx.x], fill = bn[threadIdx.x];
        sm.bn0[threadIdx.x] = fl ? (int64_t)fill : 0;
    } else if (threadIdx.x == kCkptThreads - 1) {
        sm.nrec0 = (int64_t)ldv(stat + S_NFRONT);
    }
    __syncthreads();
    const int64_t nfront = sm.nrec0;
    for (int k = 1; k < kc; ++k) {
        const int64_t n = sm.bn0[k];
        if (n == 0) continue;
        if (!solo && n > kCoopCompact) coop_compact(a, sm, dyn_smem, k, n, nbar);
        else if ((k - 1) % nctas == cta) compact_bucket(a, sm, k);
    }
    int64_t N = 0;
    if (nfront > 0) {
        CKPT_STAMP(11);
        eval_phase(a, nfront, cta, nctas);
        CKPT_STAMP(7);
#ifdef DIC_LAB_TIMING
        if (threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(&g_lab_commit[stat[S_SEQ] % 512][9], t);
        }
#endif
        if (solo) {
            __syncthreads();
        } else {
            grid_barrier(a.sync, G * ++nbar);
        }
        CKPT_STAMP(2);
        if (!capacity_over(a, sm)) {
            N = (int64_t)ldv(stat + S_NINS);
            if (N > 0) commit_phase(a, sm, (int64_t)ldv(stat + S_NADM), cta, nctas);
        }
    }
    CKPT_STAMP(3);
    // the last CTA out: sizes after the commit, then the stop's status
    __syncthreads();
    if (!solo) {
        if (threadIdx.x == 0) {
            __threadfence();
            sm.flag = atomicAdd(&a.sync[1], 1ull) == G - 1;
        }
        __syncthreads();
        if (!sm.flag) return;
        if (threadIdx.x == 0) __threadfence();
        __syncthreads();
    }
    if (N > 0) {
        unsigned long long* bn = stat + S_HEAD + 2 * a.KS;
        const int top = a.kuse < kDoffMax ? a.kuse : kDoffMax;
        for (int k = threadIdx.x; k < top; k += blockDim.x) {
            const unsigned long long n = ldv(stat + S_HEAD + a.KS + k);  // adm[k]
            if (n) bn[k] = ldv(bn + k) + n;
        }
        if (threadIdx.x == 0) stat[S_NREC] = ldv(stat + S_NREC) + (unsigned long long)N;
    }
    if (threadIdx.x == 0 && !solo) {
        a.sync[0] = 0;
        a.sync[1] = 0;
    }
    __syncthreads();
    CKPT_STAMP(4);
#ifdef DIC_LAB_TIMING
    const unsigned long long lab_seq = stat[S_SEQ];
#endif
    status_body(stat, a.KS, a.kuse, a.ring, a.ring_words, a.doff);
#ifdef DIC_LAB_TIMING
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_lab_commit[lab_seq % 512][5] = t;
        g_lab_commit[lab_seq % 512][6] = (unsigned long long)(small ? (solo ? 2 : 1) : 0);
    }
#endif
}

// The quiet tail of a run — a few hundred live itemsets or fewer, most stops
// without a promotion — costs a launch gap, a count kernel and a checkpoint
// kernel per stop for microseconds of work.  dic_engine_run therefore issues
// such stops in BATCHES: one count launch fills a delta block per chunk for the
// next `nstops` chunks (count.cu, DevCountArgs::batch), and this kernel — one
// CTA, CTA-level barriers only — runs their checkpoints one after the other.
// The counts of the later chunks hold only while the dashed vector keeps its
// slots: nothing is compacted inside a batch (flagged buckets keep their dead
// slots until the next single stop; the blocks are small), and the batch ends
// after a stop that inserted candidates (they were not counted in the later
// chunks) or that overflowed; the stops not run leave no status, and the host
// issues them again.
constexpr int64_t kBatchSlots = 2048;  // live slots of a batched stop (one delta block)
constexpr int kBatchStops = 8;

// The kernel reports what it ran in a host-mapped word — (first sequence number
// + 1) << 8 | stops run — of the parity of its launch number (a.sync[3]), so the
// host can keep two batches in flight and still read exactly the ring slots a
// finished batch wrote.
__global__ void __launch_bounds__(kCkptThreads, 1) checkpoint_batch_kernel(const __grid_constant__ CkptArgs a,
                                                                       int nstops, unsigned long long* bdelta,
                                                                       unsigned long long* report) {
    __shared__ CkptSmem sm;
    unsigned long long* stat = a.stat;
    const int64_t total0 = a.doff[a.kuse_issue];
    const unsigned long long seq0 = stat[S_SEQ], launch_no = a.sync[3];
    if (stat[S_ABORT] || total0 > kBatchSlots) {
        // skipped by the overflow recovery (its unchanged status), or refused:
        // the count launch made the same test and counted nothing
        if (stat[S_ABORT]) status_body(stat, a.KS, a.kuse, a.ring, a.ring_words, a.doff);
        if (threadIdx.x == 0) {
            report[launch_no & 1] = (seq0 + 1) << 8;
            a.sync[3] = launch_no + 1;
        }
        return;
    }
    int b = 0;
    for (; b < nstops; ++b) {
        apply_phase(a, sm, 0, 1, bdelta + (int64_t)b * kBatchSlots);
        __syncthreads();
        const int64_t nfront = (int64_t)ldv(stat + S_NFRONT);
        int64_t N = 0;
        bool over = false;
        if (nfront > 0) {
            eval_phase(a, nfront, 0, 1);
            __syncthreads();
            over = capacity_over(a, sm);
            if (!over) {
                N = (int64_t)ldv(stat + S_NINS);
                if (N > 0) commit_phase(a, sm, (int64_t)ldv(stat + S_NADM), 0, 1);
            }
        }
        __syncthreads();
        if (N > 0) {
            unsigned long long* bnw = stat + S_HEAD + 2 * a.KS;
            const int top = a.kuse < kDoffMax ? a.kuse : kDoffMax;
            for (int k = threadIdx.x; k < top; k += blockDim.x) {
                const unsigned long long n = ldv(stat + S_HEAD + a.KS + k);  // adm[k]
                if (n) bnw[k] = ldv(bnw + k) + n;
            }
            if (threadIdx.x == 0) stat[S_NREC] = ldv(stat + S_NREC) + (unsigned long long)N;
        }
        __syncthreads();
        status_body(stat, a.KS, a.kuse, a.ring, a.ring_words, a.doff);
        __syncthreads();
        // may the next chunk's counts be applied to the same slots?
        if (over || N > 0) {  // (uniform)
            ++b;
            break;
        }
    }
    // the delta blocks of the stops not run go back to zero (a run stop's block
    // was re-zeroed by its apply)
    for (int64_t i = (int64_t)b * kBatchSlots + threadIdx.x; i < (int64_t)nstops * kBatchSlots; i += blockDim.x)
        if ((i % kBatchSlots) < total0) bdelta[i] = 0;
    if (threadIdx.x == 0) {
        report[launch_no & 1] = ((seq0 + 1) << 8) | (unsigned long long)b;
        a.sync[3] = launch_no + 1;
    }
}

struct TableUpdate {
    static constexpr int kMax = 16;
    int n;
    int k[kMax];
    int32_t* rec[kMax];
    uint16_t* items[kMax];
    int64_t cap[kMax];
};

__global__ void set_tables_kernel(int32_t** brec, uint16_t** bitems, int64_t* bcap, TableUpdate u) {
    const int i = threadIdx.x;
    if (i >= u.n) return;
    brec[u.k[i]] = u.rec[i];
    bitems[u.k[i]] = u.items[i];
    bcap[u.k[i]] = u.cap[i];
}

__global__ void collect_frequent_kernel(Records R, int64_t nrec, int32_t* out, unsigned long long* nout) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrec || R.shape[r] != SOLID_BOX) return;
    out[atomicAdd(nout, 1ull)] = (int32_t)r;
}

__global__ void gather_frequent_kernel(Records R, int W, const int32_t* __restrict__ ids, int64_t F,
                                       unsigned long long* masks, int32_t* sizes, int64_t* supports) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F) return;
    int32_t r = ids[i];
    for (int w = 0; w < W; ++w) masks[i * W + w] = R.mask[(int64_t)r * W + w];
    sizes[i] = R.size[r];
    supports[i] = R.support[r];
}

// Canonical order of the result (engine.py:446-455): by size, then by the
// mask as an integer — for masks of equal size, the lexicographic order of
// their item ids listed from the highest down.  Key of a frequent record of
// at most 8 items: (size, ids descending), 16 bits each; *big is raised when a
// larger itemset is met (the host then sorts instead).
struct ResKey {
    unsigned long long k0, k1, k2;
};

__global__ void result_keys_kernel(Records R, const int32_t* __restrict__ ids, int64_t F, ResKey* __restrict__ keys,
                                   unsigned long long* big) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F) return;
    const int32_t r = ids[i];
    const int sz = R.size[r];
    ResKey k{(unsigned long long)(uint32_t)sz << 48, 0ull, 0ull};
    if (sz > 8) {
        *big = 1ull;
    } else {
        const uint4 iv = *reinterpret_cast<const uint4*>(R.items + (int64_t)r * 8);
        const uint32_t w[4] = {iv.x, iv.y, iv.z, iv.w};
        for (int q = 0; q < sz; ++q) {
            const int a = sz - 1 - q;  // q-th highest id
            const unsigned long long it = (w[a >> 1] >> ((a & 1) * 16)) & 0xFFFFu;
            if (q < 3) k.k0 |= it << (32 - 16 * q);
            else if (q < 7) k.k1 |= it << (48 - 16 * (q - 3));
            else k.k2 |= it << 48;
        }
    }
    keys[i] = k;
}

// One warp per frequent record: its position is the number of smaller keys
// (distinct itemsets have distinct keys); the warp then writes the record's
// mask, size and support to that position.
__global__ void result_rank_gather_kernel(Records R, int W, const int32_t* __restrict__ ids, int64_t F,
                                          const ResKey* __restrict__ keys, unsigned long long* __restrict__ masks,
                                          int32_t* __restrict__ sizes, int64_t* __restrict__ supports) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < F; i += warps) {
        const ResKey me = keys[i];
        unsigned cnt = 0;
        for (int64_t j0 = lane; j0 < F; j0 += 128) {
            // four keys per lane and round: their loads go out together
            ResKey o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = j0 + 32 * u < F ? keys[j0 + 32 * u] : ResKey{~0ull, ~0ull, ~0ull};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool less =
                    o[u].k0 != me.k0 ? o[u].k0 < me.k0 : (o[u].k1 != me.k1 ? o[u].k1 < me.k1 : o[u].k2 < me.k2);
                cnt += less ? 1u : 0u;
            }
        }
        const int64_t pos = (int64_t)__reduce_add_sync(0xFFFFFFFFu, cnt);
        const int32_t r = ids[i];
        for (int w = lane; w < W; w += 32) masks[pos * W + w] = R.mask[(int64_t)r * W + w];
        if (lane == 0) {
            sizes[pos] = R.size[r];
            supports[pos] = R.support[r];
        }
    }
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace dic

using namespace dic;

struct Bucket {
    int32_t* rec = nullptr;
    uint16_t* items = nullptr;
    int32_t* dev_rec = nullptr;      // what the device tables hold
    uint16_t* dev_items = nullptr;
    int64_t dev_cap = 0;
    int64_t n = 0;     // filled slots (live + dead) at the last polled stop
    int64_t cap = 0;
};

// Everything a captured stop graph bakes in: a change forces a re-capture.
struct GraphKey {
    Records R;
    const hent_t* ht;
    int64_t hcap;
    int64_t kuse;
    const unsigned long long* delta;
    const unsigned long long* delta_p;  // fused reduction: the count graph's target
    const int32_t* keep;
    const int32_t* frontier;
    const void* joins;
    int64_t tmp_cap;
    int64_t kuse_status;
    const int64_t* sched;
    int64_t nsched;
    int64_t sched_first, sched_last;  // chunk sizing the pair kernel's grid
    int64_t pair_live;                // the pair kernel is still in the count graph
    bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(*this)) == 0; }
};

static int nccl_fail(ncclResult_t r, const char* what);

// Host-side resources of an engine (the mapped status ring, its events, the
// capture stream) are pooled per process: creating them costs ~1-2 ms
// (page pinning), more than a small mining run's whole checkpoint loop.
struct HostRes {
    unsigned long long* ring = nullptr;
    unsigned long long* ring_dev = nullptr;
    int64_t words = 0;
    int device = -1;
    cudaEvent_t ev[kRing] = {};
    cudaStream_t cap = nullptr;
    uint8_t* stage = nullptr;  // pinned staging for the result copies (grown on demand)
    size_t stage_bytes = 0;
    cudaGraphExec_t gx[4] = {nullptr, nullptr, nullptr, nullptr};  // stop graphs, updated in place by the next engine
};

struct dic_engine {
    const uint32_t* tids;
    int64_t n_local;
    int m, W, KS;
    int64_t need, interval, stop_max;
    int bound;
    cudaStream_t s;

    Records R;
    int64_t nrec = 0;  // at the last polled stop
    hent_t* ht = nullptr;  // hash index (entries: tag << 32 | record id)
    int64_t hcap = 0;

    std::vector<Bucket> buckets;  // index = itemset size
    int kuse = 4;                 // bucket indices < kuse may be non-empty
    int32_t** d_brec = nullptr;   // device copies of the bucket tables
    uint16_t** d_bitems = nullptr;
    int64_t* d_bcap = nullptr;
    int64_t* d_doff = nullptr;     // [KS + 1] per-stop delta offsets
    unsigned long long* d_stat = nullptr;  // status words (see S_*)
    unsigned long long* d_sync = nullptr;  // checkpoint kernel: grid-barrier arrivals, CTAs out
    int64_t slot_cap = 0;          // >= sum of bucket capacities: delta / keep / frontier size

    int32_t* level1 = nullptr;
    int64_t nL1 = 0;
    int32_t* frontier = nullptr;
    int32_t* keep = nullptr;
    unsigned long long* delta = nullptr;

    JoinRec* joins = nullptr;             // the stop's admitted joins (checkpoint kernel: eval -> commit)
    int64_t tmp_cap = 0;

    // the pair bucket as a dense triangle over the frequent items (pairs.cu)
    const uint32_t* pair_tids = nullptr;  // tids restricted to level1 (or tids itself)
    uint32_t* pair_tids_own = nullptr;
    int32_t* rank = nullptr;              // item -> position in level1, -1 if infrequent
    unsigned long long* tri = nullptr;    // [L(L-1)/2] per-stop pair counts
    int64_t tri_len = 0;

    // pipelining
    unsigned long long* ring = nullptr;  // pinned, device-mapped [kRing][S_HEAD + 3*KS] (from hres)
    unsigned long long* ring_dev = nullptr;
    cudaEvent_t* ev = nullptr;           // [kRing] (from hres)
    int64_t ring_words = 0;
    int kuse_at[kRing];                  // kuse when the slot was written
    int64_t issued = 0;                  // stops issued (sequence numbers 0..issued-1)
    int64_t polled = 0;                  // stops polled
    int64_t live = 0;                    // |dashed| after the last polled stop
    int64_t cur_first = 0, cur_last = -1;
    int kuse_issue = 4;                  // kuse of the stop between issue_count and issue_checkpoint
    bool seeded = false;
    bool counted = false;                // issue_count done, issue_checkpoint pending

    // stop graphs: count half (pair + count kernels, chunk read on the device
    // from the schedule slot S_SEQ % nsched) and checkpoint half
    int64_t* d_sched = nullptr;          // [nsched][2] local chunk per stop, rotated so slot = seq % nsched
    std::vector<int64_t> h_sched;
    int64_t nsched = 0;
    cudaStream_t cap_stream = nullptr;   // private stream to capture on (from hres)
    cudaGraphExec_t gx_count = nullptr, gx_ckpt = nullptr;
    long long nk_count = 0, nk_ckpt = 0; // kernels per graph launch
    GraphKey key_count{}, key_ckpt{};
    // dic_engine_run: a scheduled stop is ONE graph (count + checkpoint) when
    // nothing runs between its halves on the host (single GPU, or the fused
    // reduction, which is the count graph's last node)
    bool in_run = false, merged_pending = false;
    cudaGraphExec_t gx_stop = nullptr;
    long long nk_stop = 0;
    GraphKey key_stop{};
    int64_t graphs_captured = 0, graph_launches = 0;
    bool count_graphed = false;          // the pending count went through the graph

    // batches of quiet stops (dic_engine_run): kBatchStops delta blocks of kBatchSlots
    unsigned long long* bdelta = nullptr;
    cudaGraphExec_t gx_batch = nullptr;
    long long nk_batch = 0;
    GraphKey key_batch{};
    int gx_batch_n = 0;
    bool status_ready = false;  // dic_engine_poll: the stop's status is already on the host (batches)
    int64_t batch_launches = 0;  // = the device's launch number (a.sync[3])

    int32_t* res_ids = nullptr;          // result collection (dic_engine_num_frequent)
    int64_t res_cap = 0, res_F = -1;
    HostRes hres;

    // multi-GPU: per-stop sum-allreduce of the count deltas (and of the pair
    // triangle while it is dense) on the engine's stream, between the count
    // and checkpoint halves
    ncclComm_t comm = nullptr;
    bool tri_live = true;                // host view: the pair triangle may still be dense
    // fused reduction: the count kernels write this rank's
    // partial counts into NCCL symmetric windows (delta_p, tri_p); one kernel
    // per stop barriers with the peers over NVLink (LSA team), sums every
    // peer's partial into delta / tri (what the checkpoint reads) and re-zeroes
    // its partials, instead of two ncclAllReduce calls
    bool fused = false;
    ncclDevComm devc{};
    unsigned long long* delta_p = nullptr;
    unsigned long long* tri_p = nullptr;  // + 2 words: the pair kernel's grain counters
    ncclWindow_t win_delta = nullptr, win_tri = nullptr;   // partials
    ncclWindow_t win_dsum = nullptr, win_tsum = nullptr;   // sums (delta, tri) in fused mode
    std::map<const unsigned long long*, int64_t> sym_counts;  // element count of each symmetric buffer held
};

namespace {

std::mutex g_res_mu;
std::vector<HostRes> g_res_pool;

void free_host_res(HostRes& r) {
    for (int i = 0; i < kRing; ++i)
        if (r.ev[i]) cudaEventDestroy(r.ev[i]);
    if (r.ring) cudaFreeHost(r.ring);
    if (r.stage) cudaFreeHost(r.stage);
    for (cudaGraphExec_t& g : r.gx)
        if (g) cudaGraphExecDestroy(g);
    if (r.cap) cudaStreamDestroy(r.cap);
    r = HostRes();
}

int acquire_host_res(int64_t words, HostRes* out) {
    int dev = 0;
    DIC_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_res_mu);
        for (size_t i = 0; i < g_res_pool.size(); ++i)
            if (g_res_pool[i].device == dev && g_res_pool[i].words >= words) {
                *out = g_res_pool[i];
                g_res_pool.erase(g_res_pool.begin() + (long)i);
                return DIC_OK;
            }
    }
    HostRes r;
    r.device = dev;
    r.words = words;
    // the ring, then 8 pinned scratch words
    cudaError_t ce = cudaHostAlloc((void**)&r.ring, ((size_t)kRing * words + 8) * sizeof(unsigned long long),
                                   cudaHostAllocMapped);
    if (ce == cudaSuccess) ce = cudaHostGetDevicePointer((void**)&r.ring_dev, r.ring, 0);
    for (int i = 0; i < kRing && ce == cudaSuccess; ++i) ce = cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&r.cap, cudaStreamNonBlocking);
    if (ce != cudaSuccess) {
        free_host_res(r);
        return cuda_fail(ce, "engine host resources (mapped status ring, events, capture stream)");
    }
    memset(r.ring, 0, ((size_t)kRing * words + 8) * sizeof(unsigned long long));
    *out = r;
    return DIC_OK;
}

void release_host_res(HostRes& r) {
    if (!r.ring) return;
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (g_res_pool.size() < 8) {
        g_res_pool.push_back(r);
        r = HostRes();
    } else {
        free_host_res(r);
    }
}

template <class T>
int dalloc(T** p, int64_t count, cudaStream_t s) {
    *p = nullptr;
    if (count <= 0) count = 1;
    cudaError_t e = cudaMallocAsync((void**)p, (size_t)count * sizeof(T), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    return DIC_OK;
}

template <class T>
void dfree(T*& p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
}

// stream-ordered growth: the copy runs after every kernel already enqueued,
// so the FULL old capacity is copied (host sizes may lag the device)
template <class T>
int dgrow(T** p, int64_t old_cap, int64_t new_cap, cudaStream_t s) {
    T* q = nullptr;
    int rc = dalloc(&q, new_cap, s);
    if (rc) return rc;
    if (*p && old_cap > 0) {
        cudaError_t e = cudaMemcpyAsync(q, *p, (size_t)old_cap * sizeof(T), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(grow)");
    }
    dfree(*p, s);
    *p = q;
    return DIC_OK;
}

int grow_records(dic_engine* e, int64_t need_cap) {
    if (need_cap <= e->R.cap) return DIC_OK;
    const int64_t nc = std::max<int64_t>({need_cap, e->R.cap * 2, (int64_t)4096});
    Records& R = e->R;
    const int64_t oc = R.cap;
    int rc;
    if ((rc = dgrow(&R.mask, oc * e->W, nc * e->W, e->s))) return rc;
    if ((rc = dgrow(&R.hash, oc, nc, e->s))) return rc;
    if ((rc = dgrow(&R.support, oc, nc, e->s))) return rc;
    if ((rc = dgrow(&R.intervals, oc, nc, e->s))) return rc;
    if ((rc = dgrow(&R.size, oc, nc, e->s))) return rc;
    if ((rc = dgrow(&R.shape, oc, nc, e->s))) return rc;
    if ((rc = dgrow(&R.items, oc * 8, nc * 8, e->s))) return rc;
    R.cap = nc;
    return DIC_OK;
}

// the hash index rebuilt from the records (the device's count)
int rebuild_hash(dic_engine* e) {
    ht_clear_kernel<<<nblk(e->hcap), 256, 0, e->s>>>(e->ht, e->hcap);
    ::dic::note_launch();
    ht_insert_records_kernel<<<sm_count() * 8, 256, 0, e->s>>>(e->ht, (uint64_t)e->hcap - 1, e->R,
                                                               e->d_stat + S_NREC);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("rehash");
    return DIC_OK;
}

// keep the hash load factor <= 1/2; rebuild from the records on growth
int ensure_hash(dic_engine* e, int64_t nrec_after) {
    if (nrec_after * 2 <= e->hcap) return DIC_OK;
    int64_t nc = 4096;
    while (nc < nrec_after * 2) nc <<= 1;
    nc = std::max<int64_t>(nc, e->hcap * 2);
    dfree(e->ht, e->s);
    int rc = dalloc(&e->ht, nc, e->s);
    if (rc) return rc;
    e->hcap = nc;
    return rebuild_hash(e);
}

// Push the bucket tables (record / item arrays, capacities) the device has
// not seen yet, as kernel parameters: stream-ordered, no host buffer to keep
// alive, no synchronisation.
int sync_bucket_tables(dic_engine* e) {
    TableUpdate u;
    u.n = 0;
    auto flush = [&]() -> int {
        if (!u.n) return DIC_OK;
        set_tables_kernel<<<1, 32, 0, e->s>>>(e->d_brec, e->d_bitems, e->d_bcap, u);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("set_tables_kernel");
        u.n = 0;
        return DIC_OK;
    };
    int rc;
    for (int k = 0; k < e->KS; ++k) {
        Bucket& b = e->buckets[k];
        if (b.rec == b.dev_rec && b.items == b.dev_items && b.cap == b.dev_cap) continue;
        u.k[u.n] = k;
        u.rec[u.n] = b.rec;
        u.items[u.n] = b.items;
        u.cap[u.n] = b.cap;
        b.dev_rec = b.rec;
        b.dev_items = b.items;
        b.dev_cap = b.cap;
        if (++u.n == TableUpdate::kMax && (rc = flush())) return rc;
    }
    return flush();
}

// NCCL symmetric buffers of the fused reduction.  Allocation + window
// registration is collective and host-synchronous (milliseconds), so buffers
// are pooled per communicator and reused by later engines (a mining run per
// bench step must not re-register); they are released by
// dic_nccl_comm_destroy.  Every rank makes the same calls in the same order:
// sizes and growth points come from the replicated statuses, and the pool's
// best-fit choice depends only on that call sequence.
struct SymBuf {
    unsigned long long* ptr;
    ncclWindow_t win;
    int64_t count;
};
std::mutex g_sym_mu;
std::map<ncclComm_t, std::vector<SymBuf>> g_sym_free;
std::map<ncclComm_t, ncclDevComm> g_devcomm;

int sym_free(dic_engine* e, unsigned long long** p, ncclWindow_t* w) {
    if (!*p) return DIC_OK;
    // kernels already enqueued may still read it; the next user zeroes it on
    // its own (same) stream order only after a host sync, so drain here
    DIC_CUDA(cudaStreamSynchronize(e->s));
    std::lock_guard<std::mutex> lk(g_sym_mu);
    g_sym_free[e->comm].push_back(SymBuf{*p, *w, e->sym_counts[*p]});
    e->sym_counts.erase(*p);
    *p = nullptr;
    *w = nullptr;
    return DIC_OK;
}

int sym_realloc(dic_engine* e, unsigned long long** p, ncclWindow_t* w, int64_t count) {
    int rc;
    if ((rc = sym_free(e, p, w))) return rc;
    count = std::max<int64_t>(count, 1);
    {
        std::lock_guard<std::mutex> lk(g_sym_mu);
        auto& fl = g_sym_free[e->comm];
        int best = -1;
        for (int i = 0; i < (int)fl.size(); ++i)
            if (fl[i].count >= count && (best < 0 || fl[i].count < fl[best].count)) best = i;
        if (best >= 0) {
            *p = fl[best].ptr;
            *w = fl[best].win;
            e->sym_counts[*p] = fl[best].count;
            fl.erase(fl.begin() + best);
        }
    }
    if (!*p) {
        const size_t bytes = (size_t)count * sizeof(unsigned long long);
        void* q = nullptr;
        ncclResult_t r = ncclMemAlloc(&q, bytes);
        if (r != ncclSuccess) return nccl_fail(r, "ncclMemAlloc");
        r = ncclCommWindowRegister(e->comm, q, bytes, w, NCCL_WIN_COLL_SYMMETRIC);
        if (r != ncclSuccess) {
            ncclMemFree(q);
            return nccl_fail(r, "ncclCommWindowRegister");
        }
        *p = static_cast<unsigned long long*>(q);
        e->sym_counts[*p] = count;
    }
    DIC_CUDA(cudaMemsetAsync(*p, 0, (size_t)e->sym_counts[*p] * sizeof(unsigned long long), e->s));
    return DIC_OK;
}

// release every pooled symmetric buffer (and the device communicator) of a
// communicator, before it dies
int sym_pool_release(ncclComm_t comm) {
    std::vector<SymBuf> fl;
    {
        std::lock_guard<std::mutex> lk(g_sym_mu);
        auto dc = g_devcomm.find(comm);
        if (dc != g_devcomm.end()) {
            ncclDevCommDestroy(comm, &dc->second);
            g_devcomm.erase(dc);
        }
        auto it = g_sym_free.find(comm);
        if (it == g_sym_free.end()) return DIC_OK;
        fl.swap(it->second);
        g_sym_free.erase(it);
    }
    for (SymBuf& b : fl) {
        ncclResult_t r = ncclCommWindowDeregister(comm, b.win);
        if (r != ncclSuccess) return nccl_fail(r, "ncclCommWindowDeregister");
        r = ncclMemFree(b.ptr);
        if (r != ncclSuccess) return nccl_fail(r, "ncclMemFree");
    }
    return DIC_OK;
}

// per-stop slot arrays (delta, keep, frontier) cover every bucket capacity
int ensure_slot_arrays(dic_engine* e) {
    int64_t need = 0;
    for (const Bucket& b : e->buckets) need += b.cap;
    need = std::max<int64_t>(need, 1);
    if (need <= e->slot_cap) return DIC_OK;
    const int64_t nc = std::max<int64_t>(need, e->slot_cap + e->slot_cap / 2);
    int rc;
    if (e->fused) {
        // peers write the stop's sums straight into delta: a symmetric window
        if ((rc = sym_realloc(e, &e->delta, &e->win_dsum, nc))) return rc;
    } else {
        dfree(e->delta, e->s);
        if ((rc = dalloc(&e->delta, nc, e->s))) return rc;
        DIC_CUDA(cudaMemsetAsync(e->delta, 0, nc * sizeof(unsigned long long), e->s));  // apply re-zeroes
    }
    dfree(e->keep, e->s);
    if ((rc = dalloc(&e->keep, nc, e->s))) return rc;
    // the frontier of a stop awaiting a candidate replay must survive growth
    if ((rc = dgrow(&e->frontier, e->slot_cap, nc, e->s))) return rc;
    if (e->fused && (rc = sym_realloc(e, &e->delta_p, &e->win_delta, nc))) return rc;
    e->slot_cap = nc;
    return DIC_OK;
}

int grow_bucket(dic_engine* e, int k, int64_t need_cap, bool* changed) {
    Bucket& b = e->buckets[k];
    if (need_cap <= b.cap) return DIC_OK;
    const int64_t nc = std::max<int64_t>({need_cap, b.cap * 2, (int64_t)1024});
    int rc;
    if ((rc = dgrow(&b.rec, b.cap, nc, e->s))) return rc;
    if ((rc = dgrow(&b.items, b.cap * k, nc * k, e->s))) return rc;
    b.cap = nc;
    *changed = true;
    e->kuse = std::max(e->kuse, std::min(k + 2, e->KS));
    if (e->kuse > kDoffMax) {
        set_error("dic_engine: itemsets of more than %d items are not supported", kDoffMax - 2);
        return DIC_EINVAL;
    }
    return DIC_OK;
}

int ensure_tmp(dic_engine* e, int64_t want) {
    if (want <= e->tmp_cap) return DIC_OK;
    const int64_t nc = std::max<int64_t>(want, e->tmp_cap * 2);
    dfree(e->joins, e->s);
    int rc;
    if ((rc = dalloc(&e->joins, nc, e->s))) return rc;
    e->tmp_cap = nc;
    return DIC_OK;
}

// Headroom for the stops in flight: >= 64k join slots and record / hash room,
// every bucket of size >= 3 in use (and the next three) with room to grow by half (>= 4096), the
// next size up allocated, slot arrays covering the capacities.
int ensure_headroom(dic_engine* e) {
    int rc;
    const int64_t room = std::max<int64_t>(1 << 16, e->nrec / 2);
    if ((rc = ensure_tmp(e, 1 << 16))) return rc;
    if ((rc = grow_records(e, e->nrec + room))) return rc;
    if ((rc = ensure_hash(e, e->nrec + room))) return rc;
    bool changed = false;
    int top = 2;
    for (int k = 2; k < e->KS; ++k)
        if (e->buckets[k].n > 0) top = k;
    // sizes up to three above the largest live one: with stops in flight a
    // new level can spawn the next before the host sees it (each miss is an
    // abort + replay round trip)
    for (int k = 3; k <= std::min(top + 3, e->KS - 1); ++k) {  // pairs are only ever seeded
        const Bucket& b = e->buckets[k];
        const int64_t want = b.n + std::max<int64_t>(4096, b.n / 2);
        if (want > b.cap && (rc = grow_bucket(e, k, want, &changed))) return rc;
    }
    if ((rc = ensure_slot_arrays(e))) return rc;
    if (changed && (rc = sync_bucket_tables(e))) return rc;
    return DIC_OK;
}

// CTAs of the checkpoint kernel: one per SM.  DIC_CKPT_CTAS overrides it (the
// layout-determinism tests vary it: the work split and the timing of every
// atomic change, the committed layout must not).
static int ckpt_ctas() {
    const char* env = getenv("DIC_CKPT_CTAS");
    const int v = env && *env ? atoi(env) : 0;
    return v > 0 ? std::min(v, sm_count()) : sm_count();
}

// The checkpoint half of a stop as one cooperative launch (every CTA is
// resident, so the grid-wide barriers cannot deadlock): apply + prune +
// finalize over every slot, compaction of the flagged buckets,
// make_candidates (device-sized, all-or-nothing), status.  replay: the
// candidate step alone (overflow recovery).
CkptArgs checkpoint_args(dic_engine* e, bool replay) {
    CkptArgs a;
    memset(&a, 0, sizeof(a));
    a.rec_tab = e->d_brec;
    a.items_tab = e->d_bitems;
    a.bcap = e->d_bcap;
    a.doff = e->d_doff;
    a.delta = e->delta;
    a.R = e->R;
    a.need = e->need;
    a.interval = e->interval;
    a.stop_max = e->stop_max;
    a.frontier = e->frontier;
    a.keep = e->keep;
    a.stat = e->d_stat;
    a.pa = PairArgs{e->tri, e->rank, e->nL1, e->tri ? e->tri_len : 0, (int64_t)e->m};
    a.level1 = e->level1;
    a.ht = e->ht;
    a.hmask = (uint64_t)e->hcap - 1;
    a.joins = e->joins;
    a.tmp_cap = e->tmp_cap;
    a.rec_cap = e->R.cap;
    a.hcap = e->hcap;
    a.ring = e->ring_dev;
    a.ring_words = e->ring_words;
    a.sync = e->d_sync;
    a.W = e->W;
    a.KS = e->KS;
    a.kuse_issue = replay ? e->kuse : e->kuse_issue;
    a.kuse = e->kuse;
    a.bound = e->bound;
    a.replay = replay ? 1 : 0;
    return a;
}

int launch_checkpoint(dic_engine* e, cudaStream_t s, bool replay = false) {
    CkptArgs a = checkpoint_args(e, replay);
    void* params[] = {&a};
    static const bool coop = [] {
        const char* env = getenv("DIC_CKPT_COOP");
        return !(env && atoi(env) == 0);
    }();
    static bool attr = false;
    if (!attr) {
        DIC_CUDA(cudaFuncSetAttribute(checkpoint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageBytes));
        attr = true;
    }
    if (coop) {
        DIC_CUDA(cudaLaunchCooperativeKernel((const void*)checkpoint_kernel, dim3((unsigned)ckpt_ctas()),
                                             dim3(kCkptThreads), params, kStageBytes, s));
    } else {
        checkpoint_kernel<<<ckpt_ctas(), kCkptThreads, kStageBytes, s>>>(a);
        DIC_CHECK_LAUNCH("checkpoint_kernel");
    }
    ::dic::note_launch();
    return DIC_OK;
}

// A batch of quiet stops (checkpoint_batch_kernel): one count launch over the
// next n chunks into the batch's delta blocks, then their checkpoints on one CTA.
int launch_batch(dic_engine* e, int n, cudaStream_t s) {
    const unsigned long long* bn = e->d_stat + S_HEAD + 2 * e->KS;
    int rc;
    if ((rc = count_dev_launch(e->tids, e->n_local, e->m, 0, e->n_local > 0 ? e->n_local - 1 : 0, e->kuse_issue,
                               e->d_bitems, bn, e->d_doff, e->bdelta, e->d_stat + S_ABORT,
                               e->tri ? e->tri_len : 0, s, e->d_sched, e->d_stat + S_SEQ, (int)e->nsched, n,
                               kBatchSlots)))
        return rc;
    const CkptArgs a = checkpoint_args(e, false);
    // (the report words: two of the pinned scratch words past the status ring)
    checkpoint_batch_kernel<<<1, kCkptThreads, 0, s>>>(a, n, e->bdelta, e->ring_dev + kRing * e->hres.words + 2);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("checkpoint_batch_kernel");
    return DIC_OK;
}

// Fused reduction of a stop's counts over NVLink peer memory (SURVEY 8(f)
// row 1): one launch instead of two ncclAllReduce calls, sized on the device
// by the live slots (doff[kuse]) instead of the slot capacity.  A reduce-
// scatter + all-gather over the LSA team (every rank in one NVLink domain):
// the slots are cut into G x P slices; CTA b of rank r owns slice (b, r).
//   1. LSA barrier b: CTA b of every rank has started, so every rank's count
//      kernels (earlier on its stream) have finished their partials;
//   2. the owner sums slice (b, r) over the P partials (peer loads) and stores
//      the sum into every rank's sum buffer (peer stores): (P-1)/P of the data
//      in and out per rank, like a ring or NVLS allreduce;
//   3. LSA barrier b again: every rank's CTA b has read slices (b, *) of this
//      rank's partials and delivered its sums, so CTA b re-zeroes slices
//      (b, *) of the local partials for the next stop's count.
// The checkpoint graph then reads the local sums (delta / tri) exactly as on
// one GPU.  Every rank runs both barriers whatever its data (abort and
// density are replicated decisions), so the barrier epochs stay matched.
__device__ __forceinline__ void fused_slices(ncclWindow_t wpart, ncclWindow_t wsum, int64_t n, int P, int me,
                                             unsigned long long* const* part, unsigned long long* const* sum) {
    const int64_t S = (int64_t)gridDim.x * P;
    const int64_t q = (int64_t)blockIdx.x * P + me;
    const int64_t lo = n * q / S, hi = n * (q + 1) / S;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        unsigned long long v = 0;
        for (int p = 0; p < P; ++p) v += part[p][i];
        for (int p = 0; p < P; ++p) sum[p][i] = v;
    }
}

__device__ __forceinline__ void fused_zero(unsigned long long* mine, int64_t n, int P) {
    const int64_t S = (int64_t)gridDim.x * P;
    const int64_t lo = n * ((int64_t)blockIdx.x * P) / S, hi = n * ((int64_t)blockIdx.x * P + P) / S;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) mine[i] = 0;
}

__global__ void __launch_bounds__(256) fused_reduce_kernel(ncclDevComm dc, ncclWindow_t wdp, ncclWindow_t wds,
                                                           ncclWindow_t wtp, ncclWindow_t wts,
                                                           const int64_t* __restrict__ doff, int kuse,
                                                           int64_t tri_len, const unsigned long long* bn2,
                                                           const unsigned long long* abort_flag) {
    __shared__ unsigned long long* ptr[4][kFusedMaxPeers];  // delta part / sum, tri part / sum per peer
    const int P = dc.lsaSize, me = dc.lsaRank;
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        ptr[0][p] = static_cast<unsigned long long*>(ncclGetLsaPointer(wdp, 0, p));
        ptr[1][p] = static_cast<unsigned long long*>(ncclGetLsaPointer(wds, 0, p));
        if (wtp) {
            ptr[2][p] = static_cast<unsigned long long*>(ncclGetLsaPointer(wtp, 0, p));
            ptr[3][p] = static_cast<unsigned long long*>(ncclGetLsaPointer(wts, 0, p));
        }
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);  // also publishes ptr[][] to the CTA
    const bool skip = *abort_flag != 0;
    const int64_t nlive = skip ? 0 : doff[kuse];
    const bool dense = !skip && wtp != nullptr && tri_len > 0 && 2 * (int64_t)*bn2 >= tri_len;
    fused_slices(wdp, wds, nlive, P, me, ptr[0], ptr[1]);
    if (dense) fused_slices(wtp, wts, tri_len, P, me, ptr[2], ptr[3]);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    fused_zero(ptr[0][me], nlive, P);
    if (dense) fused_zero(ptr[2][me], tri_len, P);
}

int launch_fused_reduce(dic_engine* e, cudaStream_t s) {
    const unsigned long long* bn = e->d_stat + S_HEAD + 2 * e->KS;
    fused_reduce_kernel<<<kFusedCtas, 256, 0, s>>>(e->devc, e->win_delta, e->win_dsum, e->tri ? e->win_tri : nullptr,
                                                   e->tri ? e->win_tsum : nullptr, e->d_doff, (int)e->kuse_issue,
                                                   e->tri ? e->tri_len : 0, bn + 2, e->d_stat + S_ABORT);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("fused_reduce_kernel");
    return DIC_OK;
}

// the count half: the pair triangle and every dashed bucket over the chunk
// [lfirst, llast]; sched != nullptr: the chunk is read on the device from the
// schedule slot S_SEQ % nsched ([lfirst, llast] then only sizes the grid)
int launch_count(dic_engine* e, int64_t lfirst, int64_t llast, const int64_t* sched, cudaStream_t s) {
    const unsigned long long* abort_flag = e->d_stat + S_ABORT;
    const unsigned long long* bn = e->d_stat + S_HEAD + 2 * e->KS;
    const unsigned long long* seq = e->d_stat + S_SEQ;
    const int ring = (int)e->nsched;
    int rc;
    // once the host has seen the pair bucket leave dense mode (it never
    // returns) the pair kernel, a no-op from then on, leaves the graph
    if (e->tri && e->tri_live) {
        // the pair kernel's grain counters live past the triangle (tri[tri_len..+2));
        // fused reduction: this rank's partial triangle in its symmetric window
        unsigned long long* tri = e->fused ? e->tri_p : e->tri;
        if ((rc = count_pairs_dev_launch(e->pair_tids, e->n_local, (int)e->nL1, lfirst, llast, tri, bn + 2,
                                         e->tri_len, abort_flag, s, sched, seq, ring, tri + e->tri_len)))
            return rc;
    }
    if ((rc = count_dev_launch(e->tids, e->n_local, e->m, lfirst, llast, e->kuse_issue, e->d_bitems, bn, e->d_doff,
                               e->fused ? e->delta_p : e->delta, abort_flag, e->tri ? e->tri_len : 0, s, sched,
                               seq, ring)))
        return rc;
    // sharded, fused: the cross-rank sum of this stop's partials over NVLink
    return e->fused ? launch_fused_reduce(e, s) : DIC_OK;
}

GraphKey graph_key(const dic_engine* e, bool with_sched) {
    GraphKey k;
    memset(&k, 0, sizeof(k));
    k.R = e->R;
    k.ht = e->ht;
    k.hcap = e->hcap;
    k.kuse = e->kuse_issue;
    k.delta = e->delta;
    k.delta_p = e->delta_p;
    k.pair_live = e->tri && e->tri_live;
    k.keep = e->keep;
    k.frontier = e->frontier;
    k.joins = e->joins;
    k.tmp_cap = e->tmp_cap;
    k.kuse_status = e->kuse;
    if (with_sched) {
        k.sched = e->d_sched;
        k.nsched = e->nsched;
        // the chunk with the most tiles sizes the pair kernel's grid
        int64_t best = -1;
        for (int64_t i = 0; i < e->nsched; ++i) {
            const int64_t f = e->h_sched[2 * i], l = e->h_sched[2 * i + 1];
            if (l < f) continue;
            const int64_t nt = (l >> 5) - (f >> 5);
            if (nt > best) {
                best = nt;
                k.sched_first = f;
                k.sched_last = l;
            }
        }
        if (best < 0) k.sched_last = -1;
    }
    return k;
}

// Capture `body` on the private stream into *gx (replacing it); the kernels it
// noted are re-noted per graph launch instead.
template <class F>
int capture_graph(dic_engine* e, cudaGraphExec_t* gx, long long* nk, F body) {
    const long long before = (long long)dic_launch_count();
    DIC_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeRelaxed));
    const int rc = body(e->cap_stream);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &g);
    const long long n = (long long)dic_launch_count() - before;
    ::dic::note_launches(-n);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
    if (*gx) {
        // same topology (the usual case): update the executable graph's
        // parameters in place, far cheaper than a new instantiation
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(*gx, g, &info) == cudaSuccess) {
            cudaGraphDestroy(g);
            *nk = n;
            ++e->graphs_captured;
            return DIC_OK;
        }
        cudaGetLastError();  // clear the update failure
        cudaGraphExecDestroy(*gx);
        *gx = nullptr;
    }
    const cudaError_t ie = cudaGraphInstantiate(gx, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return cuda_fail(ie, "cudaGraphInstantiate");
    *nk = n;
    ++e->graphs_captured;
    return DIC_OK;
}

int launch_graph(dic_engine* e, cudaGraphExec_t gx, long long nk) {
    DIC_CUDA(cudaGraphLaunch(gx, e->s));
    ::dic::note_launches(nk);
    ++e->graph_launches;
    return DIC_OK;
}

}  // namespace

extern "C" int dic_engine_create(const uint32_t* tids, int64_t n_local, int32_t m, int64_t need, int64_t interval,
                                 int64_t stop_max, int32_t prune_bound, void* stream, dic_engine** out) {
    DIC_REQUIRE(out, "dic_engine_create: out is null");
    DIC_REQUIRE(m >= 1 && m <= 65535, "dic_engine_create: m=%d outside [1, 65535]", m);
    DIC_REQUIRE(n_local >= 0 && (tids || n_local == 0), "dic_engine_create: bad tids/n_local");
    DIC_REQUIRE(interval >= 1 && stop_max >= 1, "dic_engine_create: bad interval/stop_max");
    retain_pool();
    dic_engine* e = new dic_engine();
    e->tids = tids;
    e->n_local = n_local;
    e->m = m;
    e->W = (m + 63) / 64;
    e->KS = m + 2;
    e->kuse = std::min(4, e->KS);
    e->need = need;
    e->interval = interval;
    e->stop_max = stop_max;
    e->bound = prune_bound ? 1 : 0;
    e->s = as_stream(stream);
    e->buckets.resize(e->KS);
    const int KS = e->KS;
    e->ring_words = S_HEAD + 3 * (int64_t)KS;
    int rc = 0;
    if ((rc = dalloc(&e->d_brec, KS, e->s)) || (rc = dalloc(&e->d_bitems, KS, e->s)) ||
        (rc = dalloc(&e->d_bcap, KS, e->s)) || (rc = dalloc(&e->d_doff, KS + 1, e->s)) ||
        (rc = dalloc(&e->d_stat, e->ring_words + KS, e->s)) || (rc = dalloc(&e->level1, m, e->s)) ||
        (rc = dalloc(&e->d_sync, 4 + 2048, e->s)) ||
        (rc = dalloc(&e->bdelta, (int64_t)kBatchStops * kBatchSlots, e->s))) {
        delete e;
        return rc;
    }
    if ((rc = acquire_host_res(e->ring_words, &e->hres))) {
        delete e;
        return rc;
    }
    e->ring = e->hres.ring;
    e->ring_dev = e->hres.ring_dev;
    e->ev = e->hres.ev;
    e->cap_stream = e->hres.cap;
    e->gx_count = e->hres.gx[0];  // stale until the first capture updates them
    e->gx_ckpt = e->hres.gx[1];
    e->gx_stop = e->hres.gx[2];
    e->gx_batch = e->hres.gx[3];
    e->hres.gx[0] = e->hres.gx[1] = e->hres.gx[2] = e->hres.gx[3] = nullptr;
    for (int i = 0; i < kRing; ++i) e->kuse_at[i] = 0;
    cudaMemsetAsync(e->d_stat, 0, (e->ring_words + KS) * sizeof(unsigned long long), e->s);
    cudaMemsetAsync(e->d_sync, 0, (4 + 2048) * sizeof(unsigned long long), e->s);
    cudaMemsetAsync(e->bdelta, 0, (size_t)kBatchStops * kBatchSlots * sizeof(unsigned long long), e->s);
    cudaMemsetAsync(e->d_brec, 0, KS * sizeof(int32_t*), e->s);
    cudaMemsetAsync(e->d_bitems, 0, KS * sizeof(uint16_t*), e->s);
    cudaMemsetAsync(e->d_bcap, 0, KS * sizeof(int64_t), e->s);
    *out = e;
    return DIC_OK;
}

extern "C" int dic_engine_destroy(dic_engine* e) {
    if (!e) return DIC_OK;
    cudaStream_t s = e->s;
    cudaStreamSynchronize(s);
    Records& R = e->R;
    dfree(R.mask, s); dfree(R.hash, s); dfree(R.support, s); dfree(R.intervals, s); dfree(R.size, s);
    dfree(R.shape, s); dfree(R.items, s);
    dfree(e->ht, s);
    for (Bucket& b : e->buckets) { dfree(b.rec, s); dfree(b.items, s); }
    dfree(e->d_brec, s); dfree(e->d_bitems, s); dfree(e->d_bcap, s); dfree(e->d_doff, s); dfree(e->d_stat, s);
    dfree(e->level1, s); dfree(e->frontier, s); dfree(e->keep, s);
    if (!e->fused) dfree(e->delta, s);
    dfree(e->d_sched, s);
    dfree(e->joins, s); dfree(e->d_sync, s); dfree(e->bdelta, s);
    dfree(e->pair_tids_own, s); dfree(e->rank, s); dfree(e->res_ids, s);
    if (!e->fused) dfree(e->tri, s);
    if (e->fused) {
        sym_free(e, &e->delta_p, &e->win_delta);
        sym_free(e, &e->tri_p, &e->win_tri);
        sym_free(e, &e->delta, &e->win_dsum);
        sym_free(e, &e->tri, &e->win_tsum);
    }
    e->hres.gx[0] = e->gx_count;  // pooled with the host resources
    e->hres.gx[1] = e->gx_ckpt;
    e->hres.gx[2] = e->gx_stop;
    e->hres.gx[3] = e->gx_batch;
    release_host_res(e->hres);  // the stream was synchronised above: no stop reads the ring any more
    delete e;
    return DIC_OK;
}

extern "C" int dic_engine_words(dic_engine* e) { return e ? e->W : DIC_EINVAL; }

#ifdef DIC_LAB_TIMING
extern "C" int dic_lab_commit_stamps(unsigned long long* host) {
    cudaDeviceSynchronize();
    DIC_CUDA(cudaMemcpyFromSymbol(host, g_lab_commit, sizeof(g_lab_commit)));
    return DIC_OK;
}
#endif

extern "C" int dic_engine_item_counts(dic_engine* e, int64_t* counts) {
    DIC_REQUIRE(e && counts, "dic_engine_item_counts: null argument");
    DIC_CUDA(cudaMemsetAsync(counts, 0, (size_t)e->m * sizeof(int64_t), e->s));
    int rc;
    if (e->n_local > 0 && (rc = item_support_launch(e->tids, e->n_local, e->m, 0, e->n_local - 1,
                                                     reinterpret_cast<unsigned long long*>(counts), e->s)))
        return rc;
    if (e->comm) {  // first_pass over the global database
        const ncclResult_t r = ncclAllReduce(counts, counts, (size_t)e->m, ncclInt64, ncclSum, e->comm, e->s);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(item counts)");
    }
    return DIC_OK;
}

extern "C" int dic_nccl_unique_id(uint8_t* out) {
    DIC_REQUIRE(out, "dic_nccl_unique_id: null buffer");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return DIC_OK;
}

extern "C" int dic_nccl_comm_init(const uint8_t* id_bytes, int32_t nranks, int32_t rank, void** comm) {
    DIC_REQUIRE(id_bytes && comm && nranks >= 1 && 0 <= rank && rank < nranks, "dic_nccl_comm_init: bad arguments");
    ncclUniqueId id;
    memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    const ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return DIC_OK;
}

extern "C" int dic_nccl_comm_destroy(void* comm) {
    if (!comm) return DIC_OK;
    const int rc = sym_pool_release(static_cast<ncclComm_t>(comm));
    if (rc) return rc;
    const ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
    return r == ncclSuccess ? DIC_OK : nccl_fail(r, "ncclCommDestroy");
}

extern "C" int dic_engine_set_comm(dic_engine* e, void* comm) {
    DIC_REQUIRE(e, "dic_engine_set_comm: null engine");
    if (e->seeded) {
        set_error("dic_engine_set_comm: set the communicator before dic_engine_item_counts / seed");
        return DIC_ESTATE;
    }
    e->comm = static_cast<ncclComm_t>(comm);
    e->fused = false;
    // the fused reduction needs every rank in one load/store-accessible (LSA)
    // team, i.e. one NVLink domain; DIC_FUSED_REDUCE=0 keeps ncclAllReduce
    const char* env = getenv("DIC_FUSED_REDUCE");
    if (e->comm && !(env && atoi(env) == 0)) {
        int nranks = 0;
        ncclResult_t r = ncclCommCount(e->comm, &nranks);
        if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
        if (ncclTeamLsa(e->comm).nRanks == nranks && nranks <= kFusedMaxPeers) {
            // one device communicator per NCCL communicator, kept with the pool
            std::lock_guard<std::mutex> lk(g_sym_mu);
            auto it = g_devcomm.find(e->comm);
            if (it == g_devcomm.end()) {
                ncclDevCommRequirements reqs;
                memset(&reqs, 0, sizeof(reqs));
                reqs.lsaBarrierCount = kFusedCtas;
                ncclDevComm dc;
                r = ncclDevCommCreate(e->comm, &reqs, &dc);
                // no device API on this communicator (e.g. no symmetric
                // memory support): keep the ncclAllReduce path
                if (r == ncclSuccess) it = g_devcomm.emplace(e->comm, dc).first;
            }
            if (it != g_devcomm.end()) {
                e->devc = it->second;
                e->fused = true;
            }
        }
    }
    return DIC_OK;
}

extern "C" int dic_engine_collective_mode(dic_engine* e) {
    DIC_REQUIRE(e, "dic_engine_collective_mode: null engine");
    return e->comm ? (e->fused ? 2 : 1) : 0;
}

extern "C" int dic_engine_seed(dic_engine* e, const int64_t* counts, int64_t* n_level1, int64_t* n_pairs) {
    DIC_REQUIRE(e && counts, "dic_engine_seed: null argument");
    if (e->seeded) { set_error("dic_engine_seed: engine already seeded"); return DIC_ESTATE; }
    const int m = e->m;
    std::vector<int64_t> hc(m);
    DIC_CUDA(cudaMemcpyAsync(hc.data(), counts, m * sizeof(int64_t), cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    std::vector<int32_t> l1;
    for (int i = 0; i < m; ++i)
        if (hc[i] >= e->need) l1.push_back(i);
    const int64_t L = (int64_t)l1.size();
    const int64_t npairs = L * (L - 1) / 2;
    int rc;
    e->nrec = m + npairs;
    // device record count first: the hash build reads it
    std::vector<unsigned long long> head(S_HEAD, 0), bn(e->KS, 0);
    head[S_NREC] = (unsigned long long)e->nrec;
    if (e->KS > 2) bn[2] = (unsigned long long)npairs;
    DIC_CUDA(cudaMemcpyAsync(e->d_stat, head.data(), S_HEAD * 8, cudaMemcpyHostToDevice, e->s));
    DIC_CUDA(cudaMemcpyAsync(e->d_stat + S_HEAD + 2 * e->KS, bn.data(), e->KS * 8, cudaMemcpyHostToDevice, e->s));
    const int64_t room = std::max<int64_t>(1 << 16, (m + npairs) / 2);
    if ((rc = grow_records(e, m + npairs + room))) return rc;
    seed_singletons_kernel<<<nblk(m), 256, 0, e->s>>>(e->R, e->W, m, counts, e->need, e->stop_max);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("seed_singletons_kernel");
    if (L > 0) DIC_CUDA(cudaMemcpyAsync(e->level1, l1.data(), L * sizeof(int32_t), cudaMemcpyHostToDevice, e->s));
    e->nL1 = L;
    bool changed = false;
    if (e->KS > 3) {
        if ((rc = grow_bucket(e, 2, std::max<int64_t>(npairs, 1024), &changed))) return rc;
        if ((rc = grow_bucket(e, 3, 4096, &changed))) return rc;
    }
    if (npairs > 0) {
        std::vector<int64_t> rs(L);
        int64_t acc = 0;
        for (int64_t a = 0; a < L; ++a) { rs[a] = acc; acc += L - 1 - a; }
        int64_t* d_rs = nullptr;
        if ((rc = dalloc(&d_rs, L, e->s))) return rc;
        DIC_CUDA(cudaMemcpyAsync(d_rs, rs.data(), L * sizeof(int64_t), cudaMemcpyHostToDevice, e->s));
        seed_pairs_kernel<<<nblk(npairs), 256, 0, e->s>>>(e->R, e->W, e->level1, L, d_rs, npairs, m,
                                                          e->buckets[2].rec, e->buckets[2].items);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("seed_pairs_kernel");
        dfree(d_rs, e->s);
        e->buckets[2].n = npairs;
    }
    if ((rc = ensure_hash(e, m + npairs + room))) return rc;  // builds from the device record count
    // dense pair counting over the frequent items
    std::vector<int32_t> rank(m, -1);
    if (L >= 2 && e->n_local > 0) {
        for (int64_t a = 0; a < L; ++a) rank[l1[a]] = (int32_t)a;
        if ((rc = dalloc(&e->rank, m, e->s))) return rc;
        DIC_CUDA(cudaMemcpyAsync(e->rank, rank.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice, e->s));
        if (L == m) {
            e->pair_tids = e->tids;  // every item frequent: level1 == identity
        } else {
            if ((rc = dalloc(&e->pair_tids_own, dic_tids_words(e->n_local, (int32_t)L), e->s))) return rc;
            if ((rc = tids_select_launch(e->tids, e->n_local, m, e->level1, (int)L, e->pair_tids_own, e->s)))
                return rc;
            e->pair_tids = e->pair_tids_own;
        }
        e->tri_len = npairs;
        // + 2 words: the pair kernel's grain counters (it re-zeroes them itself)
        if (e->fused) {
            if ((rc = sym_realloc(e, &e->tri, &e->win_tsum, npairs + 2))) return rc;
            if ((rc = sym_realloc(e, &e->tri_p, &e->win_tri, npairs + 2))) return rc;
        } else {
            if ((rc = dalloc(&e->tri, npairs + 2, e->s))) return rc;
            DIC_CUDA(cudaMemsetAsync(e->tri, 0, (npairs + 2) * sizeof(unsigned long long), e->s));  // gather re-zeroes
        }
    }
    if ((rc = ensure_headroom(e))) return rc;
    // per-stop counters zero, first stop's delta offsets
    status_kernel<<<1, 32, 0, e->s>>>(e->d_stat, e->KS, e->kuse, nullptr, 0, e->d_doff);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("status_kernel");
    if ((rc = sync_bucket_tables(e))) return rc;
    DIC_CUDA(cudaStreamSynchronize(e->s));  // the host vectors above die at return
    e->live = npairs;
    e->seeded = true;
    if (n_level1) *n_level1 = L;
    if (n_pairs) *n_pairs = npairs;
    return DIC_OK;
}

// ---------------------------------------------------------------------------
// pipelined stop API
// ---------------------------------------------------------------------------
extern "C" int dic_engine_issue_count(dic_engine* e, int64_t lfirst, int64_t llast) {
    DIC_REQUIRE(e, "dic_engine_issue_count: null engine");
    if (!e->seeded || e->counted) {
        set_error("dic_engine_issue_count: engine not seeded or checkpoint pending");
        return DIC_ESTATE;
    }
    DIC_REQUIRE(lfirst >= 0 && (llast < lfirst || llast < e->n_local),
                "dic_engine_count: local chunk [%lld, %lld] outside %lld local rows", (long long)lfirst,
                (long long)llast, (long long)e->n_local);
    int rc;
    e->cur_first = lfirst;
    e->cur_last = llast;
    e->kuse_issue = e->kuse;
    const int64_t sl = e->nsched ? e->issued % e->nsched : 0;
    const bool empty = llast < lfirst;
    if (e->nsched && (empty ? e->h_sched[2 * sl + 1] < e->h_sched[2 * sl]
                            : e->h_sched[2 * sl] == lfirst && e->h_sched[2 * sl + 1] == llast)) {
        // the scheduled chunk: one graph launch (re-captured when its baked-in
        // pointers / sizes changed) — or, inside dic_engine_run with no host
        // step between the halves, deferred into the stop graph
        if (e->in_run && (!e->comm || e->fused)) {
            e->merged_pending = true;
            e->counted = true;
            return DIC_OK;
        }
        const GraphKey k = graph_key(e, true);
        if (!e->gx_count || !(k == e->key_count)) {
            if ((rc = capture_graph(e, &e->gx_count, &e->nk_count, [&](cudaStream_t cs) {
                     return launch_count(e, k.sched_first, k.sched_last, e->d_sched, cs);
                 })))
                return rc;
            e->key_count = k;
        }
        if ((rc = launch_graph(e, e->gx_count, e->nk_count))) return rc;
    } else if (!empty) {
        if ((rc = launch_count(e, lfirst, llast, nullptr, e->s))) return rc;
    }
    e->counted = true;
    return DIC_OK;
}

extern "C" int dic_engine_set_schedule(dic_engine* e, const int64_t* lfirst, const int64_t* llast, int64_t nstops) {
    DIC_REQUIRE(e && lfirst && llast && nstops >= 1, "dic_engine_set_schedule: bad arguments");
    for (int64_t i = 0; i < nstops; ++i)
        DIC_REQUIRE(lfirst[i] >= 0 && (llast[i] < lfirst[i] || llast[i] < e->n_local),
                    "dic_engine_set_schedule: chunk %lld [%lld, %lld] outside %lld local rows", (long long)i,
                    (long long)lfirst[i], (long long)llast[i], (long long)e->n_local);
    // rotate so that the stop with sequence number s reads slot s % nstops
    std::vector<int64_t> h(2 * nstops);
    for (int64_t i = 0; i < nstops; ++i) {
        const int64_t sl = (e->issued + i) % nstops;
        h[2 * sl] = lfirst[i];
        h[2 * sl + 1] = llast[i];
    }
    int rc;
    // in-flight stops may still read the old table: replace, never overwrite
    dfree(e->d_sched, e->s);
    if ((rc = dalloc(&e->d_sched, 2 * nstops, e->s))) return rc;
    DIC_CUDA(cudaMemcpyAsync(e->d_sched, h.data(), h.size() * sizeof(int64_t), cudaMemcpyHostToDevice, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));  // h dies at return
    e->h_sched.swap(h);
    e->nsched = nstops;
    return DIC_OK;
}

extern "C" int dic_engine_graph_stats(dic_engine* e, int64_t* graphs_captured, int64_t* graph_launches) {
    DIC_REQUIRE(e && graphs_captured && graph_launches, "dic_engine_graph_stats: null argument");
    *graphs_captured = e->graphs_captured;
    *graph_launches = e->graph_launches;
    return DIC_OK;
}

extern "C" int dic_engine_delta(dic_engine* e, void** ptr, int64_t* len) {
    DIC_REQUIRE(e && ptr && len, "dic_engine_delta: null argument");
    *ptr = e->delta;
    *len = e->slot_cap;  // zero beyond the live slots: a fixed-size sum-allreduce is exact
    return DIC_OK;
}

extern "C" int dic_engine_pair_counts(dic_engine* e, void** ptr, int64_t* len) {
    DIC_REQUIRE(e && ptr && len, "dic_engine_pair_counts: null argument");
    *ptr = e->tri;
    *len = e->tri ? e->tri_len : 0;
    return DIC_OK;
}

// Diagnostics: bucket k (record ids and item lists, live and dead slots) as
// the device holds it now.  Synchronises the engine's stream.
extern "C" int dic_engine_bucket(dic_engine* e, int32_t k, int32_t* rec_host, uint16_t* items_host, int64_t cap,
                                 int64_t* n) {
    DIC_REQUIRE(e && n && k >= 1 && k < e->KS, "dic_engine_bucket: bad arguments");
    unsigned long long* pin = e->hres.ring + kRing * e->hres.words;
    DIC_CUDA(cudaMemcpyAsync(pin, e->d_stat + S_HEAD + 2 * e->KS + k, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    const int64_t fill = (int64_t)pin[0];
    *n = fill;
    if (fill == 0 || !rec_host) return DIC_OK;
    DIC_REQUIRE(items_host && cap >= fill, "dic_engine_bucket: cap %lld < %lld slots", (long long)cap,
                (long long)fill);
    const Bucket& b = e->buckets[k];
    DIC_CUDA(cudaMemcpyAsync(rec_host, b.rec, (size_t)fill * sizeof(int32_t), cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaMemcpyAsync(items_host, b.items, (size_t)fill * k * sizeof(uint16_t), cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    return DIC_OK;
}

static int nccl_fail(ncclResult_t r, const char* what) {
    set_error("%s: %s", what, ncclGetErrorString(r));
    return DIC_ECUDA;
}

// The stop's cross-rank reduction (sharded engines): every rank enqueues the
// same calls in the same order (the state machine and hence slot_cap /
// tri_live are replicated), so the collectives always match.

static int reduce_stop(dic_engine* e) {
    if (!e->comm) return DIC_OK;
    if (e->fused) return DIC_OK;  // the count graph ends with fused_reduce_kernel
    ncclResult_t r = ncclAllReduce(e->delta, e->delta, (size_t)e->slot_cap, ncclUint64, ncclSum, e->comm, e->s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(delta)");
    if (e->tri && e->tri_live) {
        r = ncclAllReduce(e->tri, e->tri, (size_t)e->tri_len, ncclUint64, ncclSum, e->comm, e->s);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(pair triangle)");
    }
    return DIC_OK;
}

extern "C" int dic_engine_issue_checkpoint(dic_engine* e, int64_t* seq) {
    DIC_REQUIRE(e && seq, "dic_engine_issue_checkpoint: null argument");
    if (!e->counted) { set_error("dic_engine_issue_checkpoint: no count issued"); return DIC_ESTATE; }
    if (e->issued - e->polled >= kRing - 1) {
        set_error("dic_engine_issue_checkpoint: more than %d stops in flight", kRing - 1);
        return DIC_ESTATE;
    }
    e->counted = false;
    int rc;
    if (e->merged_pending) {
        // count + checkpoint of a scheduled stop as one graph launch
        e->merged_pending = false;
        const GraphKey k = graph_key(e, true);
        if (!e->gx_stop || !(k == e->key_stop)) {
            if ((rc = capture_graph(e, &e->gx_stop, &e->nk_stop, [&](cudaStream_t cs) {
                     int r = launch_count(e, k.sched_first, k.sched_last, e->d_sched, cs);
                     return r ? r : launch_checkpoint(e, cs);
                 })))
                return rc;
            e->key_stop = k;
        }
        if ((rc = launch_graph(e, e->gx_stop, e->nk_stop))) return rc;
    } else {
        if ((rc = reduce_stop(e))) return rc;
        const GraphKey k = graph_key(e, false);
        if (!e->gx_ckpt || !(k == e->key_ckpt)) {
            if ((rc = capture_graph(e, &e->gx_ckpt, &e->nk_ckpt, [&](cudaStream_t cs) { return launch_checkpoint(e, cs); })))
                return rc;
            e->key_ckpt = k;
        }
        if ((rc = launch_graph(e, e->gx_ckpt, e->nk_ckpt))) return rc;
    }
    const int slot = (int)(e->issued % kRing);
    e->kuse_at[slot] = e->kuse;
    DIC_CUDA(cudaEventRecord(e->ev[slot], e->s));
    *seq = e->issued++;
    return DIC_OK;
}

extern "C" int dic_engine_poll(dic_engine* e, int64_t seq, dic_stop_status* st, int32_t* replayed) {
    DIC_REQUIRE(e && st && replayed, "dic_engine_poll: null argument");
    if (seq != e->polled || seq >= e->issued) {
        set_error("dic_engine_poll: stop %lld polled out of order (next %lld, issued %lld)", (long long)seq,
                  (long long)e->polled, (long long)e->issued);
        return DIC_ESTATE;
    }
    const int KS = e->KS;
    const size_t u = sizeof(unsigned long long);
    const int slot = (int)(seq % kRing);
    if (!e->status_ready) DIC_CUDA(cudaEventSynchronize(e->ev[slot]));
    unsigned long long* h = e->ring + (int64_t)slot * e->ring_words;
    int ku = e->kuse_at[slot];
    *replayed = 0;
    int rc, replays = 0;
    while (h[S_OVERFLOW]) {
        // every later stop was skipped (abort flag): grow, replay this stop's
        // candidate step, and tell the caller to re-issue the skipped stops
        if (++replays > 4) {
            set_error("dic_engine_poll: candidate capacity did not converge");
            return DIC_ENOMEM;
        }
        DIC_CUDA(cudaStreamSynchronize(e->s));
        std::vector<unsigned long long> adm(KS), bn(KS);
        DIC_CUDA(cudaMemcpyAsync(adm.data(), e->d_stat + S_HEAD + KS, KS * u, cudaMemcpyDeviceToHost, e->s));
        DIC_CUDA(cudaMemcpyAsync(bn.data(), e->d_stat + S_HEAD + 2 * KS, KS * u, cudaMemcpyDeviceToHost, e->s));
        DIC_CUDA(cudaStreamSynchronize(e->s));
        const int64_t na = (int64_t)h[S_NADM];
        e->nrec = (int64_t)h[S_NREC];
        if ((rc = ensure_tmp(e, na))) return rc;
        if ((rc = grow_records(e, e->nrec + na))) return rc;
        // the aborted candidate step left its joins' temporary entries in the
        // index: rebuild it from the records (none of that stop was committed)
        {
            const int64_t hc0 = e->hcap;
            if ((rc = ensure_hash(e, e->nrec + na))) return rc;
            if (e->hcap == hc0 && (rc = rebuild_hash(e))) return rc;
        }
        bool changed = false;
        for (int k = 0; k < KS; ++k) {
            if (!adm[k]) continue;
            e->buckets[k].n = (int64_t)bn[k];
            if ((rc = grow_bucket(e, k, (int64_t)(bn[k] + adm[k]), &changed))) return rc;
        }
        if ((rc = ensure_slot_arrays(e))) return rc;
        if (changed && (rc = sync_bucket_tables(e))) return rc;
        // reset the join counters and the abort flag; NFRONT / frontier / apply results stay
        DIC_CUDA(cudaMemsetAsync(e->d_stat + S_NADM, 0, 3 * u, e->s));  // NADM, NINS, OVERFLOW
        DIC_CUDA(cudaMemsetAsync(e->d_stat + S_ABORT, 0, u, e->s));
        DIC_CUDA(cudaMemsetAsync(e->d_stat + S_HEAD + KS, 0, (size_t)KS * u, e->s));
        if ((rc = launch_checkpoint(e, e->s, true))) return rc;  // ends with the stop's status
        e->kuse_at[slot] = e->kuse;
        DIC_CUDA(cudaStreamSynchronize(e->s));
        ku = e->kuse_at[slot];
        // the skipped stops are re-issued by the caller
        e->issued = seq + 1;
        e->counted = false;
        e->merged_pending = false;
        *replayed = 1;
    }
    e->polled = seq + 1;
    // bookkeeping from the status words
    const int64_t pruned = (int64_t)h[S_NPRUNED], finalized = (int64_t)h[S_NFINAL];
    const int64_t inserted = (int64_t)h[S_NINS], survivors = (int64_t)h[S_SURV];
    st->dashed_at_start = e->live;
    st->promoted = (int64_t)h[S_NFRONT];
    st->pruned = pruned;
    st->finalized = finalized;
    st->inserted = inserted;
    st->dashed_peak = survivors + inserted;
    e->live = e->live - pruned - finalized + inserted;
    st->dashed_at_end = e->live;
    e->nrec = (int64_t)h[S_NREC];
    st->records = e->nrec;
    if ((int64_t)h[S_SEQ] != seq) {
        set_error("dic_engine_poll: status slot holds stop %lld, expected %lld", (long long)h[S_SEQ], (long long)seq);
        return DIC_ESTATE;
    }
    for (int k = 0; k < ku; ++k) e->buckets[k].n = (int64_t)h[S_HEAD + 3 * k + 2];
    // the pair bucket only shrinks after seeding: once the device's dense test
    // (2*bn[2] >= tri_len) fails it fails for every later stop
    if (e->tri && ku > 2 && 2 * (int64_t)h[S_HEAD + 3 * 2 + 2] < e->tri_len) e->tri_live = false;
    // headroom for the stops issued next (growth is stream-ordered)
    if ((rc = ensure_headroom(e))) return rc;
    return DIC_OK;
}

// Synchronous forms (one stop at a time): count, then checkpoint = issue + poll.
extern "C" int dic_engine_count(dic_engine* e, int64_t lfirst, int64_t llast) {
    return dic_engine_issue_count(e, lfirst, llast);
}

extern "C" int dic_engine_checkpoint(dic_engine* e, dic_stop_status* st) {
    DIC_REQUIRE(e && st, "dic_engine_checkpoint: null argument");
    int64_t seq = 0;
    int rc = dic_engine_issue_checkpoint(e, &seq);
    if (rc) return rc;
    int32_t replayed = 0;
    return dic_engine_poll(e, seq, st, &replayed);
}

// The whole pipelined checkpoint loop of one unsharded GPU, natively (the
// host side of _run, engine.py:422-441, with up to `depth` stops in flight).
extern "C" int dic_engine_run(dic_engine* e, const int64_t* lfirst, const int64_t* llast, const int64_t* rows,
                              int64_t stop_max, int32_t depth, dic_run_stats* out, float* count_ms,
                              int64_t* dashed, int64_t max_stops) {
    DIC_REQUIRE(e && lfirst && llast && rows && out, "dic_engine_run: null argument");
    DIC_REQUIRE(stop_max >= 1 && depth >= 1 && depth < kRing, "dic_engine_run: bad stop_max/depth");
    if (!e->seeded) { set_error("dic_engine_run: engine not seeded"); return DIC_ESTATE; }
    memset(out, 0, sizeof(*out));
    const int64_t captured0 = e->graphs_captured;
    {
        const int rc0 = dic_engine_set_schedule(e, lfirst, llast, stop_max);
        if (rc0) return rc0;
    }
    struct Flight { int64_t seq; int64_t stop; };
    std::deque<Flight> inflight;
    cudaEvent_t t0[kRing], t1[kRing];
    const bool timed = count_ms != nullptr;
    // one graph per scheduled stop unless the count half is timed on its own
    // (DIC_STOP_GRAPH=0: two graphs per stop)
    {
        const char* env = getenv("DIC_STOP_GRAPH");
        e->in_run = !timed && !(env && atoi(env) == 0);
    }
    if (timed)
        for (int i = 0; i < kRing; ++i) {
            DIC_CUDA(cudaEventCreate(&t0[i]));
            DIC_CUDA(cudaEventCreate(&t1[i]));
        }
    int rc = DIC_OK;
    int64_t stop = 0;
    bool done = e->live == 0;
    using clk = std::chrono::steady_clock;
    auto us_since = [](clk::time_point t) {
        return std::chrono::duration<double, std::micro>(clk::now() - t).count();
    };
    // one stop's status into the run's totals; returns false once the run is over
    auto account = [&](const Flight& f, const dic_stop_status& st, int32_t replayed) {
        out->replays += replayed;
        const int64_t i = out->stops;
        if (i < max_stops) {
            if (timed) cudaEventElapsedTime(&count_ms[i], t0[f.seq % kRing], t1[f.seq % kRing]);
            if (dashed) dashed[i] = st.dashed_at_start;
        }
        out->stops++;
        out->interval_counts += st.dashed_at_start;
        out->scanned += rows[f.stop - 1];
        out->candidates_generated += st.inserted;
        out->candidates_pruned += st.pruned;
        out->peak_dashed = std::max<int64_t>(out->peak_dashed, st.dashed_peak);
        if (st.dashed_at_end == 0) done = true;
    };
    // Batches of quiet stops (checkpoint_batch_kernel): with the pipeline
    // drained the host knows the dashed vector exactly; once it is small and
    // the pair bucket has left its dense phase, the next stops go out
    // kBatchStops at a time (DIC_BATCH_STOPS: 0 or 1 disables).
    int batch_n = kBatchStops;
    {
        const char* env = getenv("DIC_BATCH_STOPS");
        if (env && *env) batch_n = std::max(0, std::min(atoi(env), (int)kBatchStops));
    }
    const bool batch_ok = e->in_run && !e->comm && depth > 1 && batch_n > 1 && stop_max == e->nsched;
    // (as of the last polled stop; exact once nothing is in flight)
    auto batch_wanted = [&]() {
        if (!batch_ok || done || e->live <= 0 || e->live > kBatchSlots / 2) return false;
        if (e->tri && e->tri_live) return false;
        int64_t fill = 0;
        for (const Bucket& b : e->buckets) fill += b.n;
        return fill <= kBatchSlots;
    };
    while (rc == DIC_OK) {
        if (inflight.empty() && batch_wanted()) {
            // Batch mode, up to two batches in flight: the second is launched
            // before the first one's statuses are read, so the GPU does not wait
            // for the host between batches.  The device keeps its own stop
            // counter, so the second batch simply continues where the first one
            // ended (a batch may end early); each reports how many stops it ran.
            struct InBatch { int par; int kuse; };
            std::deque<InBatch> bq;
            bool more = true;
            volatile unsigned long long* report = e->hres.ring + kRing * e->hres.words + 2;
            while (rc == DIC_OK && (more || !bq.empty())) {
                const clk::time_point tb = clk::now();
                while (rc == DIC_OK && more && (int)bq.size() < 2) {
                    e->kuse_issue = e->kuse;
                    const GraphKey k = graph_key(e, true);
                    if (!e->gx_batch || e->gx_batch_n != batch_n || !(k == e->key_batch)) {
                        if ((rc = capture_graph(e, &e->gx_batch, &e->nk_batch,
                                                [&](cudaStream_t cs) { return launch_batch(e, batch_n, cs); })))
                            break;
                        e->key_batch = k;
                        e->gx_batch_n = batch_n;
                    }
                    const int par = (int)(e->batch_launches & 1);
                    report[par] = 0;
                    if ((rc = launch_graph(e, e->gx_batch, e->nk_batch))) break;
                    if (const cudaError_t ce = cudaEventRecord(e->ev[par], e->s)) {
                        rc = cuda_fail(ce, "cudaEventRecord(batch)");
                        break;
                    }
                    ++e->batch_launches;
                    bq.push_back({par, e->kuse});
                    ++out->batches;
                }
                out->issue_us += us_since(tb);
                if (rc || bq.empty()) break;
                const clk::time_point tp = clk::now();
                const InBatch ib = bq.front();
                bq.pop_front();
                if (const cudaError_t ce = cudaEventSynchronize(e->ev[ib.par])) {
                    rc = cuda_fail(ce, "cudaEventSynchronize(batch)");
                    break;
                }
                const unsigned long long rep = report[ib.par];
                const int nrun = (int)(rep & 0xFF);
                if (nrun > 0 && (rep >> 8) != (unsigned long long)e->issued + 1) {
                    set_error("dic_engine_run: a batch reports stop %lld, expected %lld", (long long)(rep >> 8) - 1,
                              (long long)e->issued);
                    rc = DIC_ESTATE;
                    break;
                }
                if (nrun == 0) more = false;  // refused or skipped: back to single stops
                for (int i = 0; i < nrun && rc == DIC_OK; ++i) {
                    const int64_t seq = e->issued;
                    const int slot = (int)(seq % kRing);
                    e->kuse_at[slot] = ib.kuse;
                    ++e->issued;
                    stop = stop < stop_max ? stop + 1 : 1;
                    dic_stop_status st;
                    int32_t replayed = 0;
                    e->status_ready = true;  // (its kernel has finished: no event to wait for)
                    rc = dic_engine_poll(e, seq, &st, &replayed);
                    e->status_ready = false;
                    if (rc) break;
                    if (done) {  // (a stop run past the last live one)
                        out->replays += replayed;
                        continue;
                    }
                    ++out->batched_stops;
                    account(Flight{seq, stop}, st, replayed);
                    if (replayed) more = false;  // (it overflowed: a later batch in flight was skipped)
                }
                if (done || !batch_wanted()) more = false;
                out->poll_us += us_since(tp);
            }
            if (rc) break;
            if (!done && batch_wanted()) {
                // (refused although wanted: cannot happen with an exact view of the
                // dashed vector; one single stop guarantees progress anyway)
                stop = stop < stop_max ? stop + 1 : 1;
                if ((rc = dic_engine_issue_count(e, lfirst[stop - 1], llast[stop - 1]))) break;
                int64_t seq = 0;
                if ((rc = dic_engine_issue_checkpoint(e, &seq))) break;
                inflight.push_back({seq, stop});
            } else {
                continue;
            }
        }
        const clk::time_point ti = clk::now();
        // (no new single stops once a batch is wanted: the pipeline drains first)
        while (!done && (int64_t)inflight.size() < depth && !batch_wanted()) {
            stop = stop < stop_max ? stop + 1 : 1;
            const int slot = (int)(e->issued % kRing);
            if (timed) cudaEventRecord(t0[slot], e->s);
            if ((rc = dic_engine_issue_count(e, lfirst[stop - 1], llast[stop - 1]))) break;
            if (timed) cudaEventRecord(t1[slot], e->s);
            int64_t seq = 0;
            if ((rc = dic_engine_issue_checkpoint(e, &seq))) break;
            inflight.push_back({seq, stop});
        }
        out->issue_us += us_since(ti);
        if (rc || inflight.empty()) break;
        const Flight f = inflight.front();
        inflight.pop_front();
        dic_stop_status st;
        int32_t replayed = 0;
        const clk::time_point tp = clk::now();
        if ((rc = dic_engine_poll(e, f.seq, &st, &replayed))) break;
        out->poll_us += us_since(tp);
        if (done) {  // a no-op stop issued after the last live one
            out->replays += replayed;
            continue;
        }
        account(f, st, replayed);
        if (replayed) {  // stops after f.seq were skipped on the device: re-issue them
            inflight.clear();
            stop = f.stop;
        }
    }
    out->graphs_captured = e->graphs_captured - captured0;
    e->in_run = false;
    if (timed)
        for (int i = 0; i < kRing; ++i) {
            cudaEventDestroy(t0[i]);
            cudaEventDestroy(t1[i]);
        }
    return rc;
}

// Collect the SOLID_BOX record ids into res_ids (kept for dic_engine_frequent).
extern "C" int dic_engine_num_frequent(dic_engine* e, int64_t* F) {
    DIC_REQUIRE(e && F, "dic_engine_num_frequent: null argument");
    unsigned long long* pin = e->hres.ring + kRing * e->hres.words;  // pinned scratch words past the ring
    DIC_CUDA(cudaMemcpyAsync(pin, e->d_stat + S_NREC, sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    e->nrec = (int64_t)pin[0];
    int rc;
    if (e->nrec > e->res_cap) {
        dfree(e->res_ids, e->s);
        if ((rc = dalloc(&e->res_ids, e->nrec, e->s))) return rc;
        e->res_cap = e->nrec;
    }
    unsigned long long* cnt = e->d_stat + S_SCRATCH;
    DIC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), e->s));
    collect_frequent_kernel<<<nblk(e->nrec), 256, 0, e->s>>>(e->R, e->nrec, e->res_ids, cnt);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("collect_frequent_kernel");
    DIC_CUDA(cudaMemcpyAsync(pin, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    e->res_F = (int64_t)pin[0];
    *F = e->res_F;
    return DIC_OK;
}

extern "C" int dic_engine_frequent(dic_engine* e, uint64_t* masks_host, int32_t* sizes_host, int64_t* supports_host,
                                   int64_t F) {
    DIC_REQUIRE(e && masks_host && sizes_host && supports_host, "dic_engine_frequent: null argument");
    int rc;
    if (e->res_F < 0) {
        int64_t F2 = 0;
        if ((rc = dic_engine_num_frequent(e, &F2))) return rc;
    }
    if (F != e->res_F) {
        set_error("dic_engine_frequent: F=%lld but %lld frequent records", (long long)F, (long long)e->res_F);
        return DIC_EINVAL;
    }
    e->res_F = -1;  // ids consumed
    const int W = e->W;
    if (F == 0) return DIC_OK;
    // one device buffer and one pinned staging buffer: masks | supports | sizes | flag
    const size_t mb = (size_t)F * W * 8, sb = ((size_t)F * 4 + 7) & ~(size_t)7, pb = (size_t)F * 8;
    const size_t total = mb + pb + sb + 8;
    uint8_t* dbuf = nullptr;
    if ((rc = dalloc(&dbuf, (int64_t)total, e->s))) return rc;
    auto* dm = reinterpret_cast<unsigned long long*>(dbuf);
    auto* dsu = reinterpret_cast<int64_t*>(dbuf + mb);
    auto* dsz = reinterpret_cast<int32_t*>(dbuf + mb + pb);
    auto* dflag = reinterpret_cast<unsigned long long*>(dbuf + mb + pb + sb);
    // up to kDevSortMax itemsets (of at most 8 items each) are put in the
    // result's canonical order on the device: rank by counting, F^2 / 32 warp
    // steps, a few microseconds for the thousands of itemsets a run finds
    constexpr int64_t kDevSortMax = 24576;
    bool dev_sorted = F <= kDevSortMax;
    DIC_CUDA(cudaMemsetAsync(dflag, 0, 8, e->s));
    if (dev_sorted) {
        ResKey* keys = nullptr;
        if ((rc = dalloc(&keys, F, e->s))) return rc;
        result_keys_kernel<<<nblk(F), 256, 0, e->s>>>(e->R, e->res_ids, F, keys, dflag);
        ::dic::note_launch();
        result_rank_gather_kernel<<<sm_count() * 4, 256, 0, e->s>>>(e->R, W, e->res_ids, F, keys, dm, dsz, dsu);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("result_rank_gather_kernel");
        dfree(keys, e->s);
    } else {
        gather_frequent_kernel<<<nblk(F), 256, 0, e->s>>>(e->R, W, e->res_ids, F, dm, dsz, dsu);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("gather_frequent_kernel");
    }
    HostRes& hr = e->hres;
    if (hr.stage_bytes < total) {
        if (hr.stage) cudaFreeHost(hr.stage);
        hr.stage = nullptr;
        hr.stage_bytes = 0;
        const size_t want = std::max(total, (size_t)1 << 20);
        DIC_CUDA(cudaHostAlloc((void**)&hr.stage, want, cudaHostAllocDefault));
        hr.stage_bytes = want;
    }
    DIC_CUDA(cudaMemcpyAsync(hr.stage, dbuf, total, cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    if (dev_sorted && *reinterpret_cast<const unsigned long long*>(hr.stage + mb + pb + sb) != 0) {
        // an itemset of more than 8 items: gather unordered, sort on the host
        dev_sorted = false;
        gather_frequent_kernel<<<nblk(F), 256, 0, e->s>>>(e->R, W, e->res_ids, F, dm, dsz, dsu);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("gather_frequent_kernel");
        DIC_CUDA(cudaMemcpyAsync(hr.stage, dbuf, total, cudaMemcpyDeviceToHost, e->s));
        DIC_CUDA(cudaStreamSynchronize(e->s));
    }
    dfree(dbuf, e->s);
    const uint64_t* m1 = reinterpret_cast<const uint64_t*>(hr.stage);
    const int64_t* p1 = reinterpret_cast<const int64_t*>(hr.stage + mb);
    const int32_t* s1 = reinterpret_cast<const int32_t*>(hr.stage + mb + pb);
    if (dev_sorted) {
        memcpy(masks_host, m1, mb);
        memcpy(sizes_host, s1, (size_t)F * 4);
        memcpy(supports_host, p1, pb);
        return DIC_OK;
    }
    // canonical order of the reference's result (engine.py:446-455): by size,
    // then by the mask as an integer.  For masks of equal size that order is
    // the lexicographic order of their item ids listed from the highest down,
    // so each key is (size, item ids descending, 4 x 16 bits per word) and a
    // comparison touches ceil(k/4) + 1 words.
    int kmax = 1;
    for (int64_t i = 0; i < F; ++i) kmax = std::max(kmax, (int)s1[i]);
    const int KW = 1 + (kmax + 3) / 4;
    std::vector<uint64_t> keys((size_t)F * KW, 0);
    for (int64_t i = 0; i < F; ++i) {
        uint64_t* k = keys.data() + (size_t)i * KW;
        k[0] = (uint64_t)(uint32_t)s1[i];
        int j = 0;
        for (int w = W - 1; w >= 0; --w) {
            uint64_t x = m1[(size_t)i * W + w];
            while (x) {
                const int b = 63 - __builtin_clzll(x);
                x &= ~(1ull << b);
                k[1 + j / 4] |= (uint64_t)(uint16_t)(w * 64 + b) << (48 - 16 * (j % 4));
                ++j;
            }
        }
    }
    std::vector<int64_t> idx(F);
    if (KW <= 3) {
        // itemsets of up to 8 items (every config): keys sorted in place as
        // 32-byte records (key words + index), not through an index array
        struct Rec {
            uint64_t k[3];
            int64_t i;
        };
        std::vector<Rec> recs((size_t)F);
        for (int64_t i = 0; i < F; ++i) {
            Rec& r = recs[(size_t)i];
            for (int q = 0; q < 3; ++q) r.k[q] = q < KW ? keys[(size_t)i * KW + q] : 0;
            r.i = i;
        }
        std::sort(recs.begin(), recs.end(), [](const Rec& a, const Rec& b) {
            if (a.k[0] != b.k[0]) return a.k[0] < b.k[0];
            if (a.k[1] != b.k[1]) return a.k[1] < b.k[1];
            return a.k[2] < b.k[2];
        });
        for (int64_t i = 0; i < F; ++i) idx[(size_t)i] = recs[(size_t)i].i;
    } else {
        std::iota(idx.begin(), idx.end(), 0);
        const uint64_t* kp = keys.data();
        std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
            const uint64_t* x = kp + (size_t)a * KW;
            const uint64_t* y = kp + (size_t)b * KW;
            for (int q = 0; q < KW; ++q)
                if (x[q] != y[q]) return x[q] < y[q];
            return false;
        });
    }
    for (int64_t i = 0; i < F; ++i) {
        const int64_t j = idx[i];
        memcpy(masks_host + (size_t)i * W, m1 + (size_t)j * W, W * sizeof(uint64_t));
        sizes_host[i] = s1[j];
        supports_host[i] = p1[j];
    }
    return DIC_OK;
}
