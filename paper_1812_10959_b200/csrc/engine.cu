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
// Phase fusion (exactness argued in DESIGN.md §Engine): check_full_pass runs
// in the same kernel as prune because finalisation never changes box-ness
// (DASHED_BOX->SOLID_BOX, DASHED_CIRCLE->SOLID_CIRCLE) and freshly inserted
// candidates have intervals_counted == 0 < stop_max, so make_candidates sees
// the same admissions and check_full_pass the same records either way.
// prune's superset-NIL loop (:311-315) is provably dead in the engine (a
// dashed circle's proper subsets are boxes, and boxes never revert), so the
// engine omits it; the API-level prune on host catalogs keeps it.
#include "common.cuh"

#include <cub/device/device_scan.cuh>

#include <vector>

namespace dic {

struct BucketIn {
    const uint16_t* items;
    unsigned long long* out;
    int64_t C;
    int k;
};
int count_buckets_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                         const BucketIn* bk, int nbk, cudaStream_t s);
int item_support_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                        unsigned long long* counts, cudaStream_t s);

enum : uint8_t { DASHED_CIRCLE = 0, DASHED_BOX = 1, SOLID_CIRCLE = 2, SOLID_BOX = 3, NIL = 4 };

__host__ __device__ inline bool is_box(uint8_t s) { return s == DASHED_BOX || s == SOLID_BOX; }
__host__ __device__ inline bool is_dashed(uint8_t s) { return s == DASHED_CIRCLE || s == DASHED_BOX; }

__host__ __device__ inline uint64_t zob(uint32_t item) {
    return mix64(0x5A0B1157ull + (uint64_t)item * 0x9E3779B97F4A7C15ull);
}

constexpr int32_t kEmpty = -1;
constexpr int32_t kTempFlag = 0x40000000;

// Device counters (one struct, read back with a single copy).
struct Counters {
    unsigned long long nfront;
    unsigned long long npruned;
    unsigned long long nfinal;
    unsigned long long survivors;  // non-NIL dashed after prune (incl. finalised)
    unsigned long long nadm;       // admissible joins found by eval (pre-dedup)
    unsigned long long ninserted;  // distinct new candidates committed
    unsigned long long nrec;       // records
    unsigned long long pad;
};

struct Records {
    unsigned long long* mask = nullptr;  // [cap][W]
    uint64_t* hash = nullptr;
    int64_t* support = nullptr;
    int64_t* intervals = nullptr;
    int32_t* size = nullptr;
    uint8_t* shape = nullptr;
    int64_t cap = 0;
};

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

__device__ __forceinline__ int32_t ht_lookup(const int32_t* __restrict__ ht, uint64_t hmask,
                                             const Records& R, int W, uint64_t h, const MaskView& v) {
    uint64_t slot = mix64(h) & hmask;
    while (true) {
        int32_t e = ht[slot];
        if (e == kEmpty) return -1;
        if (R.hash[e] == h && mask_eq(R.mask + (int64_t)e * W, v, W)) return e;
        slot = (slot + 1) & hmask;
    }
}

// ---------------------------------------------------------------------------
// seeding / rehash
// ---------------------------------------------------------------------------
__global__ void ht_clear_kernel(int32_t* ht, int64_t cap) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
         i += (int64_t)gridDim.x * blockDim.x)
        ht[i] = kEmpty;
}

// Insert records [r0, r1) (known to be distinct) into the hash index.
__global__ void ht_insert_records_kernel(int32_t* ht, uint64_t hmask, Records R, int64_t r0, int64_t r1) {
    int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    uint64_t slot = mix64(R.hash[r]) & hmask;
    while (atomicCAS(ht + slot, kEmpty, (int32_t)r) != kEmpty) slot = (slot + 1) & hmask;
}

// Singletons: record i = item i (first_pass, engine.py:125-163).
__global__ void seed_singletons_kernel(Records R, int W, int m, const int64_t* __restrict__ counts,
                                       int64_t need, int64_t stop_max) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    for (int w = 0; w < W; ++w) R.mask[(int64_t)i * W + w] = (w == (i >> 6)) ? (1ull << (i & 63)) : 0ull;
    R.hash[i] = zob((uint32_t)i);
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
    // row_start[a] = index of the first pair with first element a
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
    R.size[r] = 2;
    R.support[r] = 0;
    R.intervals[r] = 0;
    R.shape[r] = DASHED_CIRCLE;
    b_rec[p] = (int32_t)r;
    b_items[2 * p] = (uint16_t)ia;
    b_items[2 * p + 1] = (uint16_t)ib;
}

// ---------------------------------------------------------------------------
// per stop
// ---------------------------------------------------------------------------
// support += delta, intervals += 1 (count_support_interval), then prune
// (engine.py:292-310) and check_full_pass (:380-388).  keep[c] = still dashed.
__global__ void apply_prune_finalize_kernel(const int32_t* __restrict__ b_rec, int64_t nb,
                                            const unsigned long long* __restrict__ delta, Records R,
                                            int64_t need, int64_t interval, int64_t stop_max, int bound,
                                            int32_t* __restrict__ frontier, int32_t* __restrict__ keep,
                                            Counters* ctr, unsigned long long* removed_k) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool promoted = false, pruned = false, fin = false, surv = false, kept = false;
    if (c < nb) {
        int32_t r = b_rec[c];
        int64_t s = R.support[r] + (int64_t)delta[c];
        int64_t iv = R.intervals[r] + 1;
        R.support[r] = s;
        R.intervals[r] = iv;
        uint8_t sh = R.shape[r];
        if (sh == DASHED_CIRCLE) {
            if (s >= need) {
                sh = DASHED_BOX;
                promoted = true;
            } else if (bound && iv < stop_max) {
                int64_t remaining = stop_max - iv;
                if (s + interval * remaining < need) {
                    sh = NIL;
                    pruned = true;
                }
            }
        }
        if (is_dashed(sh)) {
            surv = true;
            if (iv == stop_max) {
                sh = s >= need ? SOLID_BOX : SOLID_CIRCLE;
                fin = true;
            }
        }
        R.shape[r] = sh;
        kept = is_dashed(sh);
        keep[c] = kept ? 1 : 0;
        if (promoted) {
            // order among promoted records is irrelevant to results and stats
            unsigned long long pos = atomicAdd(&ctr->nfront, 1ull);
            frontier[pos] = r;
        }
    }
    // warp-aggregated counters
    unsigned pr = __ballot_sync(0xFFFFFFFFu, pruned), fi = __ballot_sync(0xFFFFFFFFu, fin);
    unsigned su = __ballot_sync(0xFFFFFFFFu, surv), rm = __ballot_sync(0xFFFFFFFFu, c < nb && !kept);
    if ((threadIdx.x & 31) == 0) {
        if (pr) atomicAdd(&ctr->npruned, (unsigned long long)__popc(pr));
        if (fi) atomicAdd(&ctr->nfinal, (unsigned long long)__popc(fi));
        if (su) atomicAdd(&ctr->survivors, (unsigned long long)__popc(su));
        if (rm) atomicAdd(removed_k, (unsigned long long)__popc(rm));
    }
}

// make_candidates (engine.py:320-369), evaluation: thread per (frontier f,
// level1 item j).  Admission needs cand not in known and every immediate
// subset known with a box shape; the subset equal to src is a box by
// construction (it was just promoted) and is skipped.
__global__ void eval_candidates_kernel(const int32_t* __restrict__ frontier, int64_t nf,
                                       const int32_t* __restrict__ level1, int64_t L, int W, Records R,
                                       const int32_t* __restrict__ ht, uint64_t hmask,
                                       unsigned long long* __restrict__ tmp_mask, uint64_t* __restrict__ tmp_hash,
                                       int32_t* __restrict__ tmp_size, int64_t tmp_cap, Counters* ctr,
                                       unsigned long long* adm_by_size) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nf * L) return;
    int64_t f = t / L, j = t - f * L;
    int32_t src = frontier[f];
    int l = level1[j];
    const unsigned long long* sm = R.mask + (int64_t)src * W;
    if ((sm[l >> 6] >> (l & 63)) & 1ull) return;  // cand == base
    uint64_t hc = R.hash[src] ^ zob((uint32_t)l);
    MaskView cand{sm, l, -1};
    if (ht_lookup(ht, hmask, R, W, hc, cand) >= 0) return;  // already known
    for (int w = 0; w < W; ++w) {
        unsigned long long x = cand.word(w);
        while (x) {
            int b = __ffsll((long long)x) - 1;
            x &= x - 1;
            int bit = w * 64 + b;
            if (bit == l) continue;
            MaskView sub{sm, l, bit};
            int32_t e = ht_lookup(ht, hmask, R, W, hc ^ zob((uint32_t)bit), sub);
            if (e < 0 || !is_box(R.shape[e])) return;
        }
    }
    unsigned long long pos = atomicAdd(&ctr->nadm, 1ull);
    int sz = R.size[src] + 1;
    atomicAdd(adm_by_size + sz, 1ull);
    if ((int64_t)pos < tmp_cap) {
        for (int w = 0; w < W; ++w) tmp_mask[(int64_t)pos * W + w] = cand.word(w);
        tmp_hash[pos] = hc;
        tmp_size[pos] = sz;
    }
}

// Dedup the admissible joins: claim a hash slot per distinct mask.  Slots
// hold either a record id or kTempFlag | tmp index (resolved by commit).
__global__ void insert_candidates_kernel(int64_t na, int W, const unsigned long long* __restrict__ tmp_mask,
                                         const uint64_t* __restrict__ tmp_hash, Records R, int32_t* ht,
                                         uint64_t hmask, int64_t* __restrict__ tmp_slot) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= na) return;
    uint64_t h = tmp_hash[t];
    const unsigned long long* mk = tmp_mask + t * W;
    uint64_t slot = mix64(h) & hmask;
    tmp_slot[t] = -1;
    while (true) {
        int32_t prev = atomicCAS(ht + slot, kEmpty, kTempFlag | (int32_t)t);
        if (prev == kEmpty) {
            tmp_slot[t] = (int64_t)slot;
            return;
        }
        bool same;
        if (prev & kTempFlag) {
            int64_t o = prev & ~kTempFlag;
            same = tmp_hash[o] == h;
            for (int w = 0; same && w < W; ++w) same = tmp_mask[o * W + w] == mk[w];
        } else {
            same = R.hash[prev] == h;
            for (int w = 0; same && w < W; ++w) same = R.mask[(int64_t)prev * W + w] == mk[w];
        }
        if (same) return;  // duplicate of a join admitted by another thread
        slot = (slot + 1) & hmask;
    }
}

__global__ void commit_candidates_kernel(int64_t na, int W, const unsigned long long* __restrict__ tmp_mask,
                                         const uint64_t* __restrict__ tmp_hash, const int32_t* __restrict__ tmp_size,
                                         const int64_t* __restrict__ tmp_slot, Records R, int32_t* ht,
                                         Counters* ctr, int32_t* const* __restrict__ b_rec_tab,
                                         uint16_t* const* __restrict__ b_items_tab,
                                         unsigned long long* __restrict__ b_n) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= na) return;
    int64_t slot = tmp_slot[t];
    if (slot < 0) return;
    int64_t r = (int64_t)atomicAdd(&ctr->nrec, 1ull);
    atomicAdd(&ctr->ninserted, 1ull);
    int sz = tmp_size[t];
    for (int w = 0; w < W; ++w) R.mask[r * W + w] = tmp_mask[t * W + w];
    R.hash[r] = tmp_hash[t];
    R.size[r] = sz;
    R.support[r] = 0;
    R.intervals[r] = 0;
    R.shape[r] = DASHED_CIRCLE;
    ht[slot] = (int32_t)r;
    unsigned long long pos = atomicAdd(b_n + sz, 1ull);
    b_rec_tab[sz][pos] = (int32_t)r;
    uint16_t* it = b_items_tab[sz] + (int64_t)pos * sz;
    int j = 0;
    for (int w = 0; w < W; ++w) {
        unsigned long long x = tmp_mask[t * W + w];
        while (x) {
            int b = __ffsll((long long)x) - 1;
            x &= x - 1;
            it[j++] = (uint16_t)(w * 64 + b);
        }
    }
}

// Order-preserving compaction of one bucket (compact_dashed).
__global__ void compact_bucket_kernel(int64_t nb, int k, const int32_t* __restrict__ keep,
                                      const int32_t* __restrict__ pos, const int32_t* __restrict__ rec_in,
                                      const uint16_t* __restrict__ items_in, int32_t* __restrict__ rec_out,
                                      uint16_t* __restrict__ items_out) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nb || !keep[c]) return;
    int64_t d = pos[c];
    rec_out[d] = rec_in[c];
    for (int j = 0; j < k; ++j) items_out[d * k + j] = items_in[c * k + j];
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

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace dic

using namespace dic;

struct Bucket {
    int32_t* rec = nullptr;
    uint16_t* items = nullptr;
    int64_t n = 0, cap = 0;
};

struct dic_engine {
    const uint32_t* tids;
    int64_t n_local;
    int m, W;
    int64_t need, interval, stop_max;
    int bound;
    cudaStream_t s;

    Records R;
    int64_t nrec = 0;
    int32_t* ht = nullptr;
    int64_t hcap = 0;

    std::vector<Bucket> buckets;  // index = itemset size
    int32_t** d_brec = nullptr;   // device copies of bucket pointer tables
    uint16_t** d_bitems = nullptr;
    unsigned long long* d_bn = nullptr;       // [m+2] bucket sizes (device mirror)
    unsigned long long* d_removed = nullptr;  // [m+2]
    unsigned long long* d_adm = nullptr;      // [m+2] admitted joins by size

    int32_t* level1 = nullptr;
    int64_t nL1 = 0;
    int32_t* frontier = nullptr;
    int64_t front_cap = 0;
    int32_t* keep = nullptr;
    int32_t* pos = nullptr;
    int64_t keep_cap = 0;
    void* scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0;

    unsigned long long* delta = nullptr;
    int64_t delta_cap = 0, delta_len = 0;
    std::vector<int64_t> delta_off;

    unsigned long long* tmp_mask = nullptr;
    uint64_t* tmp_hash = nullptr;
    int32_t* tmp_size = nullptr;
    int64_t* tmp_slot = nullptr;
    int64_t tmp_cap = 0;

    Counters* ctr = nullptr;   // device
    Counters* hctr = nullptr;  // pinned host
    bool seeded = false;
    bool counted = false;
};

namespace {

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

template <class T>
int dgrow(T** p, int64_t old_count, int64_t new_count, cudaStream_t s) {
    T* q = nullptr;
    int rc = dalloc(&q, new_count, s);
    if (rc) return rc;
    if (*p && old_count > 0) {
        cudaError_t e = cudaMemcpyAsync(q, *p, (size_t)old_count * sizeof(T), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(grow)");
    }
    dfree(*p, s);
    *p = q;
    return DIC_OK;
}

int grow_records(dic_engine* e, int64_t need_cap) {
    if (need_cap <= e->R.cap) return DIC_OK;
    int64_t nc = std::max<int64_t>(need_cap, e->R.cap * 2);
    nc = std::max<int64_t>(nc, 1024);
    Records& R = e->R;
    int rc;
    if ((rc = dgrow(&R.mask, e->nrec * e->W, nc * e->W, e->s))) return rc;
    if ((rc = dgrow(&R.hash, e->nrec, nc, e->s))) return rc;
    if ((rc = dgrow(&R.support, e->nrec, nc, e->s))) return rc;
    if ((rc = dgrow(&R.intervals, e->nrec, nc, e->s))) return rc;
    if ((rc = dgrow(&R.size, e->nrec, nc, e->s))) return rc;
    if ((rc = dgrow(&R.shape, e->nrec, nc, e->s))) return rc;
    R.cap = nc;
    return DIC_OK;
}

// keep the hash load factor <= 1/2; rebuild from the records on growth
int ensure_hash(dic_engine* e, int64_t nrec_after) {
    if (nrec_after * 2 <= e->hcap) return DIC_OK;
    int64_t nc = 1024;
    while (nc < nrec_after * 2) nc <<= 1;
    nc = std::max<int64_t>(nc, e->hcap * 2);
    dfree(e->ht, e->s);
    int rc = dalloc(&e->ht, nc, e->s);
    if (rc) return rc;
    e->hcap = nc;
    ht_clear_kernel<<<nblk(nc), 256, 0, e->s>>>(e->ht, nc); ::dic::note_launch();
    if (e->nrec > 0) {
        ht_insert_records_kernel<<<nblk(e->nrec), 256, 0, e->s>>>(e->ht, (uint64_t)nc - 1, e->R, 0, e->nrec); ::dic::note_launch();
    }
    DIC_CHECK_LAUNCH("rehash");
    return DIC_OK;
}

int sync_bucket_tables(dic_engine* e) {
    std::vector<int32_t*> r(e->m + 2, nullptr);
    std::vector<uint16_t*> it(e->m + 2, nullptr);
    for (size_t k = 0; k < e->buckets.size() && k < (size_t)e->m + 2; ++k) {
        r[k] = e->buckets[k].rec;
        it[k] = e->buckets[k].items;
    }
    DIC_CUDA(cudaMemcpyAsync(e->d_brec, r.data(), r.size() * sizeof(int32_t*), cudaMemcpyHostToDevice, e->s));
    DIC_CUDA(cudaMemcpyAsync(e->d_bitems, it.data(), it.size() * sizeof(uint16_t*), cudaMemcpyHostToDevice, e->s));
    // the host vectors die at return: make the copies complete first
    DIC_CUDA(cudaStreamSynchronize(e->s));
    return DIC_OK;
}

int grow_bucket(dic_engine* e, int k, int64_t need_cap, bool* changed) {
    Bucket& b = e->buckets[k];
    if (need_cap <= b.cap) return DIC_OK;
    int64_t nc = std::max<int64_t>(need_cap, b.cap * 2);
    nc = std::max<int64_t>(nc, 256);
    int rc;
    if ((rc = dgrow(&b.rec, b.n, nc, e->s))) return rc;
    if ((rc = dgrow(&b.items, b.n * k, nc * k, e->s))) return rc;
    b.cap = nc;
    *changed = true;
    return DIC_OK;
}

int ensure_scratch(dic_engine* e, int64_t nb) {
    if (nb <= e->keep_cap) return DIC_OK;
    int64_t nc = std::max<int64_t>(nb, e->keep_cap * 2);
    dfree(e->keep, e->s);
    dfree(e->pos, e->s);
    int rc;
    if ((rc = dalloc(&e->keep, nc, e->s))) return rc;
    if ((rc = dalloc(&e->pos, nc, e->s))) return rc;
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int)nc, e->s);
    if (bytes > e->scan_tmp_bytes) {
        if (e->scan_tmp) cudaFreeAsync(e->scan_tmp, e->s);
        DIC_CUDA(cudaMallocAsync(&e->scan_tmp, bytes, e->s));
        e->scan_tmp_bytes = bytes;
    }
    e->keep_cap = nc;
    return DIC_OK;
}

int read_counters(dic_engine* e) {
    DIC_CUDA(cudaMemcpyAsync(e->hctr, e->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    return DIC_OK;
}

int64_t total_dashed(const dic_engine* e) {
    int64_t t = 0;
    for (const Bucket& b : e->buckets) t += b.n;
    return t;
}

}  // namespace

extern "C" int dic_engine_create(const uint32_t* tids, int64_t n_local, int32_t m, int64_t need,
                                 int64_t interval, int64_t stop_max, int32_t prune_bound, void* stream,
                                 dic_engine** out) {
    DIC_REQUIRE(out, "dic_engine_create: out is null");
    DIC_REQUIRE(m >= 1 && m <= 65535, "dic_engine_create: m=%d outside [1, 65535]", m);
    DIC_REQUIRE(n_local >= 0 && (tids || n_local == 0), "dic_engine_create: bad tids/n_local");
    DIC_REQUIRE(interval >= 1 && stop_max >= 1, "dic_engine_create: bad interval/stop_max");
    dic_engine* e = new dic_engine();
    e->tids = tids;
    e->n_local = n_local;
    e->m = m;
    e->W = (m + 63) / 64;
    e->need = need;
    e->interval = interval;
    e->stop_max = stop_max;
    e->bound = prune_bound ? 1 : 0;
    e->s = as_stream(stream);
    e->buckets.resize(m + 2);
    int rc = 0;
    if ((rc = dalloc(&e->d_brec, m + 2, e->s)) || (rc = dalloc(&e->d_bitems, m + 2, e->s)) ||
        (rc = dalloc(&e->d_bn, m + 2, e->s)) || (rc = dalloc(&e->d_removed, m + 2, e->s)) ||
        (rc = dalloc(&e->d_adm, m + 2, e->s)) || (rc = dalloc(&e->ctr, 1, e->s)) ||
        (rc = dalloc(&e->level1, m, e->s))) {
        delete e;
        return rc;
    }
    cudaError_t ce = cudaMallocHost((void**)&e->hctr, sizeof(Counters));
    if (ce != cudaSuccess) {
        delete e;
        return cuda_fail(ce, "cudaMallocHost");
    }
    cudaMemsetAsync(e->d_bn, 0, (m + 2) * sizeof(unsigned long long), e->s);
    rc = sync_bucket_tables(e);
    if (rc) {
        delete e;
        return rc;
    }
    *out = e;
    return DIC_OK;
}

extern "C" int dic_engine_destroy(dic_engine* e) {
    if (!e) return DIC_OK;
    cudaStream_t s = e->s;
    Records& R = e->R;
    dfree(R.mask, s); dfree(R.hash, s); dfree(R.support, s); dfree(R.intervals, s);
    dfree(R.size, s); dfree(R.shape, s);
    dfree(e->ht, s);
    for (Bucket& b : e->buckets) { dfree(b.rec, s); dfree(b.items, s); }
    dfree(e->d_brec, s); dfree(e->d_bitems, s); dfree(e->d_bn, s); dfree(e->d_removed, s);
    dfree(e->d_adm, s); dfree(e->level1, s); dfree(e->frontier, s); dfree(e->keep, s);
    dfree(e->pos, s); dfree(e->delta, s); dfree(e->tmp_mask, s); dfree(e->tmp_hash, s);
    dfree(e->tmp_size, s); dfree(e->tmp_slot, s); dfree(e->ctr, s);
    if (e->scan_tmp) cudaFreeAsync(e->scan_tmp, s);
    cudaStreamSynchronize(s);
    if (e->hctr) cudaFreeHost(e->hctr);
    delete e;
    return DIC_OK;
}

extern "C" int dic_engine_words(dic_engine* e) { return e ? e->W : DIC_EINVAL; }

extern "C" int dic_engine_item_counts(dic_engine* e, int64_t* counts) {
    DIC_REQUIRE(e && counts, "dic_engine_item_counts: null argument");
    DIC_CUDA(cudaMemsetAsync(counts, 0, (size_t)e->m * sizeof(int64_t), e->s));
    if (e->n_local > 0)
        return item_support_launch(e->tids, e->n_local, e->m, 0, e->n_local - 1,
                                   reinterpret_cast<unsigned long long*>(counts), e->s);
    return DIC_OK;
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
    if ((rc = grow_records(e, m + npairs + 1024))) return rc;
    e->nrec = 0;
    if ((rc = ensure_hash(e, m + npairs))) return rc;
    seed_singletons_kernel<<<nblk(m), 256, 0, e->s>>>(e->R, e->W, m, counts, e->need, e->stop_max); ::dic::note_launch();
    DIC_CHECK_LAUNCH("seed_singletons_kernel");
    if (L > 0) DIC_CUDA(cudaMemcpyAsync(e->level1, l1.data(), L * sizeof(int32_t), cudaMemcpyHostToDevice, e->s));
    e->nL1 = L;
    if (npairs > 0) {
        bool changed = false;
        if ((rc = grow_bucket(e, 2, npairs, &changed))) return rc;
        std::vector<int64_t> rs(L);
        int64_t acc = 0;
        for (int64_t a = 0; a < L; ++a) { rs[a] = acc; acc += L - 1 - a; }
        int64_t* d_rs = nullptr;
        if ((rc = dalloc(&d_rs, L, e->s))) return rc;
        DIC_CUDA(cudaMemcpyAsync(d_rs, rs.data(), L * sizeof(int64_t), cudaMemcpyHostToDevice, e->s));
        seed_pairs_kernel<<<nblk(npairs), 256, 0, e->s>>>(e->R, e->W, e->level1, L, d_rs, npairs, m,
                                                          e->buckets[2].rec, e->buckets[2].items); ::dic::note_launch();
        DIC_CHECK_LAUNCH("seed_pairs_kernel");
        dfree(d_rs, e->s);
        e->buckets[2].n = npairs;
        if (changed && (rc = sync_bucket_tables(e))) return rc;
    }
    e->nrec = m + npairs;
    ht_insert_records_kernel<<<nblk(e->nrec), 256, 0, e->s>>>(e->ht, (uint64_t)e->hcap - 1, e->R, 0, e->nrec); ::dic::note_launch();
    DIC_CHECK_LAUNCH("ht_insert_records_kernel");
    // device mirror of bucket sizes
    std::vector<unsigned long long> bn(m + 2, 0);
    bn[2] = (unsigned long long)npairs;
    DIC_CUDA(cudaMemcpyAsync(e->d_bn, bn.data(), bn.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, e->s));
    DIC_CUDA(cudaStreamSynchronize(e->s));
    e->seeded = true;
    if (n_level1) *n_level1 = L;
    if (n_pairs) *n_pairs = npairs;
    return DIC_OK;
}

extern "C" int dic_engine_count(dic_engine* e, int64_t lfirst, int64_t llast) {
    DIC_REQUIRE(e, "dic_engine_count: null engine");
    if (!e->seeded) { set_error("dic_engine_count: engine not seeded"); return DIC_ESTATE; }
    DIC_REQUIRE(lfirst >= 0 && (llast < lfirst || llast < e->n_local),
                "dic_engine_count: local chunk [%lld, %lld] outside %lld local rows", (long long)lfirst,
                (long long)llast, (long long)e->n_local);
    const int64_t tot = total_dashed(e);
    if (tot > e->delta_cap) {
        dfree(e->delta, e->s);
        int64_t nc = std::max<int64_t>(tot, e->delta_cap * 2);
        int rc = dalloc(&e->delta, nc, e->s);
        if (rc) return rc;
        e->delta_cap = nc;
    }
    e->delta_len = tot;
    e->delta_off.assign(e->buckets.size(), 0);
    if (tot > 0) DIC_CUDA(cudaMemsetAsync(e->delta, 0, tot * sizeof(unsigned long long), e->s));
    int64_t off = 0;
    std::vector<BucketIn> bk;
    for (size_t k = 0; k < e->buckets.size(); ++k) {
        const Bucket& b = e->buckets[k];
        e->delta_off[k] = off;
        if (b.n > 0) bk.push_back(BucketIn{b.items, e->delta + off, b.n, (int)k});
        off += b.n;
    }
    if (!bk.empty() && llast >= lfirst) {
        int rc = count_buckets_launch(e->tids, e->n_local, e->m, lfirst, llast, bk.data(), (int)bk.size(), e->s);
        if (rc) return rc;
    }
    e->counted = true;
    return DIC_OK;
}

extern "C" int dic_engine_delta(dic_engine* e, void** ptr, int64_t* len) {
    DIC_REQUIRE(e && ptr && len, "dic_engine_delta: null argument");
    *ptr = e->delta;
    *len = e->delta_len;
    return DIC_OK;
}

extern "C" int dic_engine_checkpoint(dic_engine* e, dic_stop_status* st) {
    DIC_REQUIRE(e && st, "dic_engine_checkpoint: null argument");
    if (!e->counted) { set_error("dic_engine_checkpoint: no count since the last checkpoint"); return DIC_ESTATE; }
    e->counted = false;
    int rc;
    const int64_t tot = e->delta_len;
    st->dashed_at_start = tot;
    // 1. apply + prune + finalize, per bucket
    if ((rc = ensure_scratch(e, std::max<int64_t>(tot, 1)))) return rc;
    if (tot > e->front_cap) {
        dfree(e->frontier, e->s);
        int64_t nc = std::max<int64_t>(tot, e->front_cap * 2);
        if ((rc = dalloc(&e->frontier, nc, e->s))) return rc;
        e->front_cap = nc;
    }
    DIC_CUDA(cudaMemsetAsync(e->ctr, 0, sizeof(Counters), e->s));
    DIC_CUDA(cudaMemsetAsync(e->d_removed, 0, (e->m + 2) * sizeof(unsigned long long), e->s));
    for (size_t k = 0; k < e->buckets.size(); ++k) {
        const Bucket& b = e->buckets[k];
        if (b.n == 0) continue;
        int64_t off = e->delta_off[k];
        apply_prune_finalize_kernel<<<nblk(b.n), 256, 0, e->s>>>(
            b.rec, b.n, e->delta + off, e->R, e->need, e->interval, e->stop_max, e->bound, e->frontier,
            e->keep + off, e->ctr, e->d_removed + k); ::dic::note_launch();
    }
    DIC_CHECK_LAUNCH("apply_prune_finalize_kernel");
    std::vector<unsigned long long> removed(e->buckets.size(), 0);
    DIC_CUDA(cudaMemcpyAsync(removed.data(), e->d_removed, removed.size() * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, e->s));
    if ((rc = read_counters(e))) return rc;
    const int64_t nfront = (int64_t)e->hctr->nfront;
    st->promoted = nfront;
    st->pruned = (int64_t)e->hctr->npruned;
    st->finalized = (int64_t)e->hctr->nfinal;
    const int64_t survivors = (int64_t)e->hctr->survivors;

    // 2. compaction (before appending, so new candidates keep their slots)
    bool tables_changed = false;
    for (size_t k = 0; k < e->buckets.size(); ++k) {
        Bucket& b = e->buckets[k];
        if (b.n == 0 || removed[k] == 0) continue;
        int64_t off = e->delta_off[k];
        size_t bytes = e->scan_tmp_bytes;
        cub::DeviceScan::ExclusiveSum(e->scan_tmp, bytes, e->keep + off, e->pos + off, (int)b.n, e->s);
        int32_t* nrec_arr = nullptr;
        uint16_t* nitems = nullptr;
        if ((rc = dalloc(&nrec_arr, b.cap, e->s)) || (rc = dalloc(&nitems, b.cap * (int64_t)k, e->s))) return rc;
        compact_bucket_kernel<<<nblk(b.n), 256, 0, e->s>>>(b.n, (int)k, e->keep + off, e->pos + off, b.rec,
                                                            b.items, nrec_arr, nitems); ::dic::note_launch();
        DIC_CHECK_LAUNCH("compact_bucket_kernel");
        dfree(b.rec, e->s);
        dfree(b.items, e->s);
        b.rec = nrec_arr;
        b.items = nitems;
        b.n -= (int64_t)removed[k];
        tables_changed = true;
    }

    // 3. make_candidates from the frontier
    int64_t inserted = 0;
    if (nfront > 0 && e->nL1 > 0) {
        const int64_t pairs = nfront * e->nL1;
        int64_t want_tmp = std::min<int64_t>(pairs, std::max<int64_t>(1 << 16, e->tmp_cap));
        for (int attempt = 0; attempt < 2; ++attempt) {
            if (want_tmp > e->tmp_cap) {
                dfree(e->tmp_mask, e->s); dfree(e->tmp_hash, e->s); dfree(e->tmp_size, e->s); dfree(e->tmp_slot, e->s);
                if ((rc = dalloc(&e->tmp_mask, want_tmp * e->W, e->s)) || (rc = dalloc(&e->tmp_hash, want_tmp, e->s)) ||
                    (rc = dalloc(&e->tmp_size, want_tmp, e->s)) || (rc = dalloc(&e->tmp_slot, want_tmp, e->s)))
                    return rc;
                e->tmp_cap = want_tmp;
            }
            DIC_CUDA(cudaMemsetAsync(&e->ctr->nadm, 0, sizeof(unsigned long long), e->s));
            DIC_CUDA(cudaMemsetAsync(e->d_adm, 0, (e->m + 2) * sizeof(unsigned long long), e->s));
            eval_candidates_kernel<<<nblk(pairs), 256, 0, e->s>>>(
                e->frontier, nfront, e->level1, e->nL1, e->W, e->R, e->ht, (uint64_t)e->hcap - 1, e->tmp_mask,
                e->tmp_hash, e->tmp_size, e->tmp_cap, e->ctr, e->d_adm); ::dic::note_launch();
            DIC_CHECK_LAUNCH("eval_candidates_kernel");
            if ((rc = read_counters(e))) return rc;
            if ((int64_t)e->hctr->nadm <= e->tmp_cap) break;
            want_tmp = (int64_t)e->hctr->nadm;  // rerun once with room for every join
        }
        const int64_t na = (int64_t)e->hctr->nadm;
        if (na > 0) {
            std::vector<unsigned long long> adm(e->m + 2);
            DIC_CUDA(cudaMemcpyAsync(adm.data(), e->d_adm, adm.size() * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, e->s));
            DIC_CUDA(cudaStreamSynchronize(e->s));
            if ((rc = grow_records(e, e->nrec + na))) return rc;
            if ((rc = ensure_hash(e, e->nrec + na))) return rc;
            for (int k = 0; k < e->m + 2; ++k) {
                if (!adm[k]) continue;
                if ((rc = grow_bucket(e, k, e->buckets[k].n + (int64_t)adm[k], &tables_changed))) return rc;
            }
            if (tables_changed) {
                if ((rc = sync_bucket_tables(e))) return rc;
                tables_changed = false;
            }
            std::vector<unsigned long long> bn(e->m + 2);
            for (int k = 0; k < e->m + 2; ++k) bn[k] = (unsigned long long)e->buckets[k].n;
            DIC_CUDA(cudaMemcpyAsync(e->d_bn, bn.data(), bn.size() * sizeof(unsigned long long),
                                     cudaMemcpyHostToDevice, e->s));
            unsigned long long nrec_now = (unsigned long long)e->nrec;
            DIC_CUDA(cudaMemcpyAsync(&e->ctr->nrec, &nrec_now, sizeof(nrec_now), cudaMemcpyHostToDevice, e->s));
            insert_candidates_kernel<<<nblk(na), 256, 0, e->s>>>(na, e->W, e->tmp_mask, e->tmp_hash, e->R, e->ht,
                                                                 (uint64_t)e->hcap - 1, e->tmp_slot); ::dic::note_launch();
            DIC_CHECK_LAUNCH("insert_candidates_kernel");
            commit_candidates_kernel<<<nblk(na), 256, 0, e->s>>>(na, e->W, e->tmp_mask, e->tmp_hash, e->tmp_size,
                                                                 e->tmp_slot, e->R, e->ht, e->ctr, e->d_brec,
                                                                 e->d_bitems, e->d_bn); ::dic::note_launch();
            DIC_CHECK_LAUNCH("commit_candidates_kernel");
            DIC_CUDA(cudaMemcpyAsync(bn.data(), e->d_bn, bn.size() * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, e->s));
            if ((rc = read_counters(e))) return rc;
            inserted = (int64_t)e->hctr->ninserted;
            e->nrec = (int64_t)e->hctr->nrec;
            for (int k = 0; k < e->m + 2; ++k) e->buckets[k].n = (int64_t)bn[k];
        }
    }
    if (tables_changed && (rc = sync_bucket_tables(e))) return rc;
    st->inserted = inserted;
    st->dashed_peak = survivors + inserted;
    st->dashed_at_end = total_dashed(e);
    st->records = e->nrec;
    return DIC_OK;
}

extern "C" int dic_engine_num_frequent(dic_engine* e, int64_t* F) {
    DIC_REQUIRE(e && F, "dic_engine_num_frequent: null argument");
    int32_t* ids = nullptr;
    int rc = dalloc(&ids, std::max<int64_t>(e->nrec, 1), e->s);
    if (rc) return rc;
    DIC_CUDA(cudaMemsetAsync(&e->ctr->pad, 0, sizeof(unsigned long long), e->s));
    collect_frequent_kernel<<<nblk(e->nrec), 256, 0, e->s>>>(e->R, e->nrec, ids, &e->ctr->pad); ::dic::note_launch();
    DIC_CHECK_LAUNCH("collect_frequent_kernel");
    if ((rc = read_counters(e))) return rc;
    dfree(ids, e->s);
    *F = (int64_t)e->hctr->pad;
    return DIC_OK;
}

extern "C" int dic_engine_frequent(dic_engine* e, uint64_t* masks_host, int32_t* sizes_host, int64_t* supports_host,
                                   int64_t F) {
    DIC_REQUIRE(e && masks_host && sizes_host && supports_host, "dic_engine_frequent: null argument");
    int rc;
    int32_t* ids = nullptr;
    unsigned long long* dm = nullptr;
    int32_t* dsz = nullptr;
    int64_t* dsu = nullptr;
    if ((rc = dalloc(&ids, std::max<int64_t>(e->nrec, 1), e->s)) || (rc = dalloc(&dm, std::max<int64_t>(F, 1) * e->W, e->s)) ||
        (rc = dalloc(&dsz, std::max<int64_t>(F, 1), e->s)) || (rc = dalloc(&dsu, std::max<int64_t>(F, 1), e->s)))
        return rc;
    DIC_CUDA(cudaMemsetAsync(&e->ctr->pad, 0, sizeof(unsigned long long), e->s));
    collect_frequent_kernel<<<nblk(e->nrec), 256, 0, e->s>>>(e->R, e->nrec, ids, &e->ctr->pad); ::dic::note_launch();
    if ((rc = read_counters(e))) return rc;
    if ((int64_t)e->hctr->pad != F) {
        set_error("dic_engine_frequent: F=%lld but %llu frequent records", (long long)F, e->hctr->pad);
        return DIC_EINVAL;
    }
    if (F > 0) {
        gather_frequent_kernel<<<nblk(F), 256, 0, e->s>>>(e->R, e->W, ids, F, dm, dsz, dsu); ::dic::note_launch();
        DIC_CHECK_LAUNCH("gather_frequent_kernel");
        DIC_CUDA(cudaMemcpyAsync(masks_host, dm, F * e->W * sizeof(uint64_t), cudaMemcpyDeviceToHost, e->s));
        DIC_CUDA(cudaMemcpyAsync(sizes_host, dsz, F * sizeof(int32_t), cudaMemcpyDeviceToHost, e->s));
        DIC_CUDA(cudaMemcpyAsync(supports_host, dsu, F * sizeof(int64_t), cudaMemcpyDeviceToHost, e->s));
    }
    dfree(ids, e->s); dfree(dm, e->s); dfree(dsz, e->s); dfree(dsu, e->s);
    DIC_CUDA(cudaStreamSynchronize(e->s));
    return DIC_OK;
}
