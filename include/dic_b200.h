/*
 * dic_b200.h — C ABI of the B200-native DIC bitmap support count.
 *
 * This is the drop-in boundary for the hot path of the reference `dicmine`
 * package (Python + NumPy; /root/reference/pkg/src/dicmine).  The reference
 * has no FFI of its own: its operator seam is the module-global kernel
 * `_count_block(arr, first, last, mask) -> int` (engine.py:43-58) selected by
 * `count_support_interval` (engine.py:176-223), plus the bitmap builder
 * `encode_transaction` / `BitDatabase` (bitops.py:24-37, database.py:13-86).
 * Each entry point below names the reference function it replaces.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; every data pointer is a DEVICE pointer
 *     unless the comment says "host"; `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream);
 *   - return 0 on success or a negative DIC_E* code; the message for the last
 *     failure on the calling thread is available from dic_last_error();
 *   - argument errors are detected on the host before any launch; data errors
 *     (item id outside [0, m), table overflow) are reported through device
 *     status words that the caller reads after synchronising — kernels never
 *     trap on data;
 *   - everything is asynchronous on `stream` except functions documented as
 *     synchronising.
 *
 * Bit layouts (shared by all kernels):
 *   rows   : uint64 [n][W], W = ceil(m/64); item p of row j is bit (p & 63)
 *            of word (p >> 6) — the reference's single-word layout
 *            (bitops.py:36) extended LSW-first to W words.
 *   tids   : the tiled bit-sliced ("vertical") copy, uint32 words.  Rows are
 *            grouped 32 per word (group g = rows 32g..32g+31, bit b <-> row
 *            32g+b).  A tile holds TW groups of all m items,
 *            TW = dic_tids_tile_groups(m) = 32 (m <= 768) or 16.  Item i's TW
 *            words of tile t form one dense row of 128 or 64 bytes — no pad
 *            words, no swizzle:
 *              word(i, g) = tids[t*m*TW + i*TW + (g - t*TW)],  t = g / TW,
 *            i.e. dic_tids_index(m, i, g).  A tile's global image equals its
 *            shared-memory image, so one bulk copy (TMA engine) stages it.
 *            Rows past n read as zero; the buffer holds
 *            dic_tids_words(n, m) = ceil(ceil(n/32)/TW) * m * TW words —
 *            exactly the bitmap's bits, rounded up to whole tiles.
 *   items  : uint16 [C][k], the k ascending item ids of each candidate of a
 *            size-k bucket (candidates of one launch share k).
 */
#ifndef DIC_B200_H
#define DIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    DIC_OK = 0,
    DIC_EINVAL = -1,   /* bad argument (mirrors the reference's ValueError)   */
    DIC_ECUDA = -2,    /* CUDA launch / runtime failure                        */
    DIC_ENOMEM = -3,   /* device allocation failed                             */
    DIC_EDATA = -4,    /* input data error (e.g. ItemOutOfRange)               */
    DIC_ESTATE = -5    /* engine used out of order                             */
};

#define DIC_ABI_VERSION 1

/* Library / error plumbing --------------------------------------------- */
int dic_abi_version(void);
const char* dic_last_error(void);
/* Number of SMs of the current device (for grid sizing by callers).       */
int dic_device_sm_count(void);
/* Number of kernels this library has launched in the process (monotonic).  */
int64_t dic_launch_count(void);

/* Encoder: CSR item lists -> row bitmap ---------------------------------
 * Replaces encode_transaction (bitops.py:24-37) applied per row, i.e.
 * database_from_transactions (database.py:89-93) / as_bit_database's ragged
 * branch (_validation.py:56).  Duplicates collapse into one bit.
 * rows must hold n*W words; it is fully overwritten.
 * status (device, int64[4], caller-zeroed NOT required — the call resets it):
 *   status[0] = number of duplicate ids collapsed (sum over rows of
 *               len - popcount), the LoadReport dedup figure (datasets.py:160-194)
 *   status[1] = flat CSR position of the FIRST out-of-range id in row-major
 *               order (the one encode_transaction would raise on), or -1
 *   status[2] = its row, or -1
 * The caller reads status after synchronising; status[1] >= 0 maps to
 * ItemOutOfRange(indices[status[1]], line=row). */
int dic_encode_csr(const int64_t* indptr, const int32_t* indices, int64_t n,
                   int32_t m, uint64_t* rows, int64_t* status, void* stream);

/* Row bitmap -> tiled bit-sliced copy (tids, layout above); every word of
 * the dic_tids_words(n, m) buffer is written.                             */
int dic_rows_to_tids(const uint64_t* rows, int64_t n, int32_t m,
                     uint32_t* tids, void* stream);
/* CSR item lists straight into the bit-sliced tiles, rows [row_begin,
 * row_end) only (tile-aligned: multiples of 32*dic_tids_tile_groups(m) rows,
 * row_end may be n), so a loader can encode each slab as soon as its H2D
 * copy lands.  indices are uint16 (index_bytes 2) or int32 (4); indptr is the
 * GLOBAL int64 [n+1] offset array.  status[4] (device int64) accumulates
 * across slabs between dic_encode_status_init and dic_encode_status_finish
 * and then holds what dic_encode_csr reports.  Replaces the same place in
 * the reference as dic_encode_csr (bitops.py:24-37, database.py:13-86).     */
int dic_encode_status_init(int64_t* status, void* stream);
int dic_encode_csr_tids(const int64_t* indptr, const void* indices,
                        int32_t index_bytes, int64_t n, int32_t m,
                        int64_t row_begin, int64_t row_end, uint32_t* tids,
                        int64_t* status, void* stream);
int dic_encode_status_finish(const int64_t* indptr, int64_t n, int64_t* status,
                             void* stream);
/* Inverse transform: bit-sliced tiles -> row bitmap uint64 [n][W] (the host
 * view BitDatabase.masks of a database encoded straight to tiles).        */
int dic_tids_to_rows(const uint32_t* tids, int64_t n, int32_t m, uint64_t* rows,
                     void* stream);
/* Layout helpers (host functions).                                         */
int64_t dic_tids_words(int64_t n, int32_t m);
int dic_tids_tile_groups(int32_t m);
/* Index (in uint32 words) of item i's word of row group g in the tids
 * layout of an m-item universe (the formula above; host callable).        */
int64_t dic_tids_index(int32_t m, int32_t item, int64_t group);

/* First pass: per-item supports -----------------------------------------
 * Replaces first_pass's singleton counting (engine.py:132-154): for every
 * item i < m, counts[i] += #{ j in [first, last] : row j holds i }.
 * counts is ACCUMULATED into (int64), so multi-GPU shards can sum locally. */
int dic_item_support(const uint32_t* tids, int64_t n, int32_t m,
                     int64_t first, int64_t last, int64_t* counts,
                     void* stream);

/* THE hot kernel: candidate support over one chunk ----------------------
 * Replaces _count_block (engine.py:43-58) as called by
 * count_support_interval (engine.py:176-223) for every dashed itemset:
 *   support_inc[c] += #{ j in [first, last] : (rows[j] & I_c) == I_c }
 * computed on the bit-sliced copy as sum_g popc(AND_{i in I_c} tids[i][g]),
 * 0 <= first <= last < n (the caller checks the reference's range rule and
 * raises ValueError; this entry returns DIC_EINVAL on violation).
 * Candidates are one size bucket: items[c*k .. c*k+k-1], 1 <= k <= m.
 * support_inc is accumulated into (uint64 counts).                         */
int dic_count_support(const uint32_t* tids, int64_t n, int32_t m,
                      int64_t first, int64_t last,
                      const uint16_t* items, int32_t k, int64_t C,
                      uint64_t* support_inc, void* stream);

/* All pairs at once: the 2-itemset bucket as a dense triangle ----------
 * For every pair of items a < b < m of a tids layout:
 *   tri[a*m - a*(a+1)/2 + (b-a-1)] += #{ j in [first, last] : row j holds a and b }
 * (a-major, the order first_pass seeds pairs in, engine.py:165-168).  The
 * count is the Gram matrix X^T X of the chunk's 0/1 matrix: for m >= 128
 * items it runs on the tensor cores (tcgen05.mma kind::i8, u8 operands
 * expanded from the bits in shared memory, s32 accumulators in TMEM, exact);
 * below that, or when selected, as a register-blocked AND/POPC kernel over
 * 64 x 64 blocks.  tri holds m*(m-1)/2 uint64 counts, accumulated into.     */
int dic_count_pairs(const uint32_t* tids, int64_t n, int32_t m,
                    int64_t first, int64_t last, uint64_t* tri, void* stream);
/* Which kernel dic_count_pairs (and the engine's pair stops) use, process-
 * wide: -1 = from the environment (DIC_PAIR_TC, default on), 0 = automatic
 * (tensor cores for m >= 128), 1 = AND/POPC, 2 = tensor cores; *previous
 * (optional) receives the mode it replaces.  Engines apply it when they next
 * capture a stop graph.                                                    */
int dic_pair_kernel_select(int32_t mode, int32_t* previous);
/* The tids layout restricted to items[0..L) (in that order, L <= m); out
 * holds dic_tids_words(n, L) words.  Lets dic_count_pairs run over the
 * frequent items only.                                                    */
int dic_tids_select(const uint32_t* tids, int64_t n, int32_t m,
                    const int32_t* items, int32_t L, uint32_t* out, void* stream);

/* The same count on the row bitmap, the literal `(T & I) == I` form of
 * _count_block (engine.py:54-56) for C multi-word masks [C][W].  Used as an
 * independent second kernel for parity checks and for callers that only
 * hold the row bitmap.  support_inc is accumulated into.                  */
int dic_count_support_rows(const uint64_t* rows, int32_t W,
                           int64_t first, int64_t last,
                           const uint64_t* masks, int64_t C,
                           uint64_t* support_inc, void* stream);

/* Candidate generation + subset pruning ---------------------------------
 * Replaces make_candidates' join/admission loop (engine.py:320-369) for the
 * API-level call on a host catalog.  `box_masks` [B][W] is the set of masks
 * currently known with a box shape, `known_masks` [K][W] every known mask
 * (any shape).  For every (s, l) with s < S, l < L:
 *   cand = src_masks[s] | (1 << level1[l]);
 *   admit[s*L + l] = cand != src && cand not in known && every immediate
 *                    subset of cand is in box_masks.
 * The caller applies the reference's first-occurrence dedup in (s, l) order.
 * Synchronising (builds a temporary device hash set).                     */
int dic_candidate_admission(const uint64_t* src_masks, int64_t S,
                            const int32_t* level1, int64_t L, int32_t W,
                            const uint64_t* known_masks, int64_t K,
                            const uint64_t* box_masks, int64_t B,
                            uint8_t* admit, void* stream);

/* Pattern containment (DicMiner.transform, estimator.py:90-99) ------------
 * P patterns as concatenated ascending item ids items[offs[p] .. offs[p+1])
 * (device uint16 / int64 [P+1]; an empty pattern is in every row, one with an
 * item >= m in none).  dic_containment writes the row-major bool matrix
 * out[n][P] (uint8 0/1); dic_containment_packed the bit matrix out[G][P]
 * (uint32, G = ceil(n/32)): bit r of word (g, p) = row 32g + r contains p. */
int dic_containment(const uint32_t* tids, int64_t n, int32_t m,
                    const uint16_t* items, const int64_t* offs, int64_t P,
                    uint8_t* out, void* stream);
int dic_containment_packed(const uint32_t* tids, int64_t n, int32_t m,
                           const uint16_t* items, const int64_t* offs, int64_t P,
                           uint32_t* out, void* stream);

/* Device-resident DIC engine ---------------------------------------------
 * The checkpoint loop of _run (engine.py:398-458) with the catalog
 * (itemsets.py:88-136) held on the device as structure-of-arrays plus a
 * hash index of every mask ever created (`known`).  One engine per rank;
 * each rank holds the LOCAL rows of its shard (chunk-sliced
 * sharding), the state machine is replicated on every rank.             */
typedef struct dic_engine dic_engine;

typedef struct dic_stop_status {
    int64_t dashed_at_start;  /* |dashed| counted at this stop (interval_counts) */
    int64_t promoted;         /* DASHED_CIRCLE -> DASHED_BOX (prune, :296-298)  */
    int64_t pruned;           /* DASHED_CIRCLE -> NIL by the bound (:299-310)    */
    int64_t inserted;         /* new candidates (make_candidates, :366-369)      */
    int64_t dashed_peak;      /* |dashed| after make_candidates (peak, :440)     */
    int64_t finalized;        /* dashed -> solid (check_full_pass, :372-390)     */
    int64_t dashed_at_end;    /* |dashed| after compaction (loop test, :423)     */
    int64_t records;          /* itemsets ever created (|known|)                 */
} dic_stop_status;

/* tids/n_local: this rank's bit-sliced rows (owned by the caller, must
 * outlive the engine).  need = ceil(minsup*n) (params.py:17-19),
 * interval = M, stop_max = ceil(n/M) over the GLOBAL n.                   */
int dic_engine_create(const uint32_t* tids, int64_t n_local,
                      int32_t m, int64_t need, int64_t interval,
                      int64_t stop_max, int32_t prune_bound, void* stream,
                      dic_engine** out);
int dic_engine_destroy(dic_engine* e);
/* first_pass (engine.py:105-173), step 1: local per-item counts into
 * counts[m] (device int64, overwritten).  Multi-GPU callers sum-allreduce
 * counts before step 2.                                                   */
int dic_engine_item_counts(dic_engine* e, int64_t* counts);
/* step 2: singleton records (SOLID_BOX / SOLID_CIRCLE, intervals=stop_max),
 * level1, and every frequent pair seeded as DASHED_CIRCLE.  Synchronising;
 * returns |level1| and the number of pairs seeded.                        */
int dic_engine_seed(dic_engine* e, const int64_t* counts,
                    int64_t* n_level1, int64_t* n_pairs);
/* Per stop, step 1: count every dashed candidate over LOCAL rows
 * [lfirst, llast] into the delta buffer (zeroed here).  lfirst > llast
 * (an empty local slice) is allowed and counts nothing.                  */
int dic_engine_count(dic_engine* e, int64_t lfirst, int64_t llast);
/* The delta buffer (device uint64/int64 [*len]) for the per-stop
 * sum-allreduce across ranks; valid until the next checkpoint.           */
int dic_engine_delta(dic_engine* e, void** ptr, int64_t* len);
/* Per stop, step 2: support += delta, intervals += 1, prune, make
 * candidates, check_full_pass, compact.  Synchronising; fills *st.       */
int dic_engine_checkpoint(dic_engine* e, dic_stop_status* st);
/* Pipelined form of the same loop (what mine_parallel uses).  Every kernel
 * of a stop reads its sizes from device memory, so the host can enqueue stop
 * s while stop s-D is still running:
 *   dic_engine_issue_count(e, lfirst, llast)   count into the delta buffer
 *   [sum-allreduce of dic_engine_delta() across ranks, same stream]
 *   dic_engine_issue_checkpoint(e, &seq)       apply / prune / candidates
 *   dic_engine_poll(e, seq, &st, &replayed)    wait for stop seq, in order
 * A stop whose new candidates do not fit raises a device abort flag that
 * turns every later kernel into a no-op; poll() then grows the arrays,
 * replays that stop's candidate step and sets *replayed = 1: the caller
 * must re-issue every stop after seq.  At most 15 stops in flight.
 * dic_engine_delta's length is the (rank-independent) slot capacity.      */
int dic_engine_issue_count(dic_engine* e, int64_t lfirst, int64_t llast);
/* Declare the chunk cycle of the coming stops: the next issued stop counts
 * local rows [lfirst[0], llast[0]], the one after [lfirst[1], llast[1]], ...
 * wrapping after nstops.  A dic_engine_issue_count() whose chunk matches the
 * schedule launches the stop's count as one captured CUDA graph (the chunk is
 * read on the device); any other chunk takes the direct launch path.  The
 * checkpoint half is always a graph.  graphs_captured / graph_launches are
 * diagnostics (dic_engine_graph_stats).                                   */
int dic_engine_set_schedule(dic_engine* e, const int64_t* lfirst,
                            const int64_t* llast, int64_t nstops);
int dic_engine_graph_stats(dic_engine* e, int64_t* graphs_captured,
                           int64_t* graph_launches);
/* The dense pair-triangle counts of the stop (device uint64/int64 [*len],
 * *len == 0 when the engine has none): sharded callers sum-allreduce it
 * together with dic_engine_delta() before the checkpoint.                 */
int dic_engine_pair_counts(dic_engine* e, void** ptr, int64_t* len);
int dic_engine_issue_checkpoint(dic_engine* e, int64_t* seq);
int dic_engine_poll(dic_engine* e, int64_t seq, dic_stop_status* st,
                    int32_t* replayed);
/* The whole pipelined loop on one unsharded GPU, natively: stop s (1-based,
 * wrapping after stop_max) counts local rows [lfirst[s-1], llast[s-1]] and
 * scans rows[s-1] global rows; `depth` stops in flight.  *out receives the
 * loop's MiningStats counters; count_ms / dashed (optional, max_stops
 * entries) the CUDA-event time of each stop's count launches and its
 * |dashed| at start.                                                      */
typedef struct dic_run_stats {
    int64_t stops;
    int64_t scanned;
    int64_t interval_counts;
    int64_t candidates_generated;
    int64_t candidates_pruned;
    int64_t peak_dashed;
    int64_t replays;     /* candidate-capacity replays (diagnostic)            */
    double issue_us;     /* host time spent enqueuing stops (diagnostic)       */
    double poll_us;      /* host time spent waiting for / reading statuses     */
    int64_t graphs_captured;  /* stop graphs (re-)captured during the run        */
    int64_t batches;          /* launches that ran several quiet stops at once   */
    int64_t batched_stops;    /* stops run by those launches                     */
} dic_run_stats;
int dic_engine_run(dic_engine* e, const int64_t* lfirst, const int64_t* llast,
                   const int64_t* rows, int64_t stop_max, int32_t depth,
                   dic_run_stats* out, float* count_ms, int64_t* dashed,
                   int64_t max_stops);
/* Multi-GPU without a Python framework in the loop: an NCCL communicator
 * built here (rank 0 draws the 128-byte id, every rank passes it to
 * dic_nccl_comm_init, which blocks until all ranks joined) and attached to the
 * engine BEFORE dic_engine_item_counts.  The engine then sum-allreduces the
 * item counts and, per stop between the count and checkpoint halves, the
 * delta buffer (and the pair triangle while it is dense) on its own stream —
 * the per-checkpoint int64 allreduce of SURVEY §8(e), also inside
 * dic_engine_run.                                                          */
int dic_nccl_unique_id(uint8_t* out /* [128] */);
int dic_nccl_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, void** comm);
int dic_nccl_comm_destroy(void* comm);
int dic_engine_set_comm(dic_engine* e, void* comm);
/* How the engine reduces a stop's counts across ranks: 0 = not sharded,
 * 1 = ncclAllReduce of the delta buffer and the dense pair triangle,
 * 2 = fused: the count kernels write per-rank partials
 *     into NCCL symmetric windows and one kernel per stop sums the partials of
 *     every NVLink (LSA) peer straight from peer memory, sized on the device
 *     by the live slots; chosen by dic_engine_set_comm when every rank is in
 *     one LSA team and DIC_FUSED_REDUCE is not 0.                          */
int dic_engine_collective_mode(dic_engine* e);

/* Results: number of SOLID_BOX records, then copy them out to HOST arrays
 * masks[F][W] (uint64), sizes[F], supports[F] in the reference's canonical
 * order (engine.py:446-455): by size, then mask as an integer (MSW first).
 * Synchronising.                                                          */
int dic_engine_num_frequent(dic_engine* e, int64_t* F);
int dic_engine_frequent(dic_engine* e, uint64_t* masks_host,
                        int32_t* sizes_host, int64_t* supports_host,
                        int64_t F);
/* Words per mask of this engine (W = ceil(m/64)).                        */
int dic_engine_words(dic_engine* e);
/* Replicated layout.  The record ids and bucket positions a stop gives its
 * new candidates are canonical: candidates of the stop are ordered by
 * (size, item ids ascending) and numbered in that order, so they depend only
 * on the set of candidates (never on thread timing), and compaction keeps
 * order.  Every rank of a sharded run therefore holds the same slot layout
 * and the slot-indexed delta / triangle reductions add counts of the same
 * itemsets (the reference reduces per record, engine.py:268-270).
 * Diagnostics: bucket k (itemsets of k items) as the device holds it now —
 * *n filled slots (live and dead); with rec_host non-null, their record ids
 * and item lists (items_host[n][k], ascending) are copied out (cap >= *n).
 * Synchronises the engine's stream.                                        */
int dic_engine_bucket(dic_engine* e, int32_t k, int32_t* rec_host,
                      uint16_t* items_host, int64_t cap, int64_t* n);

/* Synthetic generators (host, multithreaded, counter-based RNG) ---------
 * Seeded restatements of BASELINE.json's config generators (DESIGN.md
 * §Inputs).  Rows are generated for the GLOBAL row ranges
 * [range_begin[i], range_begin[i] + range_len[i]) concatenated in order, so a
 * rank can generate exactly its shard; output is identical for any thread
 * count and any range split.  The result is an opaque host CSR.          */
typedef struct dic_csr dic_csr;
int dic_synth_zipf(const int64_t* range_begin, const int64_t* range_len,
                   int nranges, int32_t m, double s, double mean_len,
                   uint64_t seed, int threads, dic_csr** out);
int dic_synth_quest(const int64_t* range_begin, const int64_t* range_len,
                    int nranges, int32_t m, int32_t n_patterns,
                    double pattern_len, double mean_len, uint64_t seed,
                    int threads, dic_csr** out);
int dic_synth_dense(const int64_t* range_begin, const int64_t* range_len,
                    int nranges, int32_t m, int32_t groups,
                    int32_t group_size, double group_p, uint64_t seed,
                    int threads, dic_csr** out);
int dic_csr_info(const dic_csr* c, int64_t* n, int64_t* nnz);
/* host arrays: indptr[n+1], indices[nnz]                                  */
int dic_csr_export(const dic_csr* c, int64_t* indptr, int32_t* indices);
void dic_csr_free(dic_csr* c);

/* Transaction text format (datasets.py:150-209) --------------------------
 * Parse a whole file image into CSR (threads workers).  On a bad token the
 * call returns DIC_EDATA with st->kind 1 (not an integer) or 2 (outside
 * [0, max_item)), st->line its 1-based line (blank and comment lines
 * counted, as the reference's enumerate(fh, 1)), st->offset / length the
 * token's bytes; kind 3 = a non-ASCII byte (the caller decodes in Python).
 * On success st->line = lines read.                                        */
typedef struct dic_parse_status {
    int32_t kind;
    int32_t reserved;
    int64_t line;
    int64_t offset;
    int64_t length;
} dic_parse_status;
int dic_parse_transactions(const char* text, int64_t len, int32_t max_item,
                           int32_t threads, dic_csr** out, dic_parse_status* st);
/* Canonical text of rows [n][W] (ascending ids, one newline per row) in a malloc'd
 * buffer the caller releases with dic_free_buffer.                        */
int dic_format_transactions(const uint64_t* rows, int64_t n, int32_t W,
                            int32_t threads, char** out, int64_t* len);
void dic_free_buffer(char* p);
/* cfg5: row bitmap rows[n][W] of i.i.d. Bernoulli(p) bits, generated on the
 * device; and C candidates (host arrays) with k ~ U{kmin..kmax} items drawn
 * uniformly without replacement: cand_k[C], cand_items[C][kmax] ascending,
 * unused slots 0xFFFF.                                                    */
int dic_synth_bernoulli_rows(int64_t n, int32_t m, double p, uint64_t seed,
                             uint64_t* rows, void* stream);
int dic_synth_candidates(int64_t C, int32_t m, int32_t kmin, int32_t kmax,
                         uint64_t seed, int32_t* cand_k, uint16_t* cand_items);

/* Peak probes (for the roofline denominators) ---------------------------
 * Runs `iters` iterations of an unrolled LOP3 (op=0), POPC (op=1) or IADD
 * (op=2) chain on every thread of blocks x threads; *sink is written only
 * under a data-dependent (practically false) condition so nothing is dead.
 * Synchronising; returns the lane-ops issued and the CUDA-event time.     */
int dic_probe_int_pipe(int op, int blocks, int threads, int64_t iters,
                       uint32_t* sink, double* lane_ops, float* ms,
                       void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DIC_B200_H */
