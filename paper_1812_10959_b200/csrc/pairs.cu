// pairs.cu — the 2-itemset bucket counted as a dense triangle.
//
// first_pass seeds EVERY pair of frequent items as a candidate
// (engine.py:165-168), all in the same stop, so they are counted over the
// same chunks and finalised together: for the configs' large universes this
// C(|L1|, 2) wave is nearly all of the work (cfg4: 499,500 pairs x 10M rows).
// Counting it pair by pair re-reads both item rows for every pair.  Here a
// CTA owns a 64 x 64 block of the pair triangle and streams the chunk past it
// like a GEMM's K dimension — but on the integer pipes (AND + POPC), no
// tensor cores: each thread holds a 4 x 4 register tile of pair counters and
// per 128 rows loads 4 + 4 item words (LDS.128) for 16 AND/POPC updates, so
// shared-memory traffic per subset-test drops 8x and the POPC pipe is the
// bound.  Row blocks of a tile are contiguous in the tiled layout, so each
// operand block arrives by one bulk async copy (TMA engine), double-buffered.
#include "async.cuh"

#include <atomic>
#include <map>
#include <mutex>

namespace dic {

constexpr int kPairBlock = 64;
constexpr int kPairThreads = 256;  // 16 x 16 threads, a 4 x 4 pair tile each

__host__ __device__ inline int64_t tri_index(int64_t a, int64_t b, int64_t m) {
    // a < b < m, a-major: the order first_pass seeds pairs in
    return a * m - a * (a + 1) / 2 + (b - a - 1);
}

// Block pair bi (row-major over the upper triangle of nblk x nblk item
// blocks) -> item ranges.
struct PairBlock {
    int a0, b0, na, nb;
    bool diag;
};
__device__ __forceinline__ PairBlock pair_block(int64_t bi, int nblk, int m) {
    int y = (int)bi, I = 0;
    while (y >= nblk - I) {
        y -= nblk - I;
        ++I;
    }
    PairBlock p;
    p.a0 = I * kPairBlock;
    p.b0 = (I + y) * kPairBlock;
    p.na = min(kPairBlock, m - p.a0);
    p.nb = min(kPairBlock, m - p.b0);
    p.diag = y == 0;
    return p;
}

// One (block pair, tile) unit, decoded once by the producer thread into the
// stage's descriptor so the consumers do no 64-bit division per tile.
struct PairUnit {
    int64_t bi;  // block pair; < 0: no unit (end of the CTA's work)
    int64_t t;   // tile
    int a0, b0, na, nb;
    int diag, edge;
};
constexpr int kPairStages = 3;

// The 4 x 4 register tile over one 8-word step.  DIAG: register groups i > j
// of a diagonal block hold no pair (a = ta + 16i >= 16i > tb + 16j), so they
// are not emitted — 6 of 16 and_popc8 per step.  NJ: register columns
// j >= NJ lie past the last item of a partial B block (nb <= 16 NJ) and are
// not emitted either (cfg4: the 40-item last block, 15 of 136 block pairs).
template <bool DIAG, int CH, int NJ = 4>
__device__ __forceinline__ void pair_step(const uint8_t* A, const uint8_t* B, int RB, int ta, int tb, int q,
                                          uint32_t (&cnt)[4][4], uint32_t one) {
    // Item rows are dense (64 or 128 bytes): the 16 lanes of a half-warp read
    // 16 different A rows, so each walks the row's CH chunks from another
    // start (a pair's AND may take its row groups in any order): a
    // quarter-warp then covers 8 distinct bank groups with its A loads and
    // one contiguous B row segment.
    const int rot = CH == 8 ? ta : (ta >> 1);
    const int c0 = ((q + rot) & (CH - 1)) * 16, c1 = ((q + 1 + rot) & (CH - 1)) * 16;
    uint4 av0[4], av1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        av0[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + c0);
        av1[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + c1);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const uint4 bv0 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + c0);
        const uint4 bv1 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + c1);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (DIAG && i > j) continue;
            cnt[i][j] = and_popc8_acc(av0[i], av1[i], bv0, bv1, cnt[i][j], one);
        }
    }
}

// Producer state, in shared memory: whichever warp refills a stage runs it.
struct PairProd {
    int64_t icur, iend;  // claimed unit range
    int dry;             // no units left
};

// Persistent: the (block pair, tile) units of the chunk, block-pair major.
// The first static_pct % are split evenly over the grid (each CTA walks a
// contiguous run of tiles of one or two block pairs, so counters are flushed
// with atomics rarely); the rest is claimed in grains of `grain` units from
// sched[0], so CTAs that ran slower than their SM-mates (the warp scheduler
// does not share an SM evenly between CTAs) do not leave a tail.  The last
// CTA to finish re-zeroes sched[] for the next launch on the stream.
//
// Stages: a 3-deep ring of (descriptor, A row block, B row block), each
// filled by bulk async copies (TMA) that complete on the stage's mbarrier.
// There is no CTA-wide barrier per tile: every warp counts its arrival on
// the stage it consumed, and the LAST warp to arrive refills it (decodes the
// next unit into the descriptor and issues its copies), so no warp waits for
// a designated producer and the refill starts the moment the stage is free.
template <int TW, int MINB>
__global__ void __launch_bounds__(kPairThreads, MINB) pair_tri_kernel(const uint32_t* __restrict__ tids, int m,
                                                                   ChunkGeom geom, int64_t t_first, int64_t t_last,
                                                                   int nblk, unsigned long long* __restrict__ tri,
                                                                   const unsigned long long* bn2, int64_t tri_len,
                                                                   const unsigned long long* abort_flag,
                                                                   const int64_t* chunk_ring,
                                                                   const unsigned long long* seq, int ring,
                                                                   unsigned long long* __restrict__ sched,
                                                                   int static_pct, int grain, uint32_t one) {
    // engine use: skip while aborted, or once the pair bucket is mostly gone
    // (every CTA reads the same values, so either all return here or none)
    if (abort_flag && (*abort_flag || 2 * (int64_t)*bn2 < tri_len)) return;
    if (chunk_ring) {
        // engine graphs: the stop's chunk comes from the ring slot of *seq
        const int64_t sl = (int64_t)(*seq % (unsigned long long)ring);
        const int64_t f = chunk_ring[2 * sl], l = chunk_ring[2 * sl + 1];
        if (l < f) return;
        geom = chunk_geom(f, l);
        t_first = geom.g_first / TW;
        t_last = geom.g_last / TW;
    }
    constexpr int RW = row_words(TW);
    constexpr int RB = RW * 4;
    constexpr uint32_t BLK = kPairBlock * RB;
    constexpr int NW = kPairThreads / 32;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);                  // [kPairStages]
    uint32_t* arrived = reinterpret_cast<uint32_t*>(smem + 24);           // [kPairStages]
    PairProd* prod = reinterpret_cast<PairProd*>(smem + 40);
    PairUnit* desc = reinterpret_cast<PairUnit*>(smem + 64);              // [kPairStages]
    uint8_t* buf = smem + 256;                                            // [stage][A block, B block]

    const int64_t tile_words = (int64_t)m * RW;
    const int64_t nt = t_last - t_first + 1;
    const int64_t U = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const int64_t US = U * static_pct / 100;
    // the refilling lane: decode the next unit into desc[s] and issue it
    auto issue = [&](int s) {
        PairProd& P = *prod;
        PairUnit& d = desc[s];
        int64_t u = -1;
        if (!P.dry) {
            if (P.icur == P.iend) {
                P.icur = US + (int64_t)atomicAdd(sched, 1ull) * grain;
                P.iend = P.icur + grain < U ? P.icur + grain : U;
                if (P.icur >= U) P.dry = 1;
            }
            if (!P.dry) u = P.icur++;
        }
        if (u < 0) {
            d.bi = -1;
            mbar_arrive(&full[s]);
            return;
        }
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        const PairBlock pb = pair_block(bi, nblk, m);
        d.bi = bi;
        d.t = t;
        d.a0 = pb.a0;
        d.b0 = pb.b0;
        d.na = pb.na;
        d.nb = pb.nb;
        d.diag = pb.diag;
        d.edge = (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last);
        const uint32_t ab = (uint32_t)pb.na * RB, bb = (uint32_t)pb.nb * RB;
        uint8_t* dst = buf + (size_t)s * 2 * BLK;
        const uint32_t* src = tids + t * tile_words;
        mbar_expect_tx(&full[s], ab + (pb.diag ? 0u : bb));
        bulk_g2s(dst, src + (int64_t)pb.a0 * RW, ab, &full[s]);
        if (!pb.diag) bulk_g2s(dst + BLK, src + (int64_t)pb.b0 * RW, bb, &full[s]);
    };
    if (threadIdx.x == 0) {
        prod->icur = US * blockIdx.x / gridDim.x;
        prod->iend = US * (blockIdx.x + 1) / gridDim.x;
        prod->dry = 0;
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);
            arrived[s] = 0;
        }
        fence_mbar_init();
        for (int s = 0; s < kPairStages; ++s) issue(s);
    }
    __syncthreads();

    const int ta = threadIdx.x & 15, tb = threadIdx.x >> 4;
    const int lane = threadIdx.x & 31;
    uint32_t cnt[4][4];
    int64_t cur = -1;
    int a0 = 0, b0 = 0;
    auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int a = a0 + ta + 16 * i, b = b0 + tb + 16 * j;
                if (a < b && b < m && cnt[i][j]) atomicAdd(tri + tri_index(a, b, m), (unsigned long long)cnt[i][j]);
            }
    };

    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % kPairStages);
        mbar_wait(&full[s], (uint32_t)((k / kPairStages) & 1));
        const PairUnit& d = desc[s];
        const int64_t bi = d.bi;
        if (bi < 0) break;
        const bool diag = d.diag;
        if (bi != cur) {
            if (cur >= 0) flush();
            cur = bi;
            a0 = d.a0;
            b0 = d.b0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) cnt[i][j] = 0;
        }
        uint8_t* A = buf + (size_t)s * 2 * BLK;
        uint8_t* B = diag ? A : A + BLK;
        if (d.edge) {
            // chunk edge inside this tile: zero the rows outside [first, last]
            // (every warp meets this barrier for the same tile)
            const int na = d.na, nb = d.nb;
            const int64_t g0 = d.t * TW;
            const int rows = diag ? na : 2 * kPairBlock;
            for (int idx = threadIdx.x; idx < rows * RW; idx += kPairThreads) {
                const int r = idx / RW, slot = idx - r * RW;
                if (slot >= TW || (r < kPairBlock ? r >= na : r - kPairBlock >= nb)) continue;
                uint32_t* w = reinterpret_cast<uint32_t*>(A + (size_t)r * RB) + slot;
                *w &= group_mask(geom, g0 + slot);
            }
            __syncthreads();
        }
        // two 16-byte chunks (8 words = 256 rows) per step; per pair the 8
        // AND'ed words go through a carry-save tree (7 -> ones/twos/fours,
        // plus one leftover): 16 LOP3 + 4 POPC instead of 8 LOP3 + 8 POPC,
        // which balances the ALU (64 lanes/SM/clk) and POPC (16) pipes
        if (diag) {
#pragma unroll
            for (int q = 0; q < TW / 4; q += 2) pair_step<true, TW / 4>(A, B, RB, ta, tb, q, cnt, one);
        } else if (d.nb <= 48) {
#pragma unroll
            for (int q = 0; q < TW / 4; q += 2) pair_step<false, TW / 4, 3>(A, B, RB, ta, tb, q, cnt, one);
        } else {
#pragma unroll
            for (int q = 0; q < TW / 4; q += 2) pair_step<false, TW / 4>(A, B, RB, ta, tb, q, cnt, one);
        }
        // stage s consumed by this warp; the last warp refills it
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&arrived[s], 1u) == NW - 1) {
                arrived[s] = 0;
                __threadfence_block();
                fence_proxy_async();
                issue(s);
            }
        }
    }
    if (cur >= 0) flush();
    __syncthreads();
    if (threadIdx.x == 0) {
        // the last CTA out re-arms the grain counter for the next launch
        __threadfence();
        if (atomicAdd(sched + 1, 1ull) == gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
        }
    }
}

// Bit-sliced copy restricted to the selected items (in the given order).
__global__ void tids_select_kernel(const uint32_t* __restrict__ src, int64_t n, int m,
                                   const int32_t* __restrict__ items, int L, uint32_t* __restrict__ dst) {
    const int TWs = tile_groups(m), TWd = tile_groups(L);
    const int RWd = row_words(TWd);
    const int64_t src_groups = tile_count(n, m) * TWs;
    const int64_t total = tile_count(n, L) * (int64_t)L * RWd;
    for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < total; d += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = d / ((int64_t)L * RWd);
        const int64_t rem = d - t * L * RWd;
        const int r = (int)(rem / RWd), slot = (int)(rem - (int64_t)r * RWd);
        uint32_t v = 0;
        const int64_t g = t * TWd + slot;
        if (slot < TWd && g < src_groups) v = src[tids_index(m, TWs, (uint32_t)items[r], g)];
        dst[d] = v;
    }
}

static int g_pair_slots[4] = {0, 0, 0, 0};  // resident CTAs per SM for (TW = 16 / 32) x (MINB = 3 / 4)

static int env_int(const char* name, int dflt, int lo, int hi) {
    const char* e = getenv(name);
    if (!e || !*e) return dflt;
    return std::min(hi, std::max(lo, atoi(e)));
}
// hybrid schedule: the statically split share (percent) and the grain (units)
// of the dynamically claimed rest (cfg4 chunks: 50 / 4, tools/lab/sweep_pair.sh)
static int pair_static_pct() {
    static const int v = env_int("DIC_PAIR_STATIC_PCT", 50, 0, 100);
    return v;
}
static int pair_grain() {
    static const int v = env_int("DIC_PAIR_GRAIN", 4, 1, 1 << 20);
    return v;
}
static int pair_minb() {
    static const int v = env_int("DIC_PAIR_MINB", 3, 3, 4) == 4 ? 4 : 3;
    return v;
}

// grain counters for launches without an engine-owned pair (the C-ABI entry):
// one 2-word device buffer per (device, stream), kept for the process
static unsigned long long* stream_sched(cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, unsigned long long*> bufs;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    auto& p = bufs[{dev, s}];
    if (!p) {
        void* q = nullptr;
        if (cudaMalloc(&q, 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
        if (cudaMemsetAsync(q, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess) {
            cudaFree(q);
            return nullptr;
        }
        p = static_cast<unsigned long long*>(q);
    }
    return p;
}

template <int TW, int MINB>
int pair_launch(const uint32_t* tids, int m, ChunkGeom geom, int64_t t_first, int64_t t_last, int nblk,
                int64_t units, unsigned long long* tri, const unsigned long long* bn2, int64_t tri_len,
                const unsigned long long* abort_flag, const int64_t* chunk_ring, const unsigned long long* seq,
                int ring, unsigned long long* sched, cudaStream_t s) {
    const size_t smem = 256 + (size_t)kPairStages * 2 * kPairBlock * row_words(TW) * 4;
    int& per_sm = g_pair_slots[(TW == 32 ? 1 : 0) + (MINB == 4 ? 2 : 0)];
    if (per_sm == 0) {
        DIC_CUDA(cudaFuncSetAttribute(pair_tri_kernel<TW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        DIC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pair_tri_kernel<TW, MINB>, kPairThreads, smem));
        per_sm = std::max(per_sm, 1);
    }
    // persistent: one CTA per resident slot (fewer when the chunk is small)
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)per_sm * sm_count()));
    pair_tri_kernel<TW, MINB><<<grid, kPairThreads, smem, s>>>(tids, m, geom, t_first, t_last, nblk, tri, bn2,
                                                                tri_len, abort_flag, chunk_ring, seq, ring, sched,
                                                                pair_static_pct(), pair_grain(), 1u);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("pair_tri_kernel");
    return DIC_OK;
}

int pair_tc_launch(const uint32_t* tids, int64_t n, int L, ChunkGeom geom, unsigned long long* tri,
                   const unsigned long long* bn2, int64_t tri_len, const unsigned long long* abort_flag,
                   const int64_t* chunk_ring, const unsigned long long* seq, int ring, cudaStream_t s);

// The tensor-core triangle (pairs_mma.cu) for universes of at least
// DIC_PAIR_TC_MIN items (default 128); DIC_PAIR_TC=0 keeps the LOP3/POPC
// kernel.  dic_pair_kernel_select() overrides both (tests, A/B probes).
static std::atomic<int> g_pair_mode{-1};  // -1: from the environment, 0: auto, 1: LOP3, 2: tensor cores
static bool pair_use_tc(int m) {
    static const int on = env_int("DIC_PAIR_TC", 1, 0, 1);
    static const int lo = env_int("DIC_PAIR_TC_MIN", 128, 2, 1 << 16);
    const int mode = g_pair_mode.load();
    if (mode == 1) return false;
    if (mode == 2) return true;
    return (mode == 0 || on) && m >= lo;
}

int count_pairs_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                       unsigned long long* tri, cudaStream_t s, const unsigned long long* bn2 = nullptr,
                       int64_t tri_len = 0, const unsigned long long* abort_flag = nullptr,
                       const int64_t* chunk_ring = nullptr, const unsigned long long* seq = nullptr,
                       int ring = 0, unsigned long long* sched = nullptr) {
    // with a chunk ring, [first, last] only sizes the grid (the largest chunk)
    if (last < first || m < 2) return DIC_OK;
    if (pair_use_tc(m))
        return pair_tc_launch(tids, n, m, chunk_geom(first, last), tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring,
                              s);
    if (!sched && !(sched = stream_sched(s))) {
        set_error("dic_count_pairs: no device memory for the grain counters");
        return DIC_ENOMEM;
    }
    const int TW = tile_groups(m);
    const ChunkGeom geom = chunk_geom(first, last);
    const int64_t t_first = geom.g_first / TW, t_last = geom.g_last / TW;
    const int64_t nt = t_last - t_first + 1;
    const int nblk = (m + kPairBlock - 1) / kPairBlock;
    const int64_t units = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const bool b4 = pair_minb() == 4;
    if (TW == 32)
        return b4 ? pair_launch<32, 4>(tids, m, geom, t_first, t_last, nblk, units, tri, bn2, tri_len, abort_flag,
                                       chunk_ring, seq, ring, sched, s)
                  : pair_launch<32, 3>(tids, m, geom, t_first, t_last, nblk, units, tri, bn2, tri_len, abort_flag,
                                       chunk_ring, seq, ring, sched, s);
    return b4 ? pair_launch<16, 4>(tids, m, geom, t_first, t_last, nblk, units, tri, bn2, tri_len, abort_flag,
                                   chunk_ring, seq, ring, sched, s)
              : pair_launch<16, 3>(tids, m, geom, t_first, t_last, nblk, units, tri, bn2, tri_len, abort_flag,
                                   chunk_ring, seq, ring, sched, s);
}

int tids_select_launch(const uint32_t* src, int64_t n, int m, const int32_t* items, int L, uint32_t* dst,
                       cudaStream_t s) {
    const int64_t total = tile_count(n, L) * (int64_t)L * row_words(tile_groups(L));
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
    tids_select_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(src, n, m, items, L, dst);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("tids_select_kernel");
    return DIC_OK;
}

// engine: pairs of the current stop into the delta slots of bucket 2
int count_pairs_dev_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                           unsigned long long* tri, const unsigned long long* bn2, int64_t tri_len,
                           const unsigned long long* abort_flag, cudaStream_t s,
                           const int64_t* chunk_ring = nullptr, const unsigned long long* seq = nullptr,
                           int ring = 0, unsigned long long* sched = nullptr) {
    // tri is all-zero between stops: the gather re-zeroes every entry it reads
    return count_pairs_launch(tids, n, m, first, last, tri, s, bn2, tri_len, abort_flag, chunk_ring, seq, ring,
                              sched);
}


}  // namespace dic

using namespace dic;

extern "C" int dic_count_pairs(const uint32_t* tids, int64_t n, int32_t m, int64_t first, int64_t last,
                               uint64_t* tri, void* stream) {
    DIC_REQUIRE(m >= 2 && m <= 65535 && tids && tri, "dic_count_pairs: bad arguments (m=%d)", m);
    DIC_REQUIRE(0 <= first && first <= last && last < n, "chunk [%lld, %lld] outside database of %lld rows",
                (long long)first, (long long)last, (long long)n);
    return count_pairs_launch(tids, n, m, first, last, reinterpret_cast<unsigned long long*>(tri),
                              as_stream(stream));
}

extern "C" int dic_tids_select(const uint32_t* tids, int64_t n, int32_t m, const int32_t* items, int32_t L,
                               uint32_t* out, void* stream) {
    DIC_REQUIRE(n >= 1 && m >= 1 && L >= 1 && L <= m && tids && items && out, "dic_tids_select: bad arguments");
    return tids_select_launch(tids, n, m, items, L, out, as_stream(stream));
}

extern "C" int dic_pair_kernel_select(int32_t mode, int32_t* previous) {
    DIC_REQUIRE(mode >= -1 && mode <= 2, "dic_pair_kernel_select: mode %d (-1 env, 0 auto, 1 LOP3, 2 tensor)", mode);
    const int prev = g_pair_mode.exchange(mode);
    if (previous) *previous = prev;
    return DIC_OK;
}
