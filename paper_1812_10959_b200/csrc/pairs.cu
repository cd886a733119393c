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

// Persistent: the (block pair, tile) units of the chunk, block-pair major, are
// split evenly over the grid, so every CTA walks a contiguous run of tiles of
// one or two block pairs (counters flushed with atomics when the pair
// changes) and all SMs finish together.  Tiles arrive by TMA bulk copies
// into a 2-stage ring.
template <int TW, int MINB>
__global__ void __launch_bounds__(kPairThreads, MINB) pair_tri_kernel(const uint32_t* __restrict__ tids, int m,
                                                                   ChunkGeom geom, int64_t t_first, int64_t t_last,
                                                                   int nblk, unsigned long long* __restrict__ tri,
                                                                   const unsigned long long* bn2, int64_t tri_len,
                                                                   const unsigned long long* abort_flag,
                                                                   const int64_t* chunk_ring,
                                                                   const unsigned long long* seq, int ring) {
    // engine use: skip while aborted, or once the pair bucket is mostly gone
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
    constexpr int RW = TW + 4;
    constexpr int RB = RW * 4;
    constexpr uint32_t BLK = kPairBlock * RB;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint8_t* buf = smem + 128;  // [2 stages][A block, B block]

    const int64_t tile_words = (int64_t)m * RW;
    const int64_t nt = t_last - t_first + 1;
    const int64_t U = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const int64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;

    auto issue = [&](int64_t u, int s) {
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        const PairBlock pb = pair_block(bi, nblk, m);
        const uint32_t ab = (uint32_t)pb.na * RB, bb = (uint32_t)pb.nb * RB;
        uint8_t* dst = buf + (size_t)s * 2 * BLK;
        const uint32_t* src = tids + t * tile_words;
        mbar_expect_tx(&bar[s], ab + (pb.diag ? 0u : bb));
        bulk_g2s(dst, src + (int64_t)pb.a0 * RW, ab, &bar[s]);
        if (!pb.diag) bulk_g2s(dst + BLK, src + (int64_t)pb.b0 * RW, bb, &bar[s]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        issue(u0, 0);
        if (u0 + 1 < u1) issue(u0 + 1, 1);
    }
    __syncthreads();

    const int ta = threadIdx.x & 15, tb = threadIdx.x >> 4;
    uint32_t cnt[4][4];
    int64_t cur = -1;
    PairBlock pb{0, 0, 0, 0, true};
    auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int a = pb.a0 + ta + 16 * i, b = pb.b0 + tb + 16 * j;
                if (a < b && b < m && cnt[i][j]) atomicAdd(tri + tri_index(a, b, m), (unsigned long long)cnt[i][j]);
            }
    };

    for (int64_t u = u0; u < u1; ++u) {
        const int s = (int)((u - u0) & 1);
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        if (bi != cur) {
            if (cur >= 0) flush();
            cur = bi;
            pb = pair_block(bi, nblk, m);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) cnt[i][j] = 0;
        }
        mbar_wait(&bar[s], (uint32_t)(((u - u0) >> 1) & 1));
        uint8_t* A = buf + (size_t)s * 2 * BLK;
        uint8_t* B = pb.diag ? A : A + BLK;
        if (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last) {
            // chunk edge inside this tile: zero the rows outside [first, last]
            const int rows = pb.diag ? pb.na : 2 * kPairBlock;
            for (int idx = threadIdx.x; idx < rows * RW; idx += kPairThreads) {
                const int r = idx / RW, slot = idx - r * RW;
                if (slot >= TW || (r < kPairBlock ? r >= pb.na : r - kPairBlock >= pb.nb)) continue;
                uint32_t* w = reinterpret_cast<uint32_t*>(A + (size_t)r * RB) + slot;
                *w &= group_mask(geom, t * TW + slot);
            }
            __syncthreads();
        }
        // two 16-byte chunks (8 words = 256 rows) per step; per pair the 8
        // AND'ed words go through a carry-save tree (7 -> ones/twos/fours,
        // plus one leftover): 4 POPC + 8 LOP3 instead of 8 POPC, which moves
        // the bound from the POPC pipe (16 lanes/SM/clk) to LOP3 (64)
#pragma unroll
        for (int q = 0; q < TW / 4; q += 2) {
            uint4 av0[4], av1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                av0[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + q * 16);
                av1[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + q * 16 + 16);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 bv0 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + q * 16);
                const uint4 bv1 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + q * 16 + 16);
#pragma unroll
                for (int i = 0; i < 4; ++i) cnt[i][j] += and_popc8(av0[i], av1[i], bv0, bv1);
            }
        }
        __syncthreads();  // stage s consumed
        if (threadIdx.x == 0 && u + 2 < u1) {
            fence_proxy_async();
            issue(u + 2, s);
        }
    }
    flush();
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

template <int TW, int MINB>
int pair_launch(const uint32_t* tids, int m, ChunkGeom geom, int64_t t_first, int64_t t_last, int nblk,
                int64_t units, size_t smem, unsigned long long* tri, const unsigned long long* bn2, int64_t tri_len,
                const unsigned long long* abort_flag, const int64_t* chunk_ring, const unsigned long long* seq,
                int ring, cudaStream_t s) {
    int& per_sm = g_pair_slots[(TW == 32 ? 1 : 0) + (MINB == 4 ? 2 : 0)];
    if (per_sm == 0) {
        DIC_CUDA(cudaFuncSetAttribute(pair_tri_kernel<TW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      64 * 1024));
        DIC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pair_tri_kernel<TW, MINB>, kPairThreads, smem));
        per_sm = std::max(per_sm, 1);
    }
    // persistent: one CTA per resident slot (fewer when the chunk is small)
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)per_sm * sm_count()));
    pair_tri_kernel<TW, MINB><<<grid, kPairThreads, smem, s>>>(tids, m, geom, t_first, t_last, nblk, tri, bn2,
                                                                tri_len, abort_flag, chunk_ring, seq, ring);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("pair_tri_kernel");
    return DIC_OK;
}

static int pair_minb() {
    static int v = 0;
    if (!v) {
        const char* e = getenv("DIC_PAIR_MINB");
        v = (e && atoi(e) == 4) ? 4 : 3;
    }
    return v;
}

int count_pairs_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                       unsigned long long* tri, cudaStream_t s, const unsigned long long* bn2 = nullptr,
                       int64_t tri_len = 0, const unsigned long long* abort_flag = nullptr,
                       const int64_t* chunk_ring = nullptr, const unsigned long long* seq = nullptr,
                       int ring = 0) {
    // with a chunk ring, [first, last] only sizes the grid (the largest chunk)
    if (last < first || m < 2) return DIC_OK;
    const int TW = tile_groups(m);
    const ChunkGeom geom = chunk_geom(first, last);
    const int64_t t_first = geom.g_first / TW, t_last = geom.g_last / TW;
    const int64_t nt = t_last - t_first + 1;
    const int nblk = (m + kPairBlock - 1) / kPairBlock;
    const int64_t units = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const size_t smem = 128 + 2 * 2 * (size_t)kPairBlock * row_words(TW) * 4;
    const bool b4 = pair_minb() == 4;
    if (TW == 32)
        return b4 ? pair_launch<32, 4>(tids, m, geom, t_first, t_last, nblk, units, smem, tri, bn2, tri_len, abort_flag,
                                       chunk_ring, seq, ring, s)
                  : pair_launch<32, 3>(tids, m, geom, t_first, t_last, nblk, units, smem, tri, bn2, tri_len, abort_flag,
                                       chunk_ring, seq, ring, s);
    return b4 ? pair_launch<16, 4>(tids, m, geom, t_first, t_last, nblk, units, smem, tri, bn2, tri_len, abort_flag,
                                   chunk_ring, seq, ring, s)
              : pair_launch<16, 3>(tids, m, geom, t_first, t_last, nblk, units, smem, tri, bn2, tri_len, abort_flag,
                                   chunk_ring, seq, ring, s);
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
                           int ring = 0) {
    // tri is all-zero between stops: the gather re-zeroes every entry it reads
    return count_pairs_launch(tids, n, m, first, last, tri, s, bn2, tri_len, abort_flag, chunk_ring, seq, ring);
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
