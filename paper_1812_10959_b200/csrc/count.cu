// count.cu — support counting.
//
//   dic_item_support        first_pass singleton counts (engine.py:132-154)
//   dic_count_support       THE hot kernel: _count_block (engine.py:43-58) for
//                           a whole size-k bucket of dashed candidates over one
//                           chunk, on the bit-sliced layout
//   dic_count_support_rows  the literal (T & I) == I form on the row bitmap
//
// Design.  The reference scans the chunk once PER
// candidate with three NumPy passes.  Here the candidates are stationary
// and the chunk streams past them, like the B operand of a GEMM:
//   * a CTA owns a block of 512*R candidates of one size k (R per thread,
//     their shared-memory row offsets and counters live in registers) and a
//     range of tiles of the chunk;
//   * tiles (TW row-groups x all m items, stored in global memory already in
//     their swizzled shared-memory image) arrive by ONE cp.async.bulk each
//     (TMA engine, mbarrier completion), double-buffered so the next tile
//     lands while the current one is counted;
//   * per 32 rows a candidate costs (k-1) ANDs + 1 POPC (LDS.128 brings 4
//     words of a row; 8 lanes on 8 different items hit 8 bank groups);
//   * one atomic per (candidate, CTA) at the end instead of one per tile.
#include "common.cuh"
#include "async.cuh"

namespace dic {

// ---------------------------------------------------------------------------
// item support (first pass)
// ---------------------------------------------------------------------------
// grid.x = tile splits.  The TW/4 lanes of a group take the 16-byte chunks of
// one item row, so a warp reads 512 contiguous bytes (4 or 8 adjacent item
// rows) per load; a lane sums its chunk over the split's tiles, four tiles in
// flight, and the group's lanes are added up once at the end.
__global__ void __launch_bounds__(256) item_support_kernel(const uint32_t* __restrict__ tids, int m, int TW,
                                                           ChunkGeom geom, int64_t t_first, int64_t t_last,
                                                           unsigned long long* __restrict__ counts) {
    const int64_t nt = t_last - t_first + 1;
    const int64_t ta = t_first + nt * blockIdx.x / gridDim.x;
    const int64_t tb = t_first + nt * (blockIdx.x + 1) / gridDim.x;
    const int RW = row_words(TW), CH = TW / 4;
    const int64_t tw_words = (int64_t)m * RW;
    const int q = threadIdx.x & (CH - 1), per = blockDim.x / CH;
    const unsigned gmask = CH == 8 ? 0xFFu << (threadIdx.x & 24) : 0xFu << (threadIdx.x & 28);
    for (int i0 = 0; i0 < m; i0 += per) {
        const int i = i0 + (int)threadIdx.x / CH;
        const bool live = i < m;
        const uint4* row = reinterpret_cast<const uint4*>(tids + (int64_t)(live ? i : 0) * RW) + q;
        uint32_t acc = 0;  // <= 128 bits per tile: 2^25 tiles before it could wrap (splits hold far fewer)
        unsigned long long total = 0;
        int64_t t = ta;
        for (; t + 4 <= tb; t += 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(row + (t + u) * (tw_words / 4));
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t tt = t + u;
                if ((tt * TW <= geom.g_first) || (tt * TW + TW - 1 >= geom.g_last)) {
                    const int64_t g = tt * TW + (int64_t)(q * 4);
                    v[u].x &= group_mask(geom, g);
                    v[u].y &= group_mask(geom, g + 1);
                    v[u].z &= group_mask(geom, g + 2);
                    v[u].w &= group_mask(geom, g + 3);
                }
                acc += popc4(v[u]);
            }
            if (acc > 0xF0000000u) {
                total += acc;
                acc = 0;
            }
        }
        for (; t < tb; ++t) {
            uint4 v = __ldg(row + t * (tw_words / 4));
            if ((t * TW <= geom.g_first) || (t * TW + TW - 1 >= geom.g_last)) {
                const int64_t g = t * TW + (int64_t)(q * 4);
                v.x &= group_mask(geom, g);
                v.y &= group_mask(geom, g + 1);
                v.z &= group_mask(geom, g + 2);
                v.w &= group_mask(geom, g + 3);
            }
            acc += popc4(v);
        }
        total += acc;
        if (!live) total = 0;
        for (int o = 1; o < CH; o <<= 1) total += __shfl_xor_sync(gmask, total, o);
        if (q == 0 && live && total) atomicAdd(counts + i, total);
    }
}

// ---------------------------------------------------------------------------
// the streaming support count
// ---------------------------------------------------------------------------
// Threads per CTA (one CTA per SM).  TW = 32 tiles (m <= 768): 512 threads x 128
// registers, as many candidates per thread as fit.  TW = 16 tiles (wider
// universes, e.g. cfg4's m = 1000): 1,024 threads x 64 registers — the unit is
// bound by shared-memory load latency, and eight warps per scheduler hide it
// where four did not (ncu: short-scoreboard stalls 5.6 per issue at 512).
#ifndef DIC_TW16_THREADS
#define DIC_TW16_THREADS 512
#endif
__host__ __device__ constexpr int stream_threads(int TW) { return TW == 16 ? DIC_TW16_THREADS : 512; }
constexpr int kMaxBuckets = 16;

struct BucketDesc {
    const uint16_t* items;    // [C][k]
    unsigned long long* out;  // [C], accumulated into
    int64_t C;
    int32_t k;
    int32_t blocks;  // candidate blocks of this bucket (grid.y slices)
};

struct StreamArgs {
    const uint32_t* tids;
    int32_t m, TW;
    uint32_t tile_bytes;
    int64_t t_first, t_last;  // inclusive tile range of the chunk
    int64_t row_splits;
    ChunkGeom geom;
    int32_t nb;
    BucketDesc b[kMaxBuckets];
};

// candidates per thread: as many as the register budget allows for size k
__host__ __device__ constexpr int regs_per_thread(int K) {
    return K == 0 ? 2 : (K <= 2 ? 16 : (K <= 4 ? 8 : (K <= 6 ? 5 : 4)));
}

// Stage tile t into buffer `stage` (thread 0; one bulk async copy).
__device__ __forceinline__ void issue_tile(uint8_t* smem, const uint32_t* tids, uint32_t tb, int64_t t, int stage) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    mbar_expect_tx(&bar[stage], tb);
    bulk_g2s(smem + 128 + (size_t)stage * tb, tids + t * (int64_t)(tb / 4), tb, &bar[stage]);
}

// One work unit: candidates [blk*512*R, +512*R) of a size-k bucket against
// tiles [t0, t1).  All threads enter; the two mbarriers are initialised and
// idle; uses[s] counts the completed phases of barrier s (the wait parity),
// so units can follow each other without re-initialising.
template <int K, int TW>
__device__ __forceinline__ void stream_unit(const uint32_t* __restrict__ tids, int m, uint32_t tb,
                                            const ChunkGeom& geom, const uint16_t* __restrict__ items, int kdyn,
                                            int64_t C, unsigned long long* __restrict__ out, int64_t blk,
                                            int64_t t0, int64_t t1, uint8_t* smem, uint32_t (&uses)[2]) {
    constexpr int R = regs_per_thread(K);
    constexpr int KK = K > 0 ? K : 1;
    constexpr int CH = TW / 4;        // 16-byte chunks per item row
    constexpr int RB = row_words(TW) * 4;  // row stride in bytes
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint8_t* bufs = smem + 128;
    constexpr int NT = stream_threads(TW);
    const int64_t cbase = blk * (int64_t)NT * R;
    const int k = K > 0 ? K : kdyn;

    if (threadIdx.x == 0) {
        fence_proxy_async();  // earlier generic writes (edge masking) before the async refill
        issue_tile(smem, tids, tb, t0, 0);
        if (t0 + 1 < t1) issue_tile(smem, tids, tb, t0 + 1, 1);
    }
    uint32_t off[R][KK];
    uint32_t cnt[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int64_t c = cbase + (int64_t)r * NT + threadIdx.x;
        int64_t cc = c < C ? c : C - 1;
        cnt[r] = 0;
        if constexpr (K > 0) {
#pragma unroll
            for (int j = 0; j < K; ++j) off[r][j] = (uint32_t)__ldg(items + cc * K + j) * RB;
        } else {
            off[r][0] = (uint32_t)cc;
        }
    }

    for (int64_t t = t0; t < t1; ++t) {
        const int s = (int)((t - t0) & 1);
        mbar_wait(&bar[s], uses[s] & 1u);
        ++uses[s];
        uint8_t* base = bufs + (size_t)s * tb;
        // tiles holding a chunk edge: zero the rows outside [first, last]
        if (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last) {
            uint32_t* w = reinterpret_cast<uint32_t*>(base);
            for (int idx = threadIdx.x; idx < m * row_words(TW); idx += NT) {
                int item = idx / row_words(TW), slot = idx - item * row_words(TW);
                if (slot < TW) w[idx] &= group_mask(geom, t * TW + slot);
            }
            __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if constexpr (K > 0) {
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    uint4 v = *reinterpret_cast<const uint4*>(base + off[r][0] + q * 16);
#pragma unroll
                    for (int j = 1; j < K; ++j)
                        v = and4(v, *reinterpret_cast<const uint4*>(base + off[r][j] + q * 16));
                    cnt[r] += popc4(v);
                }
            } else {
                const uint16_t* it = items + (int64_t)off[r][0] * k;
                for (int q = 0; q < CH; ++q) {
                    // the lanes of a warp read different rows: each starts at
                    // another chunk, so they spread over the bank groups
                    const int qq = (q + (int)threadIdx.x) & (CH - 1);
                    uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);
                    for (int j = 0; j < k; ++j) {
                        uint32_t o = (uint32_t)__ldg(it + j) * RB;
                        v = and4(v, *reinterpret_cast<const uint4*>(base + o + qq * 16));
                    }
                    cnt[r] += popc4(v);
                }
            }
        }
        __syncthreads();  // buffer s fully consumed
        if (threadIdx.x == 0 && t + 2 < t1) {
            fence_proxy_async();
            issue_tile(smem, tids, tb, t + 2, s);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int64_t c = cbase + (int64_t)r * NT + threadIdx.x;
        if (c < C && cnt[r]) atomicAdd(out + c, (unsigned long long)cnt[r]);
    }
}

#ifdef DIC_LAB_TIMING
// per-CTA phase stamps for tools/lab (globaltimer ns): start, ids loaded,
// first tile landed, tiles done, end
__device__ unsigned long long g_lab_stamp[4096][6];
__device__ __forceinline__ void lab_stamp(int i) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_lab_stamp[(blockIdx.y * gridDim.x + blockIdx.x) & 4095][i] = t;
    }
}
#else
__device__ __forceinline__ void lab_stamp(int) {}
#endif

// carry-save popcount of 4 words: 3 POPC + 2 LOP3 instead of 4 POPC (the
// POPC pipe runs at a quarter of the LOP3 rate and binds for k = 2; cfg5
// k = 2 bucket: 4.2 -> 3.8 ms in tools/lab/count_ab.py)
__device__ __forceinline__ uint32_t popc4_csa(uint4 v) {
    const uint32_t s = lop3_xor3(v.x, v.y, v.z), c = lop3_maj(v.x, v.y, v.z);
    return __popc(s) + __popc(v.w) + 2u * __popc(c);
}

// Row-lane variant: SUB = TW/4 lanes share a candidate, lane `sub` reading
// 16-byte chunk `sub` of each item row, so SUB adjacent lanes always read one
// contiguous row (128 B at TW = 32, 64 B at TW = 16): conflict-free or nearly
// so whatever the items are (random candidates, e.g. cfg5), where one
// candidate per lane scatters 32 rows over the banks.  Item ids stay packed
// two per register (the row offset is one IMAD away) so a CTA still holds
// rl_slots x R candidates; each lane's partial count is reduced over its SUB
// lanes once per unit.
__host__ __device__ constexpr int rl_regs(int K, int TW) {
    return TW == 32 ? (K <= 4 ? 32 : (K == 5 ? 20 : (K == 6 ? 24 : 12)))   // cfg5-shaped (m <= 768)
           : DIC_TW16_THREADS == 1024 ? (K <= 2 ? 16 : (K <= 4 ? 12 : (K <= 6 ? 8 : 4)))  // cfg4's m = 1000 stops
                                      : (K <= 2 ? 32 : (K <= 4 ? 28 : (K <= 6 ? 20 : 12)));
}
// (tuned per size on cfg5 with tools/lab/count_ab.sh; register allocation
// across the per-size instantiations does not make this monotone)
static_assert(rl_regs(1, 32) % 4 == 0 && rl_regs(5, 32) % 4 == 0 && rl_regs(6, 32) % 4 == 0 &&
                  rl_regs(7, 32) % 4 == 0 && rl_regs(3, 16) % 4 == 0 && rl_regs(5, 16) % 4 == 0 &&
                  rl_regs(7, 16) % 4 == 0,
              "row-lane id spans are loaded 8 bytes at a time");
__host__ __device__ constexpr int rl_slots(int TW) { return stream_threads(TW) / (TW / 4); }  // candidate slots per CTA

template <int K, int TW>
__device__ __forceinline__ void stream_unit_rl(const uint32_t* __restrict__ tids, int m, uint32_t tb,
                                               const ChunkGeom& geom, const uint16_t* __restrict__ items, int64_t C,
                                               unsigned long long* __restrict__ out, int64_t blk, int64_t t0,
                                               int64_t t1, uint8_t* smem, uint32_t (&uses)[2]) {
    constexpr int RB = row_words(TW) * 4, R = rl_regs(K, TW), KP = (K + 1) / 2, SUB = TW / 4;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint8_t* bufs = smem + 128;
    const int sub = threadIdx.x & (SUB - 1), slot = threadIdx.x / SUB;
    // a thread owns R CONSECUTIVE candidates: in a sorted bucket they mostly
    // share their first item, whose chunk is then loaded once per tile
    // the bucket's blocks hold equal shares (not full blocks plus a short
    // tail): every CTA of a row split then finishes at the same time
    const int64_t cap = (int64_t)rl_slots(TW) * R;
    const int64_t nblk = (C + cap - 1) / cap;
    // shares rounded to 4 candidates keep every thread's id span 8-byte aligned
    const int64_t per = ((C + nblk - 1) / nblk + 3) & ~int64_t(3);
    const int64_t bend = min(C, (blk + 1) * per);  // this block's candidates: [blk * per, bend)
    const int64_t cbase = blk * per + (int64_t)slot * R;
    // slots past the share re-count the block's last candidate (all lanes of
    // such a warp read the same rows: broadcasts) and add nothing
    // a warp whose slots all lie past the share only keeps the barriers
    const bool warp_live = __any_sync(0xFFFFFFFFu, cbase < bend);
    lab_stamp(0);
    if (threadIdx.x == 0) {
        fence_proxy_async();
        issue_tile(smem, tids, tb, t0, 0);
        if (t0 + 1 < t1) issue_tile(smem, tids, tb, t0 + 1, 1);
    }
    uint32_t it[R][KP];
    uint32_t cnt[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cnt[r] = 0;
    if (cbase + R <= bend && ((reinterpret_cast<uintptr_t>(items + cbase * K) & 7u) == 0)) {
        // the thread's R x K ids are one contiguous, 8-byte aligned span
        // (R is a multiple of 4): R*K/4 8-byte loads instead of R*K 2-byte
        // ones, which dominated the unit's prologue (~2.7 us at R*K = 72)
        uint32_t w[R * K / 2];
        const uint2* src = reinterpret_cast<const uint2*>(items + cbase * K);
#pragma unroll
        for (int q = 0; q < R * K / 4; ++q) {
            const uint2 v = __ldg(src + q);
            w[2 * q] = v.x;
            w[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int j = 0; j < KP; ++j) {
                const int p = r * K + 2 * j;  // item p and p + 1 of the span
                const uint32_t lo = (w[p >> 1] >> ((p & 1) * 16)) & 0xFFFFu;
                const uint32_t hi = (2 * j + 1 < K) ? (w[(p + 1) >> 1] >> (((p + 1) & 1) * 16)) & 0xFFFFu : 0u;
                it[r][j] = lo | (hi << 16);
            }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t c = cbase + r;
            const int64_t cc = c < bend ? c : bend - 1;
#pragma unroll
            for (int j = 0; j < KP; ++j) {
                uint32_t lo = __ldg(items + cc * K + 2 * j);
                uint32_t hi = (2 * j + 1 < K) ? (uint32_t)__ldg(items + cc * K + 2 * j + 1) : 0u;
                it[r][j] = lo | (hi << 16);
            }
        }
    }
    lab_stamp(1);
    for (int64_t t = t0; t < t1; ++t) {
        const int s = (int)((t - t0) & 1);
        mbar_wait(&bar[s], uses[s] & 1u);
        ++uses[s];
        if (t == t0) lab_stamp(2);
        uint8_t* base = bufs + (size_t)s * tb;
        if (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last) {
            uint32_t* w = reinterpret_cast<uint32_t*>(base);
            for (int idx = threadIdx.x; idx < m * row_words(TW); idx += stream_threads(TW)) {
                int item = idx / row_words(TW), sl = idx - item * row_words(TW);
                if (sl < TW) w[idx] &= group_mask(geom, t * TW + sl);
            }
            __syncthreads();
        }
        const uint8_t* bs = base + sub * 16;
        // the row stride as an opaque value: item * stride stays an IMAD (the
        // FMA pipe, idle here) instead of becoming a shift on the ALU pipe the
        // ANDs saturate (the stride is a power of two since the rows are dense)
        uint32_t rbv = RB;
        asm volatile("" : "+r"(rbv));
        // keep the row offsets derived per tile (one IMAD each) instead of
        // letting the compiler hoist R*K of them into registers
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int j = 0; j < KP; ++j) asm volatile("" : "+r"(it[r][j]));
        uint32_t prev0 = 0xFFFFFFFFu;
        uint4 v0 = make_uint4(0u, 0u, 0u, 0u);
        if (warp_live)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t i0 = it[r][0] & 0xFFFFu;
            if (i0 != prev0) {
                v0 = *reinterpret_cast<const uint4*>(bs + i0 * rbv);
                prev0 = i0;
            }
            uint4 v = v0;
#pragma unroll
            for (int j = 1; j < K; ++j) {
                const uint32_t item = (j & 1) ? (it[r][j >> 1] >> 16) : (it[r][j >> 1] & 0xFFFFu);
                v = and4(v, *reinterpret_cast<const uint4*>(bs + item * rbv));
            }
            cnt[r] += K <= 4 ? popc4_csa(v) : popc4(v);  // sizes 5+: shared memory binds, not POPC
        }
        __syncthreads();
        if (threadIdx.x == 0 && t + 2 < t1) {
            fence_proxy_async();
            issue_tile(smem, tids, tb, t + 2, s);
        }
    }
    lab_stamp(3);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        uint32_t x = cnt[r];
#pragma unroll
        for (int o = 1; o < SUB; o <<= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        const int64_t c = cbase + r;
        if (sub == 0 && c < bend && x) atomicAdd(out + c, (unsigned long long)x);
    }
    lab_stamp(4);
}

template <int TW>
__device__ __forceinline__ void dispatch_unit_rl(int k, const uint32_t* tids, int m, uint32_t tb,
                                                 const ChunkGeom& geom, const uint16_t* items, int64_t C,
                                                 unsigned long long* out, int64_t blk, int64_t t0, int64_t t1,
                                                 uint8_t* smem, uint32_t (&uses)[2]) {
    switch (k) {
        case 1: stream_unit_rl<1, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        case 2: stream_unit_rl<2, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        case 3: stream_unit_rl<3, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        case 4: stream_unit_rl<4, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        case 5: stream_unit_rl<5, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        case 6: stream_unit_rl<6, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        case 7: stream_unit_rl<7, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
        default: stream_unit_rl<8, TW>(tids, m, tb, geom, items, C, out, blk, t0, t1, smem, uses); break;
    }
}

// candidates per block of the unit kind used for (TW, k)
__host__ __device__ inline int64_t cands_per_block(int TW, int k) {
    if (k <= 8) return (int64_t)rl_slots(TW) * rl_regs(k, TW);
    return (int64_t)stream_threads(TW) * regs_per_thread(0);
}

// itemsets of more than 8 items: one candidate per thread, ids read per use
template <int TW>
__device__ __forceinline__ void dispatch_unit(int k, const uint32_t* tids, int m, uint32_t tb, const ChunkGeom& geom,
                                              const uint16_t* items, int64_t C, unsigned long long* out,
                                              int64_t blk, int64_t t0, int64_t t1, uint8_t* smem,
                                              uint32_t (&uses)[2]) {
    stream_unit<0, TW>(tids, m, tb, geom, items, k, C, out, blk, t0, t1, smem, uses);
}

__device__ __forceinline__ void init_barriers(uint8_t* smem) {
    if (threadIdx.x == 0) {
        uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
}

// Host-sized launch (the dic_count_support API): grid = (row splits, blocks).
template <int TW>
__global__ void __launch_bounds__(stream_threads(TW), 1) count_stream_kernel(const __grid_constant__ StreamArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    int64_t blk = blockIdx.y;
    int j = 0;
    while (j + 1 < a.nb && blk >= a.b[j].blocks) {
        blk -= a.b[j].blocks;
        ++j;
    }
    const BucketDesc& B = a.b[j];
    const int64_t nt = a.t_last - a.t_first + 1;
    const int64_t t0 = a.t_first + nt * blockIdx.x / a.row_splits;
    const int64_t t1 = a.t_first + nt * (blockIdx.x + 1) / a.row_splits;
    if (t0 >= t1) return;
    init_barriers(smem);
    uint32_t uses[2] = {0u, 0u};
    if (B.k <= 8)
        dispatch_unit_rl<TW>(B.k, a.tids, a.m, a.tile_bytes, a.geom, B.items, B.C, B.out, blk, t0, t1, smem, uses);
    else
        dispatch_unit<TW>(B.k, a.tids, a.m, a.tile_bytes, a.geom, B.items, B.C, B.out, blk, t0, t1, smem, uses);
}

// Device-sized launch (the engine's per-stop count): bucket sizes, delta
// offsets and the dense-pair switch are read from device memory, so the
// host can enqueue stops without knowing the sizes.  A persistent grid walks
// the (candidate block, row split) units of every bucket.
constexpr int kDevMaxK = 64;
struct DevCountArgs {
    const uint32_t* tids;
    int32_t m, TW;
    uint32_t tile_bytes;
    int64_t t_first, t_last;
    ChunkGeom geom;
    int32_t kuse;                     // buckets 1..kuse-1 may be non-empty
    uint16_t* const* items_tab;       // per-size item arrays
    const unsigned long long* bn;     // per-size bucket fill
    const int64_t* doff;              // per-size delta offsets
    unsigned long long* delta;
    const unsigned long long* abort;  // non-zero: stop skipped (overflow recovery)
    int64_t tri_len;                  // > 0: bucket 2 counted densely when 2*bn[2] >= tri_len
    // engine graphs: the stop's local chunk [first, last] is read from
    // chunk_ring[2 * (*seq % ring)] at run time (geom/t_first/t_last unused)
    const int64_t* chunk_ring;
    const unsigned long long* seq;
    int32_t ring;
    int64_t small_max;  // at most this many sparse candidates: the unstaged path
    // batch of quiet stops (engine): the next `batch` chunks of the stop
    // counter are counted in one launch, chunk b into delta + b * batch_stride
    // (refused — nothing counted — unless the live slots fit a block and no
    // bucket is dense: the batch checkpoint kernel applies the same test)
    int32_t batch;
    int64_t batch_stride;
};

constexpr int kCountBatchMax = 8;

// The chunk geometry of this launch (host-given, or read from the ring).
__device__ __forceinline__ bool dev_chunk(const DevCountArgs& a, ChunkGeom& geom, int64_t& t_first,
                                          int64_t& t_last) {
    geom = a.geom;
    t_first = a.t_first;
    t_last = a.t_last;
    if (a.chunk_ring) {
        const int64_t sl = (int64_t)(*a.seq % (unsigned long long)a.ring);
        const int64_t f = a.chunk_ring[2 * sl], l = a.chunk_ring[2 * sl + 1];
        if (l < f) return false;
        geom = chunk_geom(f, l);
        t_first = geom.g_first / a.TW;
        t_last = geom.g_last / a.TW;
    }
    return true;
}

// Few candidates: staging whole tiles (all m item rows) costs more than the
// count.  SUB = TW/4 lanes per (candidate, tile range) load the candidate's
// item rows of each tile straight from global memory (16 B per lane, one
// contiguous row segment per lane group; the chunk is L2-resident), AND them,
// and popcount; partial counts are reduced over the group once.
template <int TW>
__device__ __forceinline__ void count_dev_small(const DevCountArgs& a, const ChunkGeom* geoms, int nb,
                                                int64_t nt_max, const int64_t* cpref, int kuse) {
    constexpr int SUB = TW / 4, RW = row_words(TW);
    const int64_t tile_words = (int64_t)a.m * RW;
    const int lane = threadIdx.x & 31, sub = lane & (SUB - 1);
    const unsigned gmask = ((1u << SUB) - 1u) << (lane & ~(SUB - 1));
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / SUB;
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / SUB;
    const int64_t Ctot = cpref[kuse];
    // work item = (chunk b, candidate, row split): every chunk of a batch in one pass
    const int64_t rs =
        std::max<int64_t>(1, std::min<int64_t>(nt_max, ngroups / std::max<int64_t>(Ctot * nb, 1)));
    const int64_t W = Ctot * rs * nb;
    for (int64_t w = gid; w < W; w += ngroups) {
        const int64_t b = w / (Ctot * rs), w1 = w - b * Ctot * rs;
        const int64_t cg = w1 / rs, r = w1 - cg * rs;
        const ChunkGeom geom = geoms[b];
        if (geom.g_last < geom.g_first) continue;  // (an empty chunk)
        const int64_t t_first = geom.g_first / TW, nt = geom.g_last / TW - t_first + 1;
        int k = 1;
        while (cpref[k + 1] <= cg) ++k;
        const int64_t c = cg - cpref[k];
        const uint16_t* it = a.items_tab[k] + c * k;
        const int64_t t0 = t_first + nt * r / rs, t1 = t_first + nt * (r + 1) / rs;
        uint32_t cnt = 0;
        // four tiles per round: the item rows of all four are requested before
        // any is used (the loop is bound by L2 latency, not by its few ANDs)
        for (int64_t t = t0; t < t1; t += 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
            for (int j = 0; j < k; ++j) {
                const int64_t row = (int64_t)__ldg(it + j) * RW + sub * 4;
                uint4 x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    x[u] = t + u < t1 ? __ldg(reinterpret_cast<const uint4*>(a.tids + (t + u) * tile_words + row))
                                      : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = and4(v[u], x[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t tt = t + u;
                if (tt < t1 && (tt * TW <= geom.g_first || tt * TW + TW - 1 >= geom.g_last)) {
                    const int64_t g = tt * TW + sub * 4;
                    v[u].x &= group_mask(geom, g);
                    v[u].y &= group_mask(geom, g + 1);
                    v[u].z &= group_mask(geom, g + 2);
                    v[u].w &= group_mask(geom, g + 3);
                }
                cnt += popc4(v[u]);
            }
        }
#pragma unroll
        for (int o = 1; o < SUB; o <<= 1) cnt += __shfl_xor_sync(gmask, cnt, o);
        if (sub == 0 && cnt)
            atomicAdd(a.delta + b * a.batch_stride + a.doff[k] + c, (unsigned long long)cnt);
    }
}

template <int TW>
__global__ void __launch_bounds__(stream_threads(TW), 1) count_dev_kernel(const __grid_constant__ DevCountArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int64_t upref[kDevMaxK + 1];  // units before bucket k
    __shared__ int64_t cpref[kDevMaxK + 1];  // candidates before bucket k
    __shared__ int32_t srs[kDevMaxK];        // row splits of bucket k's blocks
    __shared__ ChunkGeom sgeom[kCountBatchMax];
    if (*a.abort) return;
    ChunkGeom geom;
    int64_t t_first, t_last;
    if (a.batch > 1) {
        // a batch of stops: chunk b is the schedule slot of stop counter + b
        if (a.doff[a.kuse] > a.batch_stride) return;
        if ((int)threadIdx.x < a.batch) {
            const int64_t sl = (int64_t)((*a.seq + threadIdx.x) % (unsigned long long)a.ring);
            const int64_t f = a.chunk_ring[2 * sl], l = a.chunk_ring[2 * sl + 1];
            ChunkGeom g = chunk_geom(0, 0);
            g.g_first = 1;
            g.g_last = 0;  // empty
            if (l >= f) g = chunk_geom(f, l);
            sgeom[threadIdx.x] = g;
        }
        geom = chunk_geom(0, 0);
        t_first = t_last = 0;
    } else if (!dev_chunk(a, geom, t_first, t_last)) {
        return;
    }
    const int64_t nt = t_last - t_first + 1;
    // bucket fills loaded in parallel (a loop of dependent-latency loads in
    // one thread would cost one L2 round trip per size)
    if (threadIdx.x < a.kuse) cpref[threadIdx.x + 1] = (int64_t)a.bn[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool dense = a.tri_len > 0 && 2 * cpref[3] >= a.tri_len;
        // Row splits per bucket, weighted by what a block costs per tile: the
        // tile's arrival is a floor (1.6 us with every SM streaming: tools/lab/
        // count_fill.py), a full block's AND/POPC work takes 3.7 us and hides
        // it.  A bucket holding a few hundred candidates then takes fewer CTAs
        // with longer tile ranges instead of as many CTAs as a full block,
        // which stretched every other block's range (cfg4's middle stops hold
        // ~9k 3-item and a few hundred 4-item candidates).
        constexpr float kFloor = 0.45f;
        float wsum = 0.f;
        int64_t cacc = 0, nblocks = 0;
        cpref[0] = 0;
        for (int k = 1; k < a.kuse; ++k) {
            int64_t C = cpref[k + 1];
            if (k == 2 && dense) C = 0;
            const int64_t per = cands_per_block(TW, k);
            const int64_t nb = (C + per - 1) / per;
            cpref[k] = cacc;
            cacc += C;
            nblocks += nb;
            upref[k] = nb;  // (blocks, for now)
            if (nb) wsum += (float)nb * fmaxf(kFloor, (float)C / (float)(nb * per));
        }
        cpref[a.kuse] = cacc;
        int64_t uacc = 0;
        for (int k = 1; k < a.kuse; ++k) {
            const int64_t nb = upref[k];
            int64_t rs = 1;
            if (nb && nblocks < (int64_t)gridDim.x) {
                const int64_t C = cpref[k + 1] - cpref[k];
                const float w = fmaxf(kFloor, (float)C / (float)(nb * cands_per_block(TW, k)));
                rs = (int64_t)((float)gridDim.x * w / wsum);
#ifdef DIC_COUNT_UNIFORM_SPLITS
                rs = (int64_t)gridDim.x / nblocks;
#endif
                rs = max((int64_t)1, min(rs, nt));
            }
            srs[k] = (int32_t)rs;
            upref[k] = uacc;
            uacc += nb * rs;
        }
        upref[a.kuse] = uacc;
        upref[0] = 0;
    }
    __syncthreads();
    const int64_t U = upref[a.kuse];
    if (U == 0) return;
    if (a.batch > 1) {
        // (the engine batches stops only after the pair bucket left its dense phase for good)
        int64_t nt_max = 1;
        for (int b = 0; b < a.batch; ++b)
            nt_max = max(nt_max, sgeom[b].g_last / TW - sgeom[b].g_first / TW + 1);
        count_dev_small<TW>(a, sgeom, a.batch, nt_max, cpref, a.kuse);
        return;
    }
    if (cpref[a.kuse] <= a.small_max) {
        sgeom[0] = geom;
        __syncthreads();
        count_dev_small<TW>(a, sgeom, 1, nt, cpref, a.kuse);
        return;
    }
    if ((int64_t)blockIdx.x >= U) return;
    init_barriers(smem);
    uint32_t uses[2] = {0u, 0u};
    for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
        int k = 1;
        while (upref[k + 1] <= u) ++k;
        const int64_t rs = srs[k];
        const int64_t gb = (u - upref[k]) / rs, r = (u - upref[k]) - gb * rs;
        const int64_t t0 = t_first + nt * r / rs, t1 = t_first + nt * (r + 1) / rs;
        if (t0 < t1) {
            if (k <= 8)
                dispatch_unit_rl<TW>(k, a.tids, a.m, a.tile_bytes, geom, a.items_tab[k], (int64_t)a.bn[k],
                                     a.delta + a.doff[k], gb, t0, t1, smem, uses);
            else
                dispatch_unit<TW>(k, a.tids, a.m, a.tile_bytes, geom, a.items_tab[k], (int64_t)a.bn[k],
                                  a.delta + a.doff[k], gb, t0, t1, smem, uses);
        }
        __syncthreads();
    }
}

// Universes too wide to double-buffer a tile (m > 1536): plain loads of the
// same layout through L1/L2.  Work item = (candidate, tile).
__global__ void __launch_bounds__(256) count_global_kernel(const uint32_t* __restrict__ tids, int m, int TW,
                                                           ChunkGeom geom, int64_t t_first, int64_t nt,
                                                           const uint16_t* __restrict__ items, int k, int64_t C,
                                                           unsigned long long* __restrict__ out) {
    const int64_t total = C * nt;
    const int RW = row_words(TW);
    const int64_t tw_words = (int64_t)m * RW;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = w / nt, t = t_first + (w - c * nt);
        const uint16_t* it = items + c * (int64_t)k;
        uint32_t cnt = 0;
        for (int q = 0; q < TW / 4; ++q) {
            int64_t g = t * TW + q * 4;
            if (g > geom.g_last || g + 3 < geom.g_first) continue;
            uint4 v = make_uint4(group_mask(geom, g), group_mask(geom, g + 1), group_mask(geom, g + 2),
                                 group_mask(geom, g + 3));
            for (int j = 0; j < k; ++j) {
                uint32_t item = __ldg(it + j);
                const uint4* row = reinterpret_cast<const uint4*>(tids + t * tw_words + (int64_t)item * RW);
                v = and4(v, __ldg(row + q));
            }
            cnt += popc4(v);
        }
        if (cnt) atomicAdd(out + c, (unsigned long long)cnt);
    }
}

// Device-sized fallback for universes too wide to stage (and for > 64
// itemset sizes): grid-stride over (bucket, candidate, tile) with plain loads.
__global__ void __launch_bounds__(256) count_dev_global_kernel(const __grid_constant__ DevCountArgs a) {
    if (*a.abort) return;
    ChunkGeom geom;
    int64_t t_first, t_last;
    if (!dev_chunk(a, geom, t_first, t_last)) return;
    const bool dense = a.tri_len > 0 && 2 * (int64_t)a.bn[2] >= a.tri_len;
    const int TW = a.TW, RW = row_words(TW);
    const int64_t nt = t_last - t_first + 1;
    const int64_t tw_words = (int64_t)a.m * RW;
    for (int k = 1; k < a.kuse; ++k) {
        const int64_t C = (k == 2 && dense) ? 0 : (int64_t)a.bn[k];
        const uint16_t* items = a.items_tab[k];
        unsigned long long* out = a.delta + a.doff[k];
        for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < C * nt;
             w += (int64_t)gridDim.x * blockDim.x) {
            const int64_t c = w / nt, t = t_first + (w - c * nt);
            uint32_t cnt = 0;
            for (int q = 0; q < TW / 4; ++q) {
                const int64_t g = t * TW + q * 4;
                if (g > geom.g_last || g + 3 < geom.g_first) continue;
                uint4 v = make_uint4(group_mask(geom, g), group_mask(geom, g + 1), group_mask(geom, g + 2),
                                     group_mask(geom, g + 3));
                for (int j = 0; j < k; ++j) {
                    const uint32_t item = __ldg(items + c * k + j);
                    const uint4* row = reinterpret_cast<const uint4*>(a.tids + t * tw_words + (int64_t)item * RW);
                    v = and4(v, __ldg(row + q));
                }
                cnt += popc4(v);
            }
            if (cnt) atomicAdd(out + c, (unsigned long long)cnt);
        }
    }
}

static int g_max_smem = -1;
static int max_dyn_smem() {
    if (g_max_smem < 0) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        g_max_smem = v > 0 ? v : 48 * 1024;
    }
    return g_max_smem;
}

struct BucketIn {
    const uint16_t* items;
    unsigned long long* out;
    int64_t C;
    int k;
};

// Count every bucket over rows [first, last] in as few launches as possible.
int count_buckets_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                         const BucketIn* bk, int nbk, cudaStream_t s) {
    if (last < first) return DIC_OK;
    const int TW = tile_groups(m);
    const ChunkGeom geom = chunk_geom(first, last);
    const int64_t t_first = geom.g_first / TW, t_last = geom.g_last / TW;
    const int64_t nt = t_last - t_first + 1;
    const size_t tile_bytes = (size_t)m * row_words(TW) * 4;
    const size_t smem = 128 + 2 * tile_bytes;
    if (smem > (size_t)max_dyn_smem()) {
        for (int i = 0; i < nbk; ++i) {
            if (bk[i].C <= 0) continue;
            int64_t total = bk[i].C * nt;
            int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
            count_global_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
                tids, m, TW, geom, t_first, nt, bk[i].items, bk[i].k, bk[i].C, bk[i].out); ::dic::note_launch();
            DIC_CHECK_LAUNCH("count_global_kernel");
        }
        return DIC_OK;
    }
    static bool attr32 = false, attr16 = false;
    if (TW == 32 && !attr32) {
        DIC_CUDA(cudaFuncSetAttribute(count_stream_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_dyn_smem()));
        attr32 = true;
    }
    if (TW == 16 && !attr16) {
        DIC_CUDA(cudaFuncSetAttribute(count_stream_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_dyn_smem()));
        attr16 = true;
    }
    int i = 0;
    while (i < nbk) {
        StreamArgs a;
        memset(&a, 0, sizeof(a));
        a.tids = tids;
        a.m = m;
        a.TW = TW;
        a.tile_bytes = (uint32_t)tile_bytes;
        a.t_first = t_first;
        a.t_last = t_last;
        a.geom = geom;
        int64_t blocks = 0;
        for (; i < nbk && a.nb < kMaxBuckets; ++i) {
            if (bk[i].C <= 0) continue;
            const int64_t per = cands_per_block(TW, bk[i].k);
            BucketDesc& d = a.b[a.nb++];
            d.items = bk[i].items;
            d.out = bk[i].out;
            d.C = bk[i].C;
            d.k = bk[i].k;
            d.blocks = (int32_t)((bk[i].C + per - 1) / per);
            blocks += d.blocks;
        }
        if (a.nb == 0) break;
        DIC_REQUIRE(blocks <= 65535, "count: %lld candidate blocks exceed one launch", (long long)blocks);
        // about two CTAs per SM in total: one resident, one to balance the tail
        // one CTA per SM (512 threads x 128 registers fill the register
        // file): size the grid to one full wave when the blocks allow it
        const int64_t target = sm_count();
        int64_t rs = blocks >= target ? 1 : target / blocks;
        rs = std::max<int64_t>(1, std::min<int64_t>(rs, nt));
        a.row_splits = rs;
        dim3 grid((unsigned)rs, (unsigned)blocks);
        if (TW == 32)
            count_stream_kernel<32><<<grid, stream_threads(32), smem, s>>>(a);
        else
            count_stream_kernel<16><<<grid, stream_threads(16), smem, s>>>(a);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("count_stream_kernel");
    }
    return DIC_OK;
}

// The engine's per-stop count: device-sized, no host knowledge of bucket sizes.
int count_dev_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last, int kuse,
                     uint16_t* const* items_tab, const unsigned long long* bn, const int64_t* doff,
                     unsigned long long* delta, const unsigned long long* abort_flag, int64_t tri_len,
                     cudaStream_t s, const int64_t* chunk_ring = nullptr, const unsigned long long* seq = nullptr,
                     int ring = 0, int batch = 1, int64_t batch_stride = 0) {
    if (!chunk_ring && last < first) return DIC_OK;
    DIC_REQUIRE(batch >= 1 && batch <= kCountBatchMax && (batch == 1 || (chunk_ring && batch_stride > 0)),
                "count_dev_launch: bad batch");
    DevCountArgs a;
    memset(&a, 0, sizeof(a));
    a.tids = tids;
    a.m = m;
    a.TW = tile_groups(m);
    a.tile_bytes = (uint32_t)((size_t)m * row_words(a.TW) * 4);
    a.geom = chunk_geom(first, last);
    a.t_first = a.geom.g_first / a.TW;
    a.t_last = a.geom.g_last / a.TW;
    a.kuse = kuse;
    a.items_tab = items_tab;
    a.bn = bn;
    a.doff = doff;
    a.delta = delta;
    a.abort = abort_flag;
    a.tri_len = tri_len;
    a.chunk_ring = chunk_ring;
    a.seq = seq;
    a.ring = ring;
    a.batch = batch;
    a.batch_stride = batch_stride;
    static int64_t small_max = -1;
    if (small_max < 0) {
        const char* e = getenv("DIC_COUNT_SMALL_MAX");
        small_max = e ? atoll(e) : 2048;  // measured crossover on cfg4
    }
    a.small_max = small_max;
    const size_t smem = 128 + 2 * (size_t)a.tile_bytes;
    // the kernel's static shared memory (the unit prefix table) shares the budget
    static size_t static_smem = 0;
    if (!static_smem) {
        cudaFuncAttributes fa32, fa16;
        DIC_CUDA(cudaFuncGetAttributes(&fa32, count_dev_kernel<32>));
        DIC_CUDA(cudaFuncGetAttributes(&fa16, count_dev_kernel<16>));
        static_smem = std::max(fa32.sharedSizeBytes, fa16.sharedSizeBytes) + 16;
    }
    if (smem + static_smem > (size_t)max_dyn_smem() || kuse > kDevMaxK) {
        count_dev_global_kernel<<<sm_count() * 8, 256, 0, s>>>(a);
        ::dic::note_launch();
        DIC_CHECK_LAUNCH("count_dev_global_kernel");
        return DIC_OK;
    }
    static bool attr32 = false, attr16 = false;
    if (a.TW == 32 && !attr32) {
        DIC_CUDA(cudaFuncSetAttribute(count_dev_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_dyn_smem() - (int)static_smem));
        attr32 = true;
    }
    if (a.TW == 16 && !attr16) {
        DIC_CUDA(cudaFuncSetAttribute(count_dev_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_dyn_smem() - (int)static_smem));
        attr16 = true;
    }
    if (a.TW == 32)
        count_dev_kernel<32><<<sm_count(), stream_threads(32), smem, s>>>(a);
    else
        count_dev_kernel<16><<<sm_count(), stream_threads(16), smem, s>>>(a);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("count_dev_kernel");
    return DIC_OK;
}

int item_support_launch(const uint32_t* tids, int64_t n, int m, int64_t first, int64_t last,
                        unsigned long long* counts, cudaStream_t s) {
    if (last < first) return DIC_OK;
    const int TW = tile_groups(m);
    ChunkGeom geom = chunk_geom(first, last);
    const int64_t t_first = geom.g_first / TW, t_last = geom.g_last / TW;
    const int64_t nt = t_last - t_first + 1;
    int64_t splits = std::min<int64_t>(nt, (int64_t)sm_count() * 8);
    item_support_kernel<<<(unsigned)std::max<int64_t>(splits, 1), 256, 0, s>>>(tids, m, TW, geom, t_first, t_last,
                                                                             counts); ::dic::note_launch();
    DIC_CHECK_LAUNCH("item_support_kernel");
    return DIC_OK;
}

// ---------------------------------------------------------------------------
// row-form count: (T & I) == I on the row bitmap
// ---------------------------------------------------------------------------
// grid = (row tiles of 256 rows, candidate blocks of kRowCands).  A thread
// owns one row held in registers (W words); candidate masks are staged in
// shared memory and read as warp-uniform broadcasts; per candidate the warp
// ballots its 32 row tests and lane 0 accumulates the popcount.
constexpr int kRowCands = 64;

template <int W>
__global__ void __launch_bounds__(256) count_rows_kernel(
    const unsigned long long* __restrict__ rows, int Wd, int64_t first, int64_t last,
    const unsigned long long* __restrict__ masks, int64_t C, unsigned long long* __restrict__ out) {
    constexpr int WS = W > 0 ? W : 1;
    extern __shared__ unsigned long long sm_masks[];  // [kRowCands][Wr]
    __shared__ uint32_t sm_cnt[kRowCands];
    const int Wr = W > 0 ? W : Wd;
    const int64_t c0 = (int64_t)blockIdx.y * kRowCands;
    const int nc = (int)(C - c0 < (int64_t)kRowCands ? C - c0 : (int64_t)kRowCands);
    for (int i = threadIdx.x; i < nc * Wr; i += blockDim.x) sm_masks[i] = masks[c0 * Wr + i];
    for (int i = threadIdx.x; i < kRowCands; i += blockDim.x) sm_cnt[i] = 0;
    __syncthreads();
    const int64_t r = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = r <= last;
    const int lane = threadIdx.x & 31;
    if constexpr (W > 0) {
        unsigned long long t[WS];
#pragma unroll
        for (int w = 0; w < W; ++w) t[w] = valid ? __ldg(rows + r * W + w) : 0ull;
        for (int c = 0; c < nc; ++c) {
            unsigned long long acc = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) acc |= sm_masks[c * W + w] & ~t[w];
            uint32_t b = __ballot_sync(0xFFFFFFFFu, valid && acc == 0ull);
            if (lane == 0 && b) atomicAdd(&sm_cnt[c], (uint32_t)__popc(b));
        }
    } else {
        for (int c = 0; c < nc; ++c) {
            unsigned long long acc = 0;
            if (valid)
                for (int w = 0; w < Wr; ++w) acc |= sm_masks[c * Wr + w] & ~__ldg(rows + r * Wr + w);
            uint32_t b = __ballot_sync(0xFFFFFFFFu, valid && acc == 0ull);
            if (lane == 0 && b) atomicAdd(&sm_cnt[c], (uint32_t)__popc(b));
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += blockDim.x)
        if (sm_cnt[c]) atomicAdd(out + c0 + c, (unsigned long long)sm_cnt[c]);
}

template <int W>
static void launch_rows(dim3 grid, const unsigned long long* rows, int Wd, int64_t first, int64_t last,
                        const unsigned long long* masks, int64_t C, unsigned long long* out, cudaStream_t s) {
    count_rows_kernel<W><<<grid, 256, (size_t)kRowCands * Wd * 8, s>>>(rows, Wd, first, last, masks, C, out);
    ::dic::note_launch();
}

}  // namespace dic

using namespace dic;

extern "C" int64_t dic_tids_words(int64_t n, int32_t m) {
    if (n < 1 || m < 1) return 0;
    return tile_count(n, m) * tile_words(m);
}

extern "C" int dic_tids_tile_groups(int32_t m) { return m >= 1 ? tile_groups(m) : DIC_EINVAL; }

extern "C" int64_t dic_tids_index(int32_t m, int32_t item, int64_t group) {
    if (m < 1 || item < 0 || item >= m || group < 0) return DIC_EINVAL;
    return tids_index(m, tile_groups(m), (uint32_t)item, group);
}

extern "C" int dic_item_support(const uint32_t* tids, int64_t n, int32_t m, int64_t first, int64_t last,
                                int64_t* counts, void* stream) {
    DIC_REQUIRE(m >= 1 && tids && counts, "dic_item_support: bad arguments");
    DIC_REQUIRE(0 <= first && (last < first || last < n), "chunk [%lld, %lld] outside database of %lld rows",
                (long long)first, (long long)last, (long long)n);
    return item_support_launch(tids, n, m, first, last, reinterpret_cast<unsigned long long*>(counts),
                               as_stream(stream));
}

#ifdef DIC_LAB_TIMING
extern "C" int dic_lab_stamps(unsigned long long* host, int32_t n) {
    cudaDeviceSynchronize();
    DIC_CUDA(cudaMemcpyFromSymbol(host, g_lab_stamp, (size_t)n * 6 * sizeof(unsigned long long)));
    return DIC_OK;
}
#endif

extern "C" int dic_count_support(const uint32_t* tids, int64_t n, int32_t m, int64_t first, int64_t last,
                                 const uint16_t* items, int32_t k, int64_t C, uint64_t* support_inc,
                                 void* stream) {
    DIC_REQUIRE(m >= 1 && m <= 65535, "dic_count_support: m=%d outside [1, 65535]", m);
    DIC_REQUIRE(k >= 1 && k <= m, "dic_count_support: k=%d outside [1, m=%d]", k, m);
    DIC_REQUIRE(0 <= first && first <= last && last < n, "chunk [%lld, %lld] outside database of %lld rows",
                (long long)first, (long long)last, (long long)n);
    DIC_REQUIRE(C >= 0, "dic_count_support: C=%lld < 0", (long long)C);
    if (C == 0) return DIC_OK;
    BucketIn b{items, reinterpret_cast<unsigned long long*>(support_inc), C, k};
    return count_buckets_launch(tids, n, m, first, last, &b, 1, as_stream(stream));
}

extern "C" int dic_count_support_rows(const uint64_t* rows, int32_t W, int64_t first, int64_t last,
                                      const uint64_t* masks, int64_t C, uint64_t* support_inc,
                                      void* stream) {
    DIC_REQUIRE(W >= 1, "dic_count_support_rows: W=%d < 1", W);
    DIC_REQUIRE(0 <= first && first <= last, "chunk [%lld, %lld] invalid", (long long)first,
                (long long)last);
    if (C <= 0) return DIC_OK;
    cudaStream_t s = as_stream(stream);
    int64_t span = last - first + 1;
    int64_t cblocks = (C + kRowCands - 1) / kRowCands;
    DIC_REQUIRE(cblocks <= 65535, "dic_count_support_rows: C=%lld too large for one launch (max %d)",
                (long long)C, 65535 * kRowCands);
    dim3 grid((unsigned)((span + 255) / 256), (unsigned)cblocks);
    auto* r = reinterpret_cast<const unsigned long long*>(rows);
    auto* mk = reinterpret_cast<const unsigned long long*>(masks);
    auto* o = reinterpret_cast<unsigned long long*>(support_inc);
    switch (W) {
        case 1: launch_rows<1>(grid, r, W, first, last, mk, C, o, s); break;
        case 2: launch_rows<2>(grid, r, W, first, last, mk, C, o, s); break;
        case 4: launch_rows<4>(grid, r, W, first, last, mk, C, o, s); break;
        case 8: launch_rows<8>(grid, r, W, first, last, mk, C, o, s); break;
        case 16: launch_rows<16>(grid, r, W, first, last, mk, C, o, s); break;
        default:
            DIC_REQUIRE(W <= 64, "dic_count_support_rows: W=%d > 64 unsupported", W);
            launch_rows<0>(grid, r, W, first, last, mk, C, o, s);
    }
    DIC_CHECK_LAUNCH("count_rows_kernel");
    return DIC_OK;
}
