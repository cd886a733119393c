// pairs_mma.cu — the dense pair triangle on the 5th-generation tensor cores.
//
// first_pass seeds every pair of frequent items (engine.py:165-168) and the
// pair bucket is counted chunk by chunk while it stays dense.  Its count over
// one chunk is the Gram matrix X^T X of the chunk's 0/1 matrix X (rows x
// level1 items): C[a][b] = sum_r x_ra x_rb, i.e. popc(col_a & col_b).  Here
// that contraction runs as tcgen05.mma kind::mxf4 — E2M1 operands (a set bit
// becomes the 4-bit value 1.0 = 0b0010), every E8M0 block scale 1.0, f32
// accumulators in TMEM, exact because a unit spans fewer than 2^24 rows:
//
//   * a persistent CTA per SM owns a slice of the chunk's 8-word stages for
//     one 128 x 256 output tile of the upper triangle (G / T or G / T + 1
//     CTAs per tile);
//   * warp 13 streams the bits of the coming stages into a shared-memory ring
//     with TMA (cp.async.bulk.tensor over a 3-D view of the tids tiles: word,
//     item, tile — items past L come back zero-filled; 32-byte swizzle, so
//     the expanders' reads are conflict-free);
//   * 12 expander warps turn each item's 8 words into 8 x 16 bytes of E2M1
//     nibbles — nibble k of u32 q holds row 4k + (1, 0, 2, 3)[q] of the word,
//     one permutation of the K axis applied to A and B alike, so the dot
//     products are unchanged — stored straight into the canonical no-swizzle
//     K-major UMMA layout (8-row x 16-byte core matrices), then a proxy fence;
//   * one thread (warp 0) issues 4 MMAs (M=128, N=256, K=64) per stage and
//     commits them to the stage's "empty" mbarrier; at the end of a unit the
//     accumulator is committed to "acc_full", and 8 warps read it back with
//     tcgen05.ld, transpose 32 x 32 blocks through shared memory and add them
//     into the triangle (one 64-bit reduction per pair, 8 pairs per sector).
//
// The bit-to-nibble expansion is the price of having no binary tensor path on
// sm_100a (the warp-level b1 MMA is emulated: tools/lab/mmalab.cu measured
// 700 bit-MAC/clk/SM, no better than LOP3/POPC).  kind::i8 (one byte per bit,
// K = 32 per MMA) was measured at 88.6 us per cfg4 chunk against 74.6 us for
// mxf4 with the same pipeline, and removed.
#include "async.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace dic {

constexpr int kTcM = 128, kTcN = 256;     // MMA tile: A items x B items
constexpr int kTcKW = 8;                  // 32-row words per item per stage (4 MMAs of K = 64)
constexpr int kTcMmas = kTcKW / 2;
constexpr int kTcExpWarps = 12;           // expander warps: one operand row (item) per thread
constexpr int kTcThreads = 32 * (2 + kTcExpWarps);  // + warp 0 (TMEM, MMA) + warp 13 (TMA producer)
constexpr uint32_t kTcAStep = kTcM * 32;  // A bytes per MMA (32 bytes of K per row)
constexpr uint32_t kTcBStep = kTcN * 32;  // B bytes per MMA
constexpr uint32_t kTcStageBytes = kTcMmas * (kTcAStep + kTcBStep);   // 48 KB of operands
constexpr int kTcStages = 3;
constexpr uint32_t kTcBitsA = kTcM * kTcKW * 4, kTcBitsB = kTcN * kTcKW * 4;  // a stage's words: [item][8]
constexpr uint32_t kTcBitStage = kTcBitsA + kTcBitsB;                 // 12 KB
constexpr int kTcBitStages = 4;
constexpr uint32_t kTcXposeBytes = 8 * 32 * 33 * 4;  // epilogue: a 32 x 33 transpose tile per warp
constexpr size_t kTcSmem = 1024 + (size_t)kTcStages * kTcStageBytes + (size_t)kTcBitStages * kTcBitStage +
                           kTcXposeBytes;
constexpr uint32_t kTcCols = 512;  // TMEM: accumulator (256 columns) + block scales (256)

// UMMA shared-memory matrix descriptor, no swizzle, K-major: core matrices of
// 8 rows x 16 bytes stored contiguously; lbo = byte distance between the two
// 16-byte K halves of an MMA's 32 bytes of K, sbo = between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, layout type 0 = SWIZZLE_NONE
}

// instruction descriptor, kind::mxf4: A/B E2M1 (format 1 at bits 7 and 10),
// K-major, N >> 3 at 17, scale format E8M0 (bit 23), M >> 4 at 24, K = 64
constexpr uint32_t kTcIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(kTcN >> 3) << 17) | (1u << 23) |
                              ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t accumulate, uint32_t sfa,
                                       uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(
            tmem_d),
        "l"(ad), "l"(bd), "r"(kTcIdesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, uint32_t x) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
        "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
        "r"(x)
        : "memory");
}

// TMA: a 3-D box (words, items, 1 tile) of the tids view into shared memory
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// a < b < L, a-major: the order first_pass seeds pairs in (pairs.cu tri_index)
__device__ __forceinline__ int64_t tc_tri(int64_t a, int64_t b, int64_t L) { return a * L - a * (a + 1) / 2 + (b - a - 1); }

// The tile list of the upper triangle: A block ia (items 128 ia ..) against
// B block ib (items 256 ib ..) for ib >= ia / 2 (every other block pair holds
// no pair a < b).
struct TcTiles {
    int na, nb, T;
};
__device__ __forceinline__ TcTiles tc_tiles(int L) {
    TcTiles t;
    t.na = (L + kTcM - 1) / kTcM;
    t.nb = (L + kTcN - 1) / kTcN;
    t.T = 0;
    for (int ia = 0; ia < t.na; ++ia) t.T += t.nb - ia / 2;
    return t;
}
__device__ __forceinline__ void tc_tile(const TcTiles& tt, int T, int* a0, int* b0) {
    int ia = 0;
    while (T >= tt.nb - ia / 2) {
        T -= tt.nb - ia / 2;
        ++ia;
    }
    *a0 = ia * kTcM;
    *b0 = (ia / 2 + T) * kTcN;
}

// The work of a launch is T tiles x nst stages, split evenly over the grid:
// CTA b walks the contiguous range [W b / G, W (b + 1) / G) of (tile, stage)
// space as segments, one per tile it touches (at most cap stages each, so a
// segment's f32 accumulation stays below 2^24 rows).
struct TcSeg {
    int a0, b0;
    int64_t st0, st1;
};
struct TcWalk {
    TcTiles tt;
    int64_t nst, cap, w, we;
    __device__ __forceinline__ bool next(TcSeg* sg) {
        if (w >= we) return false;
        const int64_t tile = w / nst;
        sg->st0 = w - tile * nst;
        sg->st1 = min(nst, min(sg->st0 + (we - w), sg->st0 + cap));
        tc_tile(tt, (int)tile, &sg->a0, &sg->b0);
        w += sg->st1 - sg->st0;
        return true;
    }
    // The CTA's share.  With at least one CTA per tile, the grid is split
    // tile by tile (tile t gets G / T or G / T + 1 CTAs, each a contiguous
    // slice of its stages): every CTA then owns ONE segment, so no CTA drains
    // and refills its accumulator mid-way (up to 1 / (G / T) more stages for
    // the busiest CTA, against an epilogue of ~8 us).  Fewer CTAs than tiles:
    // the flat equal split of (tile, stage) space.
    __device__ __forceinline__ void share(int b, int G) {
        const int T = tt.T;
        if (G >= T) {
            const int per = G / T, extra = G % T;  // tiles t < extra get per + 1 CTAs
            const int big = extra * (per + 1);
            int t, i, c;
            if (b < big) {
                t = b / (per + 1);
                i = b - t * (per + 1);
                c = per + 1;
            } else {
                t = extra + (b - big) / per;
                i = (b - big) - (t - extra) * per;
                c = per;
            }
            w = (int64_t)t * nst + nst * i / c;
            we = (int64_t)t * nst + nst * (i + 1) / c;
        } else {
            const int64_t W = (int64_t)T * nst;
            w = W * b / G;
            we = W * (b + 1) / G;
        }
    }
};

#ifdef DIC_LAB_TIMING
// lab build: per-CTA phase stamps (globaltimer ns): start, TMEM ready,
// first stage issued, main loop done (accumulator full), epilogue done, exit
__device__ unsigned long long g_lab_tc[1024][6];
#define TC_STAMP(i)                                                          \
    do {                                                                     \
        unsigned long long _t;                                               \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));               \
        g_lab_tc[blockIdx.x][i] = _t;                                        \
    } while (0)
#else
#define TC_STAMP(i) \
    do {            \
    } while (0)
#endif

template <int TW>
__global__ void __launch_bounds__(kTcThreads, 1) pair_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                                                                 const __grid_constant__ CUtensorMap mapB, int L,
                                                                 ChunkGeom geom, unsigned long long* __restrict__ tri,
                                                                 const unsigned long long* bn2, int64_t tri_len,
                                                                 const unsigned long long* abort_flag,
                                                                 const int64_t* chunk_ring,
                                                                 const unsigned long long* seq, int ring) {
    if (abort_flag && (*abort_flag || 2 * (int64_t)*bn2 < tri_len)) return;
    if (chunk_ring) {
        const int64_t sl = (int64_t)(*seq % (unsigned long long)ring);
        const int64_t f = chunk_ring[2 * sl], l = chunk_ring[2 * sl + 1];
        if (l < f) return;
        geom = chunk_geom(f, l);
    }
    extern __shared__ __align__(1024) uint8_t smem[];
    if (threadIdx.x == 0) TC_STAMP(0);
    uint8_t* ops = smem + 1024;  // [stage][A: 4 MMAs x 4 KB][B: 4 MMAs x 8 KB]
    uint8_t* bits = ops + (size_t)kTcStages * kTcStageBytes;  // [bit stage][A items x 8 words][B items x 8 words]
    uint32_t* xpose = reinterpret_cast<uint32_t*>(bits + (size_t)kTcBitStages * kTcBitStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // operands written   [kTcStages]
    uint64_t* empty = full + kTcStages;                   // operands consumed  [kTcStages]
    uint64_t* bfull = empty + kTcStages;                  // bits landed (TMA)  [kTcBitStages]
    uint64_t* bempty = bfull + kTcBitStages;              // bits consumed      [kTcBitStages]
    uint64_t* acc_full = bempty + kTcBitStages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    TcWalk walk;
    walk.tt = tc_tiles(L);
    const int64_t g0 = geom.g_first & ~(int64_t)(kTcKW - 1);
    walk.nst = (geom.g_last - g0) / kTcKW + 1;
    walk.cap = ((int64_t)1 << 23) / (32 * kTcKW);
    walk.share(blockIdx.x, gridDim.x);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], kTcExpWarps);
            mbar_init(&empty[s], 1);
        }
        for (int r = 0; r < kTcBitStages; ++r) {
            mbar_init(&bfull[r], 1);
            mbar_init(&bempty[r], kTcExpWarps);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 8);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                     "n"(kTcCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_base;
    // block scale factors: every byte of TMEM columns 256..511 = 127 (E8M0
    // 1.0), so whatever scale-factor lanes / columns an MMA reads multiply by 1
    if (warp >= 1 && warp <= 4) {
        const uint32_t q = (uint32_t)(warp & 3) * 32u;
        for (int c = 256; c < 512; c += 32) tmem_st32(tmem + (q << 16) + (uint32_t)c, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) TC_STAMP(1);

    if (warp == 0) {
        // ---------------- MMA issuer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0, ue = 0;
            const uint32_t base = smem_u32(ops);
            TcSeg sg;
            while (walk.next(&sg)) {
                mbar_wait(acc_empty, (ue & 1) ^ 1);  // the epilogue has drained the accumulator
                tc_fence_after();
                for (int64_t st = sg.st0; st < sg.st1; ++st) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sa = base + (uint32_t)s * kTcStageBytes;
                    const uint32_t sb = sa + kTcMmas * kTcAStep;
#pragma unroll
                    for (int kk = 0; kk < kTcMmas; ++kk)
                        tc_mma(tmem, umma_desc(sa + kk * kTcAStep, kTcAStep / 2, 128),
                               umma_desc(sb + kk * kTcBStep, kTcBStep / 2, 128), (st > sg.st0 || kk > 0) ? 1u : 0u,
                               tmem + 256u, tmem + 384u);
                    tc_commit(&empty[s]);  // the stage's buffers are free once these MMAs are done
                    if (st == sg.st0 && ue == 0) TC_STAMP(2);
                    if (++s == kTcStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc_commit(acc_full);
                ++ue;
            }
        }
        __syncwarp();
    } else if (warp == 1 + kTcExpWarps) {
        // ---------------- TMA producer: the words of the coming stages
        if (lane == 0) {
            int r = 0;
            uint32_t rph = 0;
            TcSeg sg;
            while (walk.next(&sg)) {
                for (int64_t st = sg.st0; st < sg.st1; ++st) {
                    mbar_wait(&bempty[r], rph ^ 1u);
                    const int64_t g = g0 + st * kTcKW;
                    const int t = (int)(g / TW), x = (int)(g - (int64_t)t * TW);
                    uint8_t* dst = bits + (size_t)r * kTcBitStage;
                    mbar_expect_tx(&bfull[r], kTcBitStage);
                    tma_box(dst, &mapA, x, sg.a0, t, &bfull[r]);
                    tma_box(dst + kTcBitsA, &mapB, x, sg.b0, t, &bfull[r]);
                    if (++r == kTcBitStages) {
                        r = 0;
                        rph ^= 1u;
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- expanders (+ epilogue on warps 1..8)
        const int e = threadIdx.x - 32;  // 0..383: A rows 0..127, B rows 0..255
        const bool isA = e < kTcM;
        const int row = isA ? e : e - kTcM;
        const uint32_t step = isA ? kTcAStep : kTcBStep;
        const uint32_t off0 = (isA ? 0u : kTcMmas * kTcAStep) + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
        const uint32_t boff = (isA ? 0u : kTcBitsA) + (uint32_t)row * (kTcKW * 4);
        const uint32_t bsw = ((uint32_t)row >> 2 & 1u) * 16u;  // SWIZZLE_32B: chunk bit 4 ^= address bit 7
        uint32_t* xp = xpose + (warp - 1) * 32 * 33;
        int s = 0, r = 0;
        uint32_t ph = 0, rph = 0, ue = 0;
        TcSeg sg;
        while (walk.next(&sg)) {
            const int n = (int)(sg.st1 - sg.st0);
            // stages whose words may cross the chunk's ends: the chunk's first and last
            const int edge0 = sg.st0 == 0 ? 0 : -1;
            const int edge1 = (int)(walk.nst - 1 - sg.st0);
            for (int j = 0; j < n; ++j) {
                mbar_wait(&bfull[r], rph);
                // the TMA box is 32-byte swizzled (16-byte chunk c of row e at
                // chunk c ^ bit 2 of e): the 8 rows of a quarter-warp's load
                // cover all 8 bank groups
                const uint8_t* bsrc = bits + (size_t)r * kTcBitStage + boff;
                const uint4 a0 = *reinterpret_cast<const uint4*>(bsrc + bsw);
                const uint4 a1 = *reinterpret_cast<const uint4*>(bsrc + (16u ^ bsw));
                uint32_t wv[kTcKW] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                __syncwarp();
                if (lane == 0) mbar_arrive(&bempty[r]);
                if (++r == kTcBitStages) {
                    r = 0;
                    rph ^= 1u;
                }
                if (j == edge0 || j == edge1) {
                    // the chunk's first / last stage: zero the rows outside [first, last]
                    const int64_t g = g0 + (sg.st0 + j) * kTcKW;
#pragma unroll
                    for (int i = 0; i < kTcKW; ++i) wv[i] &= group_mask(geom, g + i);
                }
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* dst = ops + (size_t)s * kTcStageBytes + off0;
                // word x -> 8 nibbles per u32: nibble k = 0b0010 (E2M1 1.0) iff its bit is set
#pragma unroll
                for (int kk = 0; kk < kTcMmas; ++kk) {
                    const uint32_t x = wv[2 * kk], y = wv[2 * kk + 1];
                    uint4 lo, hi;
                    lo.x = x & 0x22222222u;
                    lo.y = (x << 1) & 0x22222222u;
                    lo.z = (x >> 1) & 0x22222222u;
                    lo.w = (x >> 2) & 0x22222222u;
                    hi.x = y & 0x22222222u;
                    hi.y = (y << 1) & 0x22222222u;
                    hi.z = (y >> 1) & 0x22222222u;
                    hi.w = (y >> 2) & 0x22222222u;
                    uint8_t* d = dst + kk * step;
                    *reinterpret_cast<uint4*>(d) = lo;
                    *reinterpret_cast<uint4*>(d + step / 2) = hi;
                }
                fence_proxy_async();  // generic-proxy stores -> visible to the tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (++s == kTcStages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            // epilogue: warps 1..8 read the accumulator back (warp w: TMEM lanes
            // 32 (w % 4) .., columns 128 ((w - 1) / 4) ..).  A 32 x 32 block is
            // transposed through shared memory so that lane t adds column t of a
            // row: the 32 reductions of one instruction hit 8 consecutive sectors
            // of the triangle row instead of 32 rows.
            if (warp <= 8) {
                mbar_wait(acc_full, ue & 1);
                tc_fence_after();
                if (threadIdx.x == 32) TC_STAMP(3);
                const int q = warp & 3, half = (warp - 1) >> 2;
                const int ar = sg.a0 + q * 32;  // first row of this warp's lanes
                for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) xp[lane * 33 + jj] = v[jj];
                    __syncwarp();
                    const int b = sg.b0 + c0 + lane;
#pragma unroll 4
                    for (int jj = 0; jj < 32; ++jj) {
                        const uint32_t cnt = __float2uint_rn(__uint_as_float(xp[jj * 33 + lane]));
                        const int a = ar + jj;
                        if (cnt && a < b && b < L)
                            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(tri + tc_tri(a, b, L)),
                                         "l"((unsigned long long)cnt)
                                         : "memory");
                    }
                    __syncwarp();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(acc_empty);
                if (threadIdx.x == 32) TC_STAMP(4);
            }
            ++ue;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TC_STAMP(5);
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcCols));
    }
}

#ifdef DIC_LAB_TIMING
extern "C" int dic_lab_tc_stamps(unsigned long long* host) {
    cudaDeviceSynchronize();
    DIC_CUDA(cudaMemcpyFromSymbol(host, g_lab_tc, sizeof(g_lab_tc)));
    return DIC_OK;
}
#endif

// ---------------------------------------------------------------------------
// host: tensor maps over the tids tiles (a 3-D view: word-in-row x item x
// tile; strides RW*4 and L*RW*4 bytes)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

static int make_map(CUtensorMap* map, const uint32_t* tids, int L, int64_t tiles, int TW, int box_items) {
    auto enc = encode_fn();
    if (!enc) {
        set_error("pair_tc: cuTensorMapEncodeTiled unavailable");
        return DIC_ECUDA;
    }
    const int RW = row_words(TW);
    cuuint64_t dims[3] = {(cuuint64_t)RW, (cuuint64_t)L, (cuuint64_t)tiles};
    cuuint64_t strides[2] = {(cuuint64_t)RW * 4, (cuuint64_t)L * RW * 4};
    cuuint32_t box[3] = {(cuuint32_t)kTcKW, (cuuint32_t)box_items, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(tids), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("pair_tc: cuTensorMapEncodeTiled failed (%d)", (int)r);
        return DIC_ECUDA;
    }
    return DIC_OK;
}

template <int TW>
static int pair_tc_go(const CUtensorMap& ma, const CUtensorMap& mb, int L, ChunkGeom geom, unsigned long long* tri,
                      const unsigned long long* bn2, int64_t tri_len, const unsigned long long* abort_flag,
                      const int64_t* chunk_ring, const unsigned long long* seq, int ring, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        DIC_CUDA(cudaFuncSetAttribute(pair_tc_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
        attr = true;
    }
    pair_tc_kernel<TW><<<(unsigned)sm_count(), kTcThreads, kTcSmem, s>>>(ma, mb, L, geom, tri, bn2, tri_len,
                                                                         abort_flag, chunk_ring, seq, ring);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("pair_tc_kernel");
    return DIC_OK;
}

// launch (pairs.cu decides when the tensor path runs); n = rows of the tids buffer
int pair_tc_launch(const uint32_t* tids, int64_t n, int L, ChunkGeom geom, unsigned long long* tri,
                   const unsigned long long* bn2, int64_t tri_len, const unsigned long long* abort_flag,
                   const int64_t* chunk_ring, const unsigned long long* seq, int ring, cudaStream_t s) {
    const int TW = tile_groups(L);
    const int64_t tiles = tile_count(n, L);
    CUtensorMap ma, mb;
    int rc;
    if ((rc = make_map(&ma, tids, L, tiles, TW, kTcM)) || (rc = make_map(&mb, tids, L, tiles, TW, kTcN))) return rc;
    return TW == 32 ? pair_tc_go<32>(ma, mb, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring, s)
                    : pair_tc_go<16>(ma, mb, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring, s);
}

}  // namespace dic
