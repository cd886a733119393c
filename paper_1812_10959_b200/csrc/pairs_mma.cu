// pairs_mma.cu — the dense pair triangle on the 5th-generation tensor cores.
//
// first_pass seeds every pair of frequent items (engine.py:165-168) and the
// pair bucket is counted chunk by chunk while it stays dense.  Its count over
// one chunk is the Gram matrix X^T X of the chunk's 0/1 matrix X (rows x
// level1 items): C[a][b] = sum_r x_ra x_rb, i.e. popc(col_a & col_b).  Here
// that contraction runs as tcgen05.mma kind::i8 (u8 x u8 -> s32 in TMEM,
// exact: a chunk has < 2^31 rows):
//
//   * a persistent CTA per SM walks units = (128 x 256 output tile of the
//     upper triangle, slice of the chunk's 32-row words);
//   * 12 expander warps turn the bit-sliced words into u8 operands: item
//     row j of the tile, 4 words per stage; word x becomes 8 u32
//     (x >> q) & 0x01010101 (q = 0..7), i.e. byte k of a 32-byte K step holds
//     row 8(k % 4) + k / 4 of the word — a permutation of K applied to A and
//     B alike, so the dot products are unchanged — stored straight into the
//     canonical no-swizzle K-major UMMA layout (8-row x 16-byte core
//     matrices) in shared memory;
//   * one thread issues 4 MMAs (M=128, N=256, K=32) per stage and commits
//     them to the stage's "empty" mbarrier; at the end of a unit the
//     accumulator is committed to "acc_full", and 8 warps read it back with
//     tcgen05.ld (32 lanes x 32 columns per load) and add it into the
//     triangle (one 64-bit reduction per pair).
//
// The bit-to-byte expansion is the price of having no binary tensor path on
// sm_100a (the warp-level b1 MMA is emulated: tools/lab/mmalab.cu measured
// 700 bit-MAC/clk/SM, no better than LOP3/POPC).  Per 32 rows a tile needs
// 384 words expanded (15 ALU ops each) against 1M MACs of MMA.
#include "async.cuh"

namespace dic {

constexpr int kTcM = 128, kTcN = 256;     // MMA tile: A items x B items
constexpr int kTcKW = 16;                 // 32-row words per item per stage
constexpr int kTcExpWarps = 12;           // expander warps: one operand row (item) per thread
constexpr int kTcThreads = 32 * (1 + kTcExpWarps);  // + warp 0: TMEM owner and MMA issuer
constexpr uint32_t kTcAStep = kTcM * 32;  // A bytes per MMA (32 bytes of K per row)
constexpr uint32_t kTcBStep = kTcN * 32;  // B bytes per MMA

// FP4 = false: kind::i8, one 32-row word per MMA (K = 32 u8), s32 accumulators.
// FP4 = true: kind::mxf4 (E2M1 operands, E8M0 block scales all 1.0), two
// words per MMA (K = 64 packed 4-bit values), f32 accumulators (exact: a unit
// spans < 2^24 rows).  Same 32 bytes of K per row and MMA either way, so the
// shared-memory layout is the same; FP4 halves the expansion and doubles the
// rows per MMA.
template <bool FP4>
struct TcCfg {
    static constexpr int WPM = FP4 ? 2 : 1;             // words per MMA
    static constexpr int MMAS = kTcKW / WPM;            // MMAs per stage
    static constexpr uint32_t StageBytes = MMAS * (kTcAStep + kTcBStep);
    static constexpr int Stages = FP4 ? 2 : 1;
    static constexpr uint32_t XposeBytes = 8 * 32 * 33 * 4;  // epilogue: a 32 x 33 transpose tile per warp
    static constexpr size_t Smem = 1024 + (size_t)Stages * StageBytes + XposeBytes;
    static constexpr uint32_t Cols = FP4 ? 512 : 256;   // accumulator (256) + scale factors (FP4)
};

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

// instruction descriptors
// kind::i8: D = s32 (bits 4-5 = 2), A/B unsigned 8-bit, K-major, N >> 3 at 17, M >> 4 at 24
constexpr uint32_t kTcIdescI8 = (2u << 4) | ((uint32_t)(kTcN >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
// kind::mxf4: A/B E2M1 (format 1 at bits 7 and 10), scale format E8M0 (bit 23), K = 64
constexpr uint32_t kTcIdescF4 = (1u << 7) | (1u << 10) | ((uint32_t)(kTcN >> 3) << 17) | (1u << 23) |
                                ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <bool FP4>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t accumulate, uint32_t sfa,
                                       uint32_t sfb) {
    if constexpr (FP4) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(
                tmem_d),
            "l"(ad), "l"(bd), "r"(kTcIdescF4), "r"(accumulate), "r"(sfa), "r"(sfb)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(kTcIdescI8), "r"(accumulate)
            : "memory");
    }
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
// space as segments, one per tile it touches (at most cap stages each).
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
};

template <int TW, bool FP4>
__global__ void __launch_bounds__(kTcThreads, 1) pair_tc_kernel(const uint32_t* __restrict__ tids, int L,
                                                                 ChunkGeom geom, unsigned long long* __restrict__ tri,
                                                                 const unsigned long long* bn2, int64_t tri_len,
                                                                 const unsigned long long* abort_flag,
                                                                 const int64_t* chunk_ring,
                                                                 const unsigned long long* seq, int ring) {
    using Cfg = TcCfg<FP4>;
    if (abort_flag && (*abort_flag || 2 * (int64_t)*bn2 < tri_len)) return;
    if (chunk_ring) {
        const int64_t sl = (int64_t)(*seq % (unsigned long long)ring);
        const int64_t f = chunk_ring[2 * sl], l = chunk_ring[2 * sl + 1];
        if (l < f) return;
        geom = chunk_geom(f, l);
    }
    constexpr int RW = TW + 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ops = smem + 1024;  // [stage][A: MMAS x 4 KB][B: MMAS x 8 KB]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);        // [Stages]
    uint64_t* empty = full + Cfg::Stages;                      // [Stages]
    uint64_t* acc_full = empty + Cfg::Stages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    TcWalk walk;
    walk.tt = tc_tiles(L);
    const int64_t g0 = geom.g_first & ~(int64_t)(kTcKW - 1);
    walk.nst = (geom.g_last - g0) / kTcKW + 1;
    walk.cap = FP4 ? ((int64_t)1 << 23) / (32 * kTcKW) : ((int64_t)1 << 40);
    const int64_t W = (int64_t)walk.tt.T * walk.nst;
    walk.w = W * blockIdx.x / gridDim.x;
    walk.we = W * (blockIdx.x + 1) / gridDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < Cfg::Stages; ++s) {
            mbar_init(&full[s], kTcExpWarps);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 8);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                     "n"(Cfg::Cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_base;
    if constexpr (FP4) {
        // block scale factors: every byte of TMEM columns 256..511 = 127 (E8M0 1.0),
        // so whatever scale-factor lanes / columns an MMA reads multiply by 1
        if (warp >= 1 && warp <= 4) {
            const uint32_t q = (uint32_t)(warp & 3) * 32u;
            for (int c = 256; c < 512; c += 32) tmem_st32(tmem + (q << 16) + (uint32_t)c, 0x7F7F7F7Fu);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }

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
                    const uint32_t sa = base + (uint32_t)s * Cfg::StageBytes;
                    const uint32_t sb = sa + Cfg::MMAS * kTcAStep;
#pragma unroll
                    for (int kk = 0; kk < Cfg::MMAS; ++kk)
                        tc_mma<FP4>(tmem, umma_desc(sa + kk * kTcAStep, kTcAStep / 2, 128),
                                    umma_desc(sb + kk * kTcBStep, kTcBStep / 2, 128), (st > sg.st0 || kk > 0) ? 1u : 0u,
                                    tmem + 256u, tmem + 384u);
                    tc_commit(&empty[s]);  // the stage's buffers are free once these MMAs are done
                    if (++s == Cfg::Stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc_commit(acc_full);
                ++ue;
            }
        }
        __syncwarp();
    } else {
        // ---------------- expanders (+ epilogue on warps 1..8)
        const int e = threadIdx.x - 32;  // 0..383: A rows 0..127, B rows 0..255
        const bool isA = e < kTcM;
        const int row = isA ? e : e - kTcM;
        const uint32_t step = isA ? kTcAStep : kTcBStep;
        const uint32_t off0 = (isA ? 0u : Cfg::MMAS * kTcAStep) + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
        const int64_t tile_vec = (int64_t)L * RW / 4;  // a tile in uint4 units
        uint32_t* xp = reinterpret_cast<uint32_t*>(ops + (size_t)Cfg::Stages * Cfg::StageBytes) + (warp - 1) * 32 * 33;
        int s = 0;
        uint32_t ph = 0, ue = 0;
        TcSeg sg;
        while (walk.next(&sg)) {
            const int item = (isA ? sg.a0 : sg.b0) + row;
            const bool live = item < L;
            const int n = (int)(sg.st1 - sg.st0);
            // running position of the next stage to load: tile row pointer + slot
            const int64_t gs = g0 + sg.st0 * kTcKW;
            const int64_t ts = gs / TW;
            const uint4* p = reinterpret_cast<const uint4*>(tids + ts * (int64_t)L * RW + (int64_t)item * RW) +
                             (gs - ts * TW) / 4;
            int slot = (int)(gs - ts * TW);
            // stages whose words may cross the chunk's ends: the chunk's first and last
            const int edge0 = sg.st0 == 0 ? 0 : -1;
            const int edge1 = (int)(walk.nst - 1 - sg.st0);
            constexpr int NV = kTcKW / 4;  // uint4 per stage
            auto load = [&](int j, uint4 (&w)[NV]) {
#pragma unroll
                for (int v = 0; v < NV; ++v) w[v] = make_uint4(0u, 0u, 0u, 0u);
                if (live && j < n) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) w[v] = __ldg(p + v);
                }
                p += NV;
                slot += kTcKW;
                if (slot == TW) {
                    slot = 0;
                    p += tile_vec - TW / 4;
                }
            };
            uint4 cur[NV], nxt[NV];
            load(0, cur);
            load(1, nxt);
            for (int j = 0; j < n; ++j) {
                uint32_t wv[kTcKW];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    wv[4 * v] = cur[v].x;
                    wv[4 * v + 1] = cur[v].y;
                    wv[4 * v + 2] = cur[v].z;
                    wv[4 * v + 3] = cur[v].w;
                    cur[v] = nxt[v];
                }
                if (j == edge0 || j == edge1) {
                    // the chunk's first / last stage: zero the rows outside [first, last]
                    const int64_t g = g0 + (sg.st0 + j) * kTcKW;
#pragma unroll
                    for (int i = 0; i < kTcKW; ++i) wv[i] &= group_mask(geom, g + i);
                }
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* dst = ops + (size_t)s * Cfg::StageBytes + off0;
                if constexpr (FP4) {
                    // word x -> 8 nibbles per u32: nibble k = 0b0010 (E2M1 1.0) iff its bit is set
#pragma unroll
                    for (int kk = 0; kk < Cfg::MMAS; ++kk) {
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
                } else {
                    // word x -> 8 u32 of bytes: byte j of u32 q = bit 8j + q
#pragma unroll
                    for (int kk = 0; kk < Cfg::MMAS; ++kk) {
                        const uint32_t x = wv[kk];
                        uint4 lo, hi;
                        lo.x = x & 0x01010101u;
                        lo.y = (x >> 1) & 0x01010101u;
                        lo.z = (x >> 2) & 0x01010101u;
                        lo.w = (x >> 3) & 0x01010101u;
                        hi.x = (x >> 4) & 0x01010101u;
                        hi.y = (x >> 5) & 0x01010101u;
                        hi.z = (x >> 6) & 0x01010101u;
                        hi.w = (x >> 7) & 0x01010101u;
                        uint8_t* d = dst + kk * step;
                        *reinterpret_cast<uint4*>(d) = lo;
                        *reinterpret_cast<uint4*>(d + step / 2) = hi;
                    }
                }
                fence_proxy_async();  // generic-proxy stores -> visible to the tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (++s == Cfg::Stages) {
                    s = 0;
                    ph ^= 1u;
                }
                // the stage after next, issued after the proxy fence (which would
                // otherwise wait for these loads too)
                load(j + 2, nxt);
            }
            // epilogue: warps 1..8 read the accumulator back (warp w: TMEM lanes
            // 32 (w % 4) .., columns 128 ((w - 1) / 4) ..).  A 32 x 32 block is
            // transposed through shared memory so that lane t adds column t of a
            // row: the 32 reductions of one instruction hit 8 consecutive sectors
            // of the triangle row instead of 32 rows.
            if (warp <= 8) {
                mbar_wait(acc_full, ue & 1);
                tc_fence_after();
                const int q = warp & 3, half = (warp - 1) >> 2;
                const int ar = sg.a0 + q * 32;  // first row of this warp's lanes
                for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) xp[lane * 33 + j] = v[j];
                    __syncwarp();
                    const int b = sg.b0 + c0 + lane;
#pragma unroll 4
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t raw = xp[j * 33 + lane];
                        const uint32_t cnt = FP4 ? __float2uint_rn(__uint_as_float(raw)) : raw;
                        const int a = ar + j;
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
            }
            ++ue;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::Cols));
    }
}

// launch (pairs.cu decides when the tensor path runs).  DIC_PAIR_TC_KIND:
// 4 = mxf4 (default), 8 = i8.
template <int TW, bool FP4>
static int pair_tc_go(const uint32_t* tids, int L, ChunkGeom geom, unsigned long long* tri,
                      const unsigned long long* bn2, int64_t tri_len, const unsigned long long* abort_flag,
                      const int64_t* chunk_ring, const unsigned long long* seq, int ring, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        DIC_CUDA(cudaFuncSetAttribute(pair_tc_kernel<TW, FP4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)TcCfg<FP4>::Smem));
        attr = true;
    }
    pair_tc_kernel<TW, FP4><<<(unsigned)sm_count(), kTcThreads, TcCfg<FP4>::Smem, s>>>(
        tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("pair_tc_kernel");
    return DIC_OK;
}

int pair_tc_launch(const uint32_t* tids, int L, ChunkGeom geom, unsigned long long* tri, const unsigned long long* bn2,
                   int64_t tri_len, const unsigned long long* abort_flag, const int64_t* chunk_ring,
                   const unsigned long long* seq, int ring, cudaStream_t s) {
    static const bool fp4 = [] {
        const char* e = getenv("DIC_PAIR_TC_KIND");
        return !(e && atoi(e) == 8);
    }();
    const int TW = tile_groups(L);
    if (fp4)
        return TW == 32 ? pair_tc_go<32, true>(tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring, s)
                        : pair_tc_go<16, true>(tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring, s);
    return TW == 32 ? pair_tc_go<32, false>(tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring, s)
                    : pair_tc_go<16, false>(tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring, seq, ring, s);
}

}  // namespace dic
