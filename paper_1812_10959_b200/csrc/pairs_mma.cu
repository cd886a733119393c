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
constexpr int kTcKS = 4;                  // 32-row words (K steps of 32 bytes) per stage
constexpr int kTcStages = 3;
constexpr int kTcExpWarps = 12;           // expander warps: one operand row (item) per thread
constexpr int kTcThreads = 32 * (kTcExpWarps + 1);  // + warp 0: TMEM owner and MMA issuer
constexpr uint32_t kTcAStep = kTcM * 32;  // A bytes per K step
constexpr uint32_t kTcBStep = kTcN * 32;  // B bytes per K step
constexpr uint32_t kTcStageBytes = kTcKS * (kTcAStep + kTcBStep);
constexpr size_t kTcSmem = 1024 + (size_t)kTcStages * kTcStageBytes;
constexpr uint32_t kTcCols = 256;         // TMEM columns: the 128 x 256 s32 accumulator

// UMMA shared-memory matrix descriptor, no swizzle, K-major: core matrices of
// 8 rows x 16 bytes stored contiguously; lbo = byte distance between the two
// 16-byte K halves of a 32-byte K step, sbo = between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, layout type 0 = SWIZZLE_NONE
}

// instruction descriptor: kind::i8, A/B unsigned 8-bit, K-major, D = s32, M x N
constexpr uint32_t kTcIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(kTcIdesc), "r"(accumulate)
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

// units: T tiles x S slices of the chunk's stages; unit u = (tile u / S, slice u % S)
struct TcUnit {
    int a0, b0;
    int64_t st0, st1;  // stage range [st0, st1)
};
__device__ __forceinline__ TcUnit tc_unit(const TcTiles& tt, int S, int64_t nst, int64_t u) {
    TcUnit r;
    tc_tile(tt, (int)(u / S), &r.a0, &r.b0);
    const int64_t sl = u % S;
    r.st0 = nst * sl / S;
    r.st1 = nst * (sl + 1) / S;
    return r;
}

template <int TW>
__global__ void __launch_bounds__(kTcThreads, 1) pair_tc_kernel(const uint32_t* __restrict__ tids, int L,
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
    constexpr int RW = TW + 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ops = smem + 1024;  // [stage][A: kTcKS x 4 KB][B: kTcKS x 8 KB]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);        // [kTcStages]
    uint64_t* empty = full + kTcStages;                          // [kTcStages]
    uint64_t* acc_full = empty + kTcStages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TcTiles tt = tc_tiles(L);
    const int S = max(1, (int)gridDim.x / tt.T);
    const int64_t U = (int64_t)tt.T * S;
    const int64_t g0 = geom.g_first & ~3ll;
    const int64_t nst = (geom.g_last - g0) / kTcKS + 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], kTcExpWarps);
            mbar_init(&empty[s], 1);
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

    if (warp == 0) {
        // ---------------- MMA issuer
        if (lane == 0) {
            int64_t it = 0, ue = 0;
            const uint32_t base = smem_u32(ops);
            for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
                const TcUnit un = tc_unit(tt, S, nst, u);
                if (un.st1 <= un.st0) continue;
                mbar_wait(acc_empty, (uint32_t)((ue & 1) ^ 1));  // the epilogue has drained the accumulator
                tc_fence_after();
                for (int64_t st = un.st0; st < un.st1; ++st, ++it) {
                    const int s = (int)(it % kTcStages);
                    mbar_wait(&full[s], (uint32_t)((it / kTcStages) & 1));
                    tc_fence_after();
                    const uint32_t sa = base + (uint32_t)s * kTcStageBytes;
                    const uint32_t sb = sa + kTcKS * kTcAStep;
#pragma unroll
                    for (int kk = 0; kk < kTcKS; ++kk)
                        tc_mma(tmem, umma_desc(sa + kk * kTcAStep, kTcAStep / 2, 128),
                               umma_desc(sb + kk * kTcBStep, kTcBStep / 2, 128), (st > un.st0 || kk > 0) ? 1u : 0u);
                    tc_commit(&empty[s]);  // the stage's buffers are free once these MMAs are done
                }
                tc_commit(acc_full);
                ++ue;
            }
        }
        __syncwarp();
    } else {
        // ---------------- expanders (+ epilogue on warps 1..8)
        const int e = threadIdx.x - 32;          // 0..383: A rows 0..127, B rows 0..255
        const bool isA = e < kTcM;
        const int row = isA ? e : e - kTcM;
        const uint32_t step = isA ? kTcAStep : kTcBStep;
        const uint32_t off0 = (isA ? 0u : kTcKS * kTcAStep) + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
        const int64_t tile_words = (int64_t)L * RW;
        int64_t it = 0, ue = 0;
        for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
            const TcUnit un = tc_unit(tt, S, nst, u);
            if (un.st1 <= un.st0) continue;
            const int item = (isA ? un.a0 : un.b0) + row;
            const bool live = item < L;
            auto load = [&](int64_t st) -> uint4 {
                uint4 w = make_uint4(0u, 0u, 0u, 0u);
                if (live && st < un.st1) {
                    const int64_t g = g0 + st * kTcKS;
                    const int64_t t = g / TW;
                    w = __ldg(reinterpret_cast<const uint4*>(tids + t * tile_words + (int64_t)item * RW + (g - t * TW)));
                    if (g <= geom.g_first || g + 3 >= geom.g_last) {  // partial words at the chunk's ends
                        w.x &= group_mask(geom, g);
                        w.y &= group_mask(geom, g + 1);
                        w.z &= group_mask(geom, g + 2);
                        w.w &= group_mask(geom, g + 3);
                    }
                }
                return w;
            };
            uint4 nx1 = load(un.st0), nx2 = load(un.st0 + 1);
            for (int64_t st = un.st0; st < un.st1; ++st, ++it) {
                const uint4 cur = nx1;
                nx1 = nx2;
                nx2 = load(st + 2);
                const int s = (int)(it % kTcStages);
                mbar_wait(&empty[s], (uint32_t)(((it / kTcStages) & 1) ^ 1));
                uint8_t* dst = ops + (size_t)s * kTcStageBytes + off0;
                const uint32_t wv[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
                for (int kk = 0; kk < kTcKS; ++kk) {
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
                    *reinterpret_cast<uint4*>(d) = lo;              // K bytes 0..15
                    *reinterpret_cast<uint4*>(d + step / 2) = hi;   // K bytes 16..31
                }
                fence_proxy_async();  // generic-proxy stores -> visible to the tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
            // epilogue: warps 1..8 read the accumulator back (warp w: TMEM lanes
            // 32 (w % 4) .., columns 128 ((w - 1) / 4) ..)
            if (warp <= 8) {
                mbar_wait(acc_full, (uint32_t)(ue & 1));
                tc_fence_after();
                const int q = warp & 3, half = (warp - 1) >> 2;
                const int a = un.a0 + q * 32 + lane;
                for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
                    if (a < L) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int b = un.b0 + c0 + j;
                            if (v[j] && a < b && b < L)
                                asm volatile("red.global.add.u64 [%0], %1;" ::"l"(tri + tc_tri(a, b, L)),
                                             "l"((unsigned long long)v[j])
                                             : "memory");
                        }
                    }
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
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcCols));
    }
}

// launch (pairs.cu decides when the tensor path runs)
int pair_tc_launch(const uint32_t* tids, int L, ChunkGeom geom, unsigned long long* tri, const unsigned long long* bn2,
                   int64_t tri_len, const unsigned long long* abort_flag, const int64_t* chunk_ring,
                   const unsigned long long* seq, int ring, cudaStream_t s) {
    static bool attr[2] = {false, false};
    const int TW = tile_groups(L);
    const int idx = TW == 32 ? 1 : 0;
    if (!attr[idx]) {
        if (TW == 32)
            DIC_CUDA(cudaFuncSetAttribute(pair_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
        else
            DIC_CUDA(cudaFuncSetAttribute(pair_tc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
        attr[idx] = true;
    }
    const unsigned grid = (unsigned)sm_count();
    if (TW == 32)
        pair_tc_kernel<32><<<grid, kTcThreads, kTcSmem, s>>>(tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring,
                                                              seq, ring);
    else
        pair_tc_kernel<16><<<grid, kTcThreads, kTcSmem, s>>>(tids, L, geom, tri, bn2, tri_len, abort_flag, chunk_ring,
                                                              seq, ring);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("pair_tc_kernel");
    return DIC_OK;
}

}  // namespace dic
