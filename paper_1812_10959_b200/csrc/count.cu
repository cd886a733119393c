// count.cu — support counting.
//
//   dic_item_support        first_pass singleton counts (engine.py:132-154)
//   dic_count_support       THE hot kernel: _count_block (engine.py:43-58) for
//                           a whole size-k bucket of dashed candidates over one
//                           chunk, on the bit-sliced layout
//   dic_count_support_rows  the literal (T & I) == I form on the row bitmap
//
// Design: the reference scans the chunk once PER
// candidate with three NumPy passes.  Here a CTA stages one tile of the chunk
// — 32 row-groups (1024 rows) x all m items, 128 B per item — in shared
// memory ONCE, then every thread walks its candidates over the tile:
//   count += popc(AND_{i in I} tile[i][g])      for the 32 groups g
// i.e. (k-1) ANDs + 1 POPC per 32 rows instead of ~2W LOP3s per row.  Rows
// are XOR-swizzled in 16-byte chunks (chunk' = chunk ^ (item & 7)) so the
// LDS.128 of 8 lanes touching 8 different items hit 8 different bank groups.
#include "common.cuh"

namespace dic {

constexpr int kCountThreads = 256;

// ---------------------------------------------------------------------------
// item support
// ---------------------------------------------------------------------------
// grid = (m, splits).  Each CTA sums popcounts of one item's words over a
// slice of the chunk's groups with 128-bit loads; edge groups are masked.
__global__ void __launch_bounds__(256) item_support_kernel(
    const uint32_t* __restrict__ tids, int64_t ld, ChunkGeom geom, int64_t groups_per_cta,
    unsigned long long* __restrict__ counts) {
    const int item = blockIdx.x;
    const uint32_t* col = tids + (int64_t)item * ld;
    int64_t gb = (geom.g_first & ~3LL) + (int64_t)blockIdx.y * groups_per_cta;
    int64_t ge = min(gb + groups_per_cta, geom.g_last + 1);
    unsigned long long acc = 0;
    for (int64_t g = gb + 4 * threadIdx.x; g < ge; g += 4 * blockDim.x) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(col + g));
        acc += __popc(v.x & group_mask(geom, g)) + __popc(v.y & group_mask(geom, g + 1)) +
               __popc(v.z & group_mask(geom, g + 2)) + __popc(v.w & group_mask(geom, g + 3));
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xFFFFFFFFu, acc, o);
    __shared__ unsigned long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        if (t) atomicAdd(counts + item, t);
    }
}

// ---------------------------------------------------------------------------
// bit-sliced support count
// ---------------------------------------------------------------------------
// Byte offset of item's 128-byte row in plane 0 with its swizzle folded in;
// logical chunk q of the row is at (off ^ (q << 4)).
__device__ __forceinline__ uint32_t row_off(uint32_t item) {
    return (item << 7) | ((item & 7u) << 4);
}

// Stage tile groups [gbase, gbase + 32*P) of all m items into shared memory,
// zeroing everything outside the chunk.  gbase is a multiple of 32 and
// ld a multiple of 32, so every 16-byte load is aligned and in bounds.
__device__ __forceinline__ void stage_tile(uint8_t* smem, const uint32_t* __restrict__ tids,
                                           int64_t ld, int m, int P, int64_t gbase,
                                           const ChunkGeom& geom) {
    const int per_plane = m * 8;
    const int total = P * per_plane;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int p = idx / per_plane;
        const int rem = idx - p * per_plane;
        const int i = rem >> 3, q = rem & 7;
        const int64_t g = gbase + p * 32 + q * 4;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (g <= geom.g_last && g + 3 >= geom.g_first) {
            v = __ldg(reinterpret_cast<const uint4*>(tids + (int64_t)i * ld + g));
            v.x &= group_mask(geom, g);
            v.y &= group_mask(geom, g + 1);
            v.z &= group_mask(geom, g + 2);
            v.w &= group_mask(geom, g + 3);
        }
        *reinterpret_cast<uint4*>(smem + (size_t)p * m * 128 + (row_off((uint32_t)i) ^ (q << 4))) = v;
    }
}

__device__ __forceinline__ uint32_t popc4(uint4 v) {
    return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
}

__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) {
    return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w);
}

template <int K>
__global__ void __launch_bounds__(kCountThreads) count_tile_kernel(
    const uint32_t* __restrict__ tids, int64_t ld, int m, int P, ChunkGeom geom, int64_t g0,
    const uint16_t* __restrict__ items, int kdyn, int64_t C, int64_t cands_per_cta,
    unsigned long long* __restrict__ out) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int64_t gbase = g0 + (int64_t)blockIdx.x * P * 32;
    stage_tile(smem, tids, ld, m, P, gbase, geom);
    __syncthreads();

    const int64_t cbeg = (int64_t)blockIdx.y * cands_per_cta;
    const int64_t cend = min(C, cbeg + cands_per_cta);
    const uint32_t plane_bytes = (uint32_t)m * 128u;
    const int k = K > 0 ? K : kdyn;
    for (int64_t c = cbeg + threadIdx.x; c < cend; c += blockDim.x) {
        uint32_t cnt = 0;
        if constexpr (K > 0) {
            uint32_t off[K];
#pragma unroll
            for (int j = 0; j < K; ++j) off[j] = row_off(__ldg(items + c * K + j));
            for (int p = 0; p < P; ++p) {
                const uint8_t* base = smem + (size_t)p * plane_bytes;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint4 a = *reinterpret_cast<const uint4*>(base + (off[0] ^ (q << 4)));
#pragma unroll
                    for (int j = 1; j < K; ++j)
                        a = and4(a, *reinterpret_cast<const uint4*>(base + (off[j] ^ (q << 4))));
                    cnt += popc4(a);
                }
            }
        } else {
            // generic size: item offsets re-read per chunk (L1-resident)
            const uint16_t* it = items + c * (int64_t)k;
            for (int p = 0; p < P; ++p) {
                const uint8_t* base = smem + (size_t)p * plane_bytes;
                for (int q = 0; q < 8; ++q) {
                    uint4 a = make_uint4(~0u, ~0u, ~0u, ~0u);
                    for (int j = 0; j < k; ++j)
                        a = and4(a, *reinterpret_cast<const uint4*>(base + (row_off(__ldg(it + j)) ^ (q << 4))));
                    cnt += popc4(a);
                }
            }
        }
        if (cnt) atomicAdd(out + c, (unsigned long long)cnt);
    }
}

// Fallback for universes too wide to stage (m * 128 B > shared memory):
// every thread reads the tids words straight from global memory / L1.
__global__ void __launch_bounds__(256) count_global_kernel(
    const uint32_t* __restrict__ tids, int64_t ld, ChunkGeom geom, int64_t g0, int64_t ngb,
    const uint16_t* __restrict__ items, int k, int64_t C, unsigned long long* __restrict__ out) {
    // work item = (candidate, block of 32 groups)
    int64_t total = C * ngb;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = w / ngb, b = w - c * ngb;
        int64_t gb = g0 + b * 32;
        const uint16_t* it = items + c * (int64_t)k;
        uint32_t cnt = 0;
        for (int q = 0; q < 8; ++q) {
            int64_t g = gb + q * 4;
            if (g > geom.g_last || g + 3 < geom.g_first) continue;
            uint4 a = make_uint4(group_mask(geom, g), group_mask(geom, g + 1),
                                 group_mask(geom, g + 2), group_mask(geom, g + 3));
            for (int j = 0; j < k; ++j)
                a = and4(a, __ldg(reinterpret_cast<const uint4*>(tids + (int64_t)__ldg(it + j) * ld + g)));
            cnt += popc4(a);
        }
        if (cnt) atomicAdd(out + c, (unsigned long long)cnt);
    }
}

// Launch geometry shared by the API entry and the engine.
struct CountPlan {
    int P = 1;
    int64_t g0 = 0, tiles = 0, csplit = 1, cands_per_cta = 0;
    size_t smem = 0;
    bool staged = true;
};

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

CountPlan plan_count(int m, ChunkGeom geom, int64_t C) {
    CountPlan pl;
    pl.g0 = geom.g_first & ~31LL;
    const int64_t span = geom.g_last + 1 - pl.g0;  // groups from the aligned base
    const size_t plane = (size_t)m * 128;
    const int smax = max_dyn_smem();
    if (plane > (size_t)smax) {
        pl.staged = false;
        return pl;
    }
    pl.P = 1;
    pl.tiles = (span + 31) / 32;
    pl.smem = plane;
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)(228 * 1024) / (plane + 1024)));
    const int64_t target = (int64_t)sm_count() * per_sm * 2;
    int64_t cs = (target + pl.tiles - 1) / pl.tiles;
    // keep at least ~2 candidates per thread per CTA so the staging amortises
    const int64_t min_cpc = 2 * kCountThreads;
    int64_t cs_max = std::max<int64_t>(1, (C + min_cpc - 1) / min_cpc);
    cs = std::max<int64_t>(1, std::min<int64_t>(cs, cs_max));
    cs = std::min<int64_t>(cs, 65535);
    pl.csplit = cs;
    pl.cands_per_cta = (C + cs - 1) / cs;
    return pl;
}

template <int K>
static int launch_count_tile(const CountPlan& pl, const uint32_t* tids, int64_t ld, int m,
                             ChunkGeom geom, const uint16_t* items, int k, int64_t C,
                             unsigned long long* out, cudaStream_t s) {
    static bool attr_done = false;
    if (!attr_done) {
        DIC_CUDA(cudaFuncSetAttribute(count_tile_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_dyn_smem()));
        attr_done = true;
    }
    // grid.x may exceed 2^31-1 only for absurd n; tiles is bounded by ld/32
    dim3 grid((unsigned)pl.tiles, (unsigned)pl.csplit);
    count_tile_kernel<K><<<grid, kCountThreads, pl.smem, s>>>(tids, ld, m, pl.P, geom, pl.g0, items, k,
                                                             C, pl.cands_per_cta, out);
    DIC_CHECK_LAUNCH("count_tile_kernel");
    return DIC_OK;
}

int count_support_launch(const uint32_t* tids, int64_t ld, int m, int64_t first, int64_t last,
                         const uint16_t* items, int k, int64_t C, unsigned long long* out,
                         cudaStream_t s) {
    if (C <= 0 || last < first) return DIC_OK;
    ChunkGeom geom = chunk_geom(first, last);
    CountPlan pl = plan_count(m, geom, C);
    if (!pl.staged) {
        int64_t ngb = (geom.g_last + 1 - pl.g0 + 31) / 32;
        int64_t total = C * ngb;
        int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
        count_global_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
            tids, ld, geom, pl.g0, ngb, items, k, C, out);
        DIC_CHECK_LAUNCH("count_global_kernel");
        return DIC_OK;
    }
    switch (k) {
        case 1: return launch_count_tile<1>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 2: return launch_count_tile<2>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 3: return launch_count_tile<3>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 4: return launch_count_tile<4>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 5: return launch_count_tile<5>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 6: return launch_count_tile<6>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 7: return launch_count_tile<7>(pl, tids, ld, m, geom, items, k, C, out, s);
        case 8: return launch_count_tile<8>(pl, tids, ld, m, geom, items, k, C, out, s);
        default: return launch_count_tile<0>(pl, tids, ld, m, geom, items, k, C, out, s);
    }
}

int item_support_launch(const uint32_t* tids, int64_t ld, int m, int64_t first, int64_t last,
                        unsigned long long* counts, cudaStream_t s) {
    if (last < first) return DIC_OK;
    ChunkGeom geom = chunk_geom(first, last);
    int64_t gb = geom.g_first & ~3LL;
    int64_t span = geom.g_last + 1 - gb;
    // aim for ~4 waves of 256-thread CTAs over m x splits
    int64_t want = (int64_t)sm_count() * 8;
    int64_t splits = std::max<int64_t>(1, (want + m - 1) / m);
    int64_t per = (span + splits - 1) / splits;
    per = std::max<int64_t>(per, 4 * 256);
    per = (per + 3) & ~3LL;
    splits = (span + per - 1) / per;
    splits = std::min<int64_t>(std::max<int64_t>(splits, 1), 65535);
    dim3 grid((unsigned)m, (unsigned)splits);
    item_support_kernel<<<grid, 256, 0, s>>>(tids, ld, geom, per, counts);
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
    __shared__ unsigned long long sm_masks[kRowCands * (W > 0 ? W : 16)];
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
                        const unsigned long long* masks, int64_t C, unsigned long long* out,
                        cudaStream_t s) {
    count_rows_kernel<W><<<grid, 256, 0, s>>>(rows, Wd, first, last, masks, C, out);
}

}  // namespace dic

using namespace dic;

extern "C" int dic_item_support(const uint32_t* tids, int64_t ld, int32_t m, int64_t first,
                                int64_t last, int64_t* counts, void* stream) {
    DIC_REQUIRE(m >= 1 && ld % 32 == 0, "dic_item_support: bad m=%d or ld=%lld", m, (long long)ld);
    DIC_REQUIRE(first >= 0 && (last < first || (last >> 5) < ld),
                "dic_item_support: chunk [%lld, %lld] outside ld=%lld groups", (long long)first,
                (long long)last, (long long)ld);
    return item_support_launch(tids, ld, m, first, last,
                               reinterpret_cast<unsigned long long*>(counts), as_stream(stream));
}

extern "C" int dic_count_support(const uint32_t* tids, int64_t ld, int32_t m, int64_t first,
                                 int64_t last, const uint16_t* items, int32_t k, int64_t C,
                                 uint64_t* support_inc, void* stream) {
    DIC_REQUIRE(m >= 1 && m <= 65535, "dic_count_support: m=%d outside [1, 65535]", m);
    DIC_REQUIRE(k >= 1 && k <= m, "dic_count_support: k=%d outside [1, m=%d]", k, m);
    DIC_REQUIRE(ld % 32 == 0, "dic_count_support: ld=%lld not a multiple of 32", (long long)ld);
    DIC_REQUIRE(0 <= first && first <= last && (last >> 5) < ld,
                "chunk [%lld, %lld] outside database", (long long)first, (long long)last);
    DIC_REQUIRE(C >= 0, "dic_count_support: C=%lld < 0", (long long)C);
    return count_support_launch(tids, ld, m, first, last, items, k, C,
                                reinterpret_cast<unsigned long long*>(support_inc), as_stream(stream));
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
            DIC_REQUIRE(W <= 16, "dic_count_support_rows: W=%d > 16 unsupported", W);
            launch_rows<0>(grid, r, W, first, last, mk, C, o, s);
    }
    DIC_CHECK_LAUNCH("count_rows_kernel");
    return DIC_OK;
}
