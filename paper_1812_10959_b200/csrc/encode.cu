// encode.cu — the transaction-bitmap encoder (CSR item lists -> row bitmap)
// and the row bitmap -> bit-sliced (item-major) transform.
//
// Reference: encode_transaction (bitops.py:24-37) ORs 1<<item per id and
// raises ItemOutOfRange(item) for an id outside the universe; BitDatabase
// (database.py:13-86) stores one uint64 per row.  Here a row is W uint64
// words (LSW first) and the whole database is encoded in one launch.
#include "common.cuh"

namespace dic {

// One thread per row: OR the row's ids into its W words held in registers
// (W <= 16; wider rows fall back to atomicOr on the zeroed output), count the
// duplicates (len - popcount) and record the first out-of-range id in
// row-major order (atomicMin on the CSR position, which orders rows first and
// then positions within a row — exactly the id encode_transaction would raise
// on first).
template <int W>
__global__ void __launch_bounds__(256) encode_csr_kernel(const int64_t* __restrict__ indptr,
                                                         const int32_t* __restrict__ indices, int64_t n, int32_t m,
                                                         int Wd, unsigned long long* __restrict__ rows,
                                                         unsigned long long* __restrict__ status) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long dup = 0;
    if (r < n) {
        const int64_t b = indptr[r], e = indptr[r + 1];
        int64_t bad = -1;
        if constexpr (W > 0) {
            unsigned long long acc[W];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = 0;
            int64_t nvalid = 0;
            for (int64_t q = b; q < e; ++q) {
                const int32_t it = __ldg(indices + q);
                if (it < 0 || it >= m) {
                    if (bad < 0) bad = q;
                    continue;
                }
                ++nvalid;
                const unsigned long long bit = 1ull << (it & 63);
                const int wi = it >> 6;
#pragma unroll
                for (int w = 0; w < W; ++w)
                    if (w == wi) acc[w] |= bit;  // static register index
            }
            int64_t bits = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                rows[r * W + w] = acc[w];
                bits += __popcll(acc[w]);
            }
            dup = (unsigned long long)(nvalid - bits);
        } else {
            unsigned long long* row = rows + r * (int64_t)Wd;  // zeroed by the caller
            for (int64_t q = b; q < e; ++q) {
                const int32_t it = indices[q];
                if (it < 0 || it >= m) {
                    if (bad < 0) bad = q;
                    continue;
                }
                atomicOr(row + (it >> 6), 1ull << (it & 63));
            }
        }
        if (bad >= 0) atomicMin(status + 1, (unsigned long long)bad);
    }
    if constexpr (W > 0) {
        for (int o = 16; o > 0; o >>= 1) dup += __shfl_down_sync(0xFFFFFFFFu, dup, o);
        if ((threadIdx.x & 31) == 0 && dup) atomicAdd(status, dup);
    }
}

__global__ void dedup_count_kernel(const int64_t* __restrict__ indptr, int64_t n, int W,
                                   const unsigned long long* __restrict__ rows,
                                   unsigned long long* __restrict__ status) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long dup = 0;
    if (r < n) {
        int64_t len = indptr[r + 1] - indptr[r];
        int64_t bits = 0;
        for (int w = 0; w < W; ++w) bits += __popcll(rows[r * (int64_t)W + w]);
        dup = (unsigned long long)(len - bits);
    }
    // warp-aggregate before the global atomic
    for (int o = 16; o > 0; o >>= 1) dup += __shfl_down_sync(0xFFFFFFFFu, dup, o);
    if ((threadIdx.x & 31) == 0 && dup) atomicAdd(status, dup);
}

__global__ void init_status_kernel(unsigned long long* status) {
    status[0] = 0;
    status[1] = ~0ull;  // "no bad id" sentinel, mapped to -1 below
    status[2] = ~0ull;
    status[3] = 0;
}

__global__ void finish_status_kernel(const int64_t* __restrict__ indptr, int64_t n,
                                     unsigned long long* status) {
    // translate the bad position into its row (binary search over indptr)
    if (status[1] == ~0ull) return;
    int64_t pos = (int64_t)status[1];
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (indptr[mid] <= pos) lo = mid; else hi = mid - 1;
    }
    // skip empty rows that share the same start
    status[2] = (unsigned long long)lo;
}

// Rows -> tiled bit-sliced copy.  A CTA owns one tile (TW groups = TW*32
// rows) and one 64-item word column at a time: warp w transposes groups
// w, w+8, ... with 64 ballots per group (bit b of lane l's word -> bit l of
// column b), stages the 64 x TW result in shared memory and writes the 64
// item rows of the tile with consecutive
// threads on consecutive words.
__global__ void __launch_bounds__(256) rows_to_tids_kernel(
    const unsigned long long* __restrict__ rows, int64_t n, int32_t m, int W, int TW,
    uint32_t* __restrict__ tids) {
    __shared__ uint32_t stage[64][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t = blockIdx.x;
    const int64_t g0 = t * TW;
    uint32_t* tile = tids + t * (int64_t)m * row_words(TW);
    for (int wb = 0; wb < W; ++wb) {
        for (int gl = warp; gl < TW; gl += 8) {
            int64_t r = (g0 + gl) * 32 + lane;
            unsigned long long x = r < n ? rows[r * (int64_t)W + wb] : 0ull;
            uint32_t lo_col = 0, hi_col = 0;
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                uint32_t v = __ballot_sync(0xFFFFFFFFu, (uint32_t)(x >> b) & 1u);
                if (lane == b) lo_col = v;
            }
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                uint32_t v = __ballot_sync(0xFFFFFFFFu, (uint32_t)(x >> (32 + b)) & 1u);
                if (lane == b) hi_col = v;
            }
            stage[lane][gl] = lo_col;
            stage[32 + lane][gl] = hi_col;
        }
        __syncthreads();
        const int items = min(64, m - wb * 64);
        const int RW = row_words(TW);
        for (int idx = threadIdx.x; idx < items * RW; idx += 256) {
            int il = idx / RW, slot = idx - il * RW;
            tile[(int64_t)(wb * 64 + il) * RW + slot] = slot < TW ? stage[il][slot] : 0u;
        }
        __syncthreads();
    }
}

// CSR item lists -> bit-sliced tiles directly, for tiles [t_begin, t_end).
// A CTA builds one tile image at a time in shared memory (zeroed, then one
// warp per row OR-ing the row's bit into each item's group word with a
// shared-memory atomic — the returned old word flags duplicates), then
// streams the image to HBM with 16-byte stores.  Tiles
// too large for shared memory are built in place with global atomics.
// Ids are uint16 or int32 (IDX); the first out-of-range id in row-major order
// is recorded as in encode_csr_kernel.
constexpr int kEncThreads = 512;
template <typename IDX>
__global__ void __launch_bounds__(kEncThreads) encode_tids_kernel(const int64_t* __restrict__ indptr,
                                                                  const IDX* __restrict__ indices, int64_t n,
                                                                  int32_t m, int64_t t_begin, int64_t t_end,
                                                                  uint32_t* __restrict__ tids,
                                                                  unsigned long long* __restrict__ status,
                                                                  int use_smem) {
    extern __shared__ __align__(16) uint32_t img[];
    const int TW = tile_groups(m), RW = row_words(TW);
    const int64_t tw = (int64_t)m * RW;  // multiple of 4 (RW is)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kEncThreads / 32;
    unsigned long long dup = 0;
    for (int64_t t = t_begin + blockIdx.x; t < t_end; t += gridDim.x) {
        uint32_t* dst = use_smem ? img : tids + t * tw;
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        for (int64_t i = threadIdx.x; i < tw / 4; i += kEncThreads) d4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        const int64_t r0 = t * TW * 32, r1 = min(n, r0 + (int64_t)TW * 32);
        for (int64_t r = r0 + warp; r < r1; r += nwarps) {
            const int64_t b = __ldg(indptr + r), e = __ldg(indptr + r + 1);
            const int gl = (int)((r - r0) >> 5);
            const uint32_t bit = 1u << (r & 31);
            for (int64_t q = b + lane; q < e; q += 32) {
                const int64_t it = (int64_t)__ldg(indices + q);
                if (it < 0 || it >= m) {
                    atomicMin(status + 1, (unsigned long long)q);
                    continue;
                }
                const uint32_t old = atomicOr(dst + it * RW + gl, bit);
                dup += (old & bit) ? 1u : 0u;
            }
        }
        __syncthreads();
        if (use_smem) {
            uint4* o4 = reinterpret_cast<uint4*>(tids + t * tw);
            for (int64_t i = threadIdx.x; i < tw / 4; i += kEncThreads) o4[i] = d4[i];
            __syncthreads();
        }
    }
    for (int o = 16; o > 0; o >>= 1) dup += __shfl_down_sync(0xFFFFFFFFu, dup, o);
    if (lane == 0 && dup) atomicAdd(status, dup);
}

// Bit-sliced tiles -> row bitmap (the inverse transform; the host view of a
// database encoded straight to tiles).  Thread per (row, 64-bit word).
__global__ void tids_to_rows_kernel(const uint32_t* __restrict__ tids, int64_t n, int32_t m, int W,
                                    unsigned long long* __restrict__ rows) {
    const int TW = tile_groups(m);
    const int64_t total = n * W;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = x / W;
        const int w = (int)(x - r * W);
        const int64_t g = r >> 5;
        const uint32_t sh = (uint32_t)(r & 31);
        unsigned long long v = 0;
        const int top = min(64, m - w * 64);
        for (int b = 0; b < top; ++b)
            v |= (unsigned long long)((__ldg(tids + tids_index(m, TW, (uint32_t)(w * 64 + b), g)) >> sh) & 1u) << b;
        rows[x] = v;
    }
}

}  // namespace dic

using namespace dic;

extern "C" int dic_encode_status_init(int64_t* status, void* stream) {
    DIC_REQUIRE(status, "dic_encode_status_init: null status");
    init_status_kernel<<<1, 1, 0, as_stream(stream)>>>(reinterpret_cast<unsigned long long*>(status));
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("init_status_kernel");
    return DIC_OK;
}

extern "C" int dic_encode_status_finish(const int64_t* indptr, int64_t n, int64_t* status, void* stream) {
    DIC_REQUIRE(indptr && status && n >= 1, "dic_encode_status_finish: bad arguments");
    finish_status_kernel<<<1, 1, 0, as_stream(stream)>>>(indptr, n, reinterpret_cast<unsigned long long*>(status));
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("finish_status_kernel");
    return DIC_OK;
}

extern "C" int dic_encode_csr_tids(const int64_t* indptr, const void* indices, int32_t index_bytes, int64_t n,
                                   int32_t m, int64_t row_begin, int64_t row_end, uint32_t* tids, int64_t* status,
                                   void* stream) {
    DIC_REQUIRE(n >= 1 && m >= 1 && m <= 65535, "dic_encode_csr_tids: need n >= 1 and 1 <= m <= 65535");
    DIC_REQUIRE(indptr && tids && status && (indices || row_end <= row_begin), "dic_encode_csr_tids: null pointer");
    DIC_REQUIRE(index_bytes == 2 || index_bytes == 4, "dic_encode_csr_tids: index_bytes must be 2 or 4, got %d",
                index_bytes);
    const int64_t rows_per_tile = (int64_t)tile_groups(m) * 32;
    DIC_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= n && row_begin % rows_per_tile == 0 &&
                    (row_end % rows_per_tile == 0 || row_end == n),
                "dic_encode_csr_tids: rows [%lld, %lld) must be tile-aligned (%lld rows) within %lld",
                (long long)row_begin, (long long)row_end, (long long)rows_per_tile, (long long)n);
    if (row_end == row_begin) return DIC_OK;
    cudaStream_t s = as_stream(stream);
    const int64_t t_begin = row_begin / rows_per_tile, t_end = (row_end + rows_per_tile - 1) / rows_per_tile;
    const size_t img = (size_t)tile_words(m) * 4;
    static int max_smem = 0;
    if (!max_smem) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        DIC_CUDA(cudaFuncSetAttribute(encode_tids_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_smem));
        DIC_CUDA(cudaFuncSetAttribute(encode_tids_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      max_smem));
    }
    const int use_smem = img <= (size_t)max_smem ? 1 : 0;
    const size_t smem = use_smem ? img : 0;
    // persistent: resident CTAs only (shared-memory bound), tiles strided over them
    const int per_sm = use_smem ? std::max(1, (int)((size_t)(228 * 1024) / (img + 1024))) : 4;
    const int64_t grid = std::min<int64_t>(t_end - t_begin, (int64_t)sm_count() * per_sm);
    auto* st = reinterpret_cast<unsigned long long*>(status);
    if (index_bytes == 2)
        encode_tids_kernel<uint16_t><<<(unsigned)grid, kEncThreads, smem, s>>>(
            indptr, static_cast<const uint16_t*>(indices), n, m, t_begin, t_end, tids, st, use_smem);
    else
        encode_tids_kernel<int32_t><<<(unsigned)grid, kEncThreads, smem, s>>>(
            indptr, static_cast<const int32_t*>(indices), n, m, t_begin, t_end, tids, st, use_smem);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("encode_tids_kernel");
    return DIC_OK;
}

extern "C" int dic_tids_to_rows(const uint32_t* tids, int64_t n, int32_t m, uint64_t* rows, void* stream) {
    DIC_REQUIRE(n >= 1 && m >= 1 && tids && rows, "dic_tids_to_rows: need n >= 1, m >= 1 and buffers");
    const int W = (m + 63) / 64;
    const int64_t total = n * W;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
    tids_to_rows_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, as_stream(stream)>>>(
        tids, n, m, W, reinterpret_cast<unsigned long long*>(rows));
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("tids_to_rows_kernel");
    return DIC_OK;
}

extern "C" int dic_encode_csr(const int64_t* indptr, const int32_t* indices, int64_t n,
                              int32_t m, uint64_t* rows, int64_t* status, void* stream) {
    DIC_REQUIRE(n >= 0 && m >= 1, "dic_encode_csr: need n >= 0 and m >= 1 (n=%lld, m=%d)",
                (long long)n, m);
    DIC_REQUIRE(indptr && rows && status, "dic_encode_csr: null pointer");
    cudaStream_t s = as_stream(stream);
    const int W = (m + 63) / 64;
    auto* st = reinterpret_cast<unsigned long long*>(status);
    init_status_kernel<<<1, 1, 0, s>>>(st); ::dic::note_launch();
    if (n == 0) { DIC_CHECK_LAUNCH("init_status_kernel"); return DIC_OK; }
    const int T = 256;
    const int64_t blocks = (n + T - 1) / T;
    auto* out = reinterpret_cast<unsigned long long*>(rows);
    switch (W) {
#define DIC_ENC(WW) \
        case WW: encode_csr_kernel<WW><<<(unsigned)blocks, T, 0, s>>>(indptr, indices, n, m, W, out, st); break;
        DIC_ENC(1) DIC_ENC(2) DIC_ENC(3) DIC_ENC(4) DIC_ENC(5) DIC_ENC(6) DIC_ENC(7) DIC_ENC(8)
        DIC_ENC(9) DIC_ENC(10) DIC_ENC(11) DIC_ENC(12) DIC_ENC(13) DIC_ENC(14) DIC_ENC(15) DIC_ENC(16)
#undef DIC_ENC
        default:
            DIC_CUDA(cudaMemsetAsync(rows, 0, (size_t)n * W * sizeof(uint64_t), s));
            encode_csr_kernel<0><<<(unsigned)blocks, T, 0, s>>>(indptr, indices, n, m, W, out, st);
            ::dic::note_launch();
            dedup_count_kernel<<<(unsigned)blocks, T, 0, s>>>(indptr, n, W, out, st);
    }
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("encode_csr_kernel");
    finish_status_kernel<<<1, 1, 0, s>>>(indptr, n, st); ::dic::note_launch();
    DIC_CHECK_LAUNCH("finish_status_kernel");
    return DIC_OK;
}

extern "C" int dic_rows_to_tids(const uint64_t* rows, int64_t n, int32_t m, uint32_t* tids, void* stream) {
    DIC_REQUIRE(n >= 1 && m >= 1 && rows && tids, "dic_rows_to_tids: need n >= 1, m >= 1 and buffers");
    const int W = (m + 63) / 64;
    const int TW = tile_groups(m);
    const int64_t tiles = tile_count(n, m);
    rows_to_tids_kernel<<<(unsigned)tiles, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const unsigned long long*>(rows), n, m, W, TW, tids); ::dic::note_launch();
    DIC_CHECK_LAUNCH("rows_to_tids_kernel");
    return DIC_OK;
}
