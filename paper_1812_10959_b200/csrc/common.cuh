// common.cuh — shared plumbing for the DIC B200 kernels: error reporting,
// launch checking and small device helpers.  Internal to libdicb200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>

#include <algorithm>

#include "../../include/dic_b200.h"

namespace dic {

// Thread-local message for dic_last_error().
void set_error(const char* fmt, ...);

inline int cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? DIC_ENOMEM : DIC_ECUDA;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();
void retain_pool();
// Count of kernels this library launched (dic_launch_count()).
void note_launch();
// Adjust that count by n (graphs: kernels captured are noted per graph launch).
void note_launches(long long n);

#define DIC_CHECK_LAUNCH(what)                                   \
    do {                                                         \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return ::dic::cuda_fail(_e, what); \
    } while (0)

#define DIC_CUDA(call)                                           \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) return ::dic::cuda_fail(_e, #call); \
    } while (0)

#define DIC_REQUIRE(cond, ...)                                   \
    do {                                                         \
        if (!(cond)) { ::dic::set_error(__VA_ARGS__); return DIC_EINVAL; } \
    } while (0)

// ----------------------------------------------------------------------------
// Chunk geometry on the bit-sliced layout.  Row j lives in group j>>5, bit
// j&31.  A chunk [first, last] (inclusive, the reference's convention,
// params.py:67-75) touches groups g_first..g_last with partial masks at the
// two ends.
struct ChunkGeom {
    int64_t g_first, g_last;   // inclusive group range
    uint32_t first_mask;       // bits of g_first inside the chunk
    uint32_t last_mask;        // bits of g_last inside the chunk
};

__host__ __device__ inline ChunkGeom chunk_geom(int64_t first, int64_t last) {
    ChunkGeom c;
    c.g_first = first >> 5;
    c.g_last = last >> 5;
    c.first_mask = 0xFFFFFFFFu << (uint32_t)(first & 31);
    uint32_t lb = (uint32_t)(last & 31);
    c.last_mask = lb == 31 ? 0xFFFFFFFFu : ((1u << (lb + 1)) - 1u);
    return c;
}

// Mask of the rows of group g that lie inside the chunk.
__device__ __forceinline__ uint32_t group_mask(const ChunkGeom& c, int64_t g) {
    uint32_t mk = (g < c.g_first || g > c.g_last) ? 0u : 0xFFFFFFFFu;
    if (g == c.g_first) mk &= c.first_mask;
    if (g == c.g_last) mk &= c.last_mask;
    return mk;
}

// ----------------------------------------------------------------------------
// Tiled bit-sliced layout ("tids"; include/dic_b200.h).  A tile holds TW
// row-groups (TW*32 rows) of all m items: item i's TW words form one dense row
// (64 or 128 bytes, no pad, no swizzle), so HBM holds exactly the bitmap's
// bits.  The tile's global image equals its shared-memory image: one bulk copy
// stages it.  Readers keep shared-memory accesses conflict-free by how lanes
// are assigned, not by padding: the row-lane count units give the TW/4 chunks
// of one row to adjacent lanes (a contiguous 64/128-byte segment), and the
// AND/POPC pair kernel and the one-candidate-per-lane unit walk a row's chunks
// in an order rotated by the lane.
constexpr int kRowPad = 0;
__host__ __device__ constexpr int tile_groups(int m) { return m <= 768 ? 32 : 16; }
__host__ __device__ constexpr int row_words(int TW) { return TW + kRowPad; }
__host__ __device__ inline int64_t tile_count(int64_t n, int m) {
    int64_t groups = (n + 31) / 32;
    int TW = tile_groups(m);
    return (groups + TW - 1) / TW;
}
__host__ __device__ inline int64_t tile_words(int m) { return (int64_t)m * row_words(tile_groups(m)); }
// uint32 index of (item, group)
__host__ __device__ inline int64_t tids_index(int m, int TW, uint32_t item, int64_t g) {
    int64_t t = g / TW;
    return t * (int64_t)m * row_words(TW) + (int64_t)item * row_words(TW) + (g - t * TW);
}

// 64-bit mixer (SplitMix64 finalizer, the constants of datasets.py:44-53's
// generator family).  Used for hashing masks and for counter-based RNG.
__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__host__ __device__ inline uint64_t hash_words(const uint64_t* w, int W) {
    uint64_t h = 0x9E3779B97F4A7C15ull * (uint64_t)(W + 1);
    for (int i = 0; i < W; ++i) h = mix64(h ^ (w[i] + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1)));
    return h;
}

}  // namespace dic
