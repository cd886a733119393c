// encode.cu — the transaction-bitmap encoder (CSR item lists -> row bitmap)
// and the row bitmap -> bit-sliced (item-major) transform.
//
// Reference: encode_transaction (bitops.py:24-37) ORs 1<<item per id and
// raises ItemOutOfRange(item) for an id outside the universe; BitDatabase
// (database.py:13-86) stores one uint64 per row.  Here a row is W uint64
// words (LSW first) and the whole database is encoded in one launch.
#include "common.cuh"

namespace dic {

// One thread per row: OR the row's ids into its W words, count duplicates,
// and record the first out-of-range id in row-major order (atomicMin on the
// CSR position, which orders rows first and then positions within a row —
// exactly the id encode_transaction would raise on first).
__global__ void encode_csr_kernel(const int64_t* __restrict__ indptr,
                                  const int32_t* __restrict__ indices, int64_t n,
                                  int32_t m, int W, unsigned long long* __restrict__ rows,
                                  unsigned long long* __restrict__ status) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t b = indptr[r], e = indptr[r + 1];
    unsigned long long* row = rows + r * (int64_t)W;
    int64_t bad = -1;
    for (int64_t q = b; q < e; ++q) {
        int32_t it = indices[q];
        if (it < 0 || it >= m) {
            if (bad < 0) bad = q;
            continue;
        }
        atomicOr(row + (it >> 6), 1ull << (it & 63));
    }
    if (bad >= 0) atomicMin(status + 1, (unsigned long long)bad);
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

// Rows -> bit-sliced copy.  A CTA owns 32 consecutive groups (1024 rows) and
// one 64-item word column at a time: warp w transposes groups w, w+8, ...
// with 64 ballots per group (bit b of lane l's word -> bit l of column b),
// stages the 64 x 32 result in shared memory and writes each item's 32
// group words as one 128-byte line.
__global__ void __launch_bounds__(256) rows_to_tids_kernel(
    const unsigned long long* __restrict__ rows, int64_t n, int32_t m, int W,
    uint32_t* __restrict__ tids, int64_t ld) {
    __shared__ uint32_t stage[64][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g0 = (int64_t)blockIdx.x * 32;
    for (int wb = 0; wb < W; ++wb) {
        for (int gl = warp; gl < 32; gl += 8) {
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
        // write out: 64 items x 32 groups; thread t -> item t/4.., 8 words
        for (int idx = threadIdx.x; idx < 64 * 32; idx += 256) {
            int il = idx >> 5, gl = idx & 31;
            int item = wb * 64 + il;
            if (item < m && g0 + gl < ld) tids[(int64_t)item * ld + g0 + gl] = stage[il][gl];
        }
        __syncthreads();
    }
}

}  // namespace dic

using namespace dic;

extern "C" int64_t dic_tids_ld(int64_t n) {
    int64_t groups = (n + 31) / 32;
    return ((groups + 31) / 32) * 32;
}

extern "C" int dic_encode_csr(const int64_t* indptr, const int32_t* indices, int64_t n,
                              int32_t m, uint64_t* rows, int64_t* status, void* stream) {
    DIC_REQUIRE(n >= 0 && m >= 1, "dic_encode_csr: need n >= 0 and m >= 1 (n=%lld, m=%d)",
                (long long)n, m);
    DIC_REQUIRE(indptr && rows && status, "dic_encode_csr: null pointer");
    cudaStream_t s = as_stream(stream);
    const int W = (m + 63) / 64;
    auto* st = reinterpret_cast<unsigned long long*>(status);
    init_status_kernel<<<1, 1, 0, s>>>(st);
    if (n == 0) { DIC_CHECK_LAUNCH("init_status_kernel"); return DIC_OK; }
    DIC_CUDA(cudaMemsetAsync(rows, 0, (size_t)n * W * sizeof(uint64_t), s));
    const int T = 256;
    int64_t blocks = (n + T - 1) / T;
    encode_csr_kernel<<<(unsigned)blocks, T, 0, s>>>(indptr, indices, n, m, W,
                                                     reinterpret_cast<unsigned long long*>(rows), st);
    DIC_CHECK_LAUNCH("encode_csr_kernel");
    dedup_count_kernel<<<(unsigned)blocks, T, 0, s>>>(
        indptr, n, W, reinterpret_cast<const unsigned long long*>(rows), st);
    DIC_CHECK_LAUNCH("dedup_count_kernel");
    finish_status_kernel<<<1, 1, 0, s>>>(indptr, n, st);
    DIC_CHECK_LAUNCH("finish_status_kernel");
    return DIC_OK;
}

extern "C" int dic_rows_to_tids(const uint64_t* rows, int64_t n, int32_t m, uint32_t* tids,
                                int64_t ld, void* stream) {
    DIC_REQUIRE(n >= 1 && m >= 1, "dic_rows_to_tids: need n >= 1 and m >= 1");
    DIC_REQUIRE(ld % 32 == 0 && ld * 32 >= n, "dic_rows_to_tids: ld=%lld must be a multiple of 32 covering n=%lld rows",
                (long long)ld, (long long)n);
    cudaStream_t s = as_stream(stream);
    const int W = (m + 63) / 64;
    // words past n inside each item row must read as zero
    DIC_CUDA(cudaMemsetAsync(tids, 0, (size_t)m * ld * sizeof(uint32_t), s));
    int64_t blocks = ld / 32;
    rows_to_tids_kernel<<<(unsigned)blocks, 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(rows), n, m, W, tids, ld);
    DIC_CHECK_LAUNCH("rows_to_tids_kernel");
    return DIC_OK;
}
