// probe.cu — integer-pipe peak probes (the roofline denominators the
// measured-peaks file does not carry) and the device-side cfg5 generator.
#include "common.cuh"

namespace dic {

// 8 independent chains x 16 steps per iteration; the operand registers differ
// per step so ptxas cannot fold consecutive LOP3s into one.
template <int OP>
__global__ void __launch_bounds__(1024) int_pipe_kernel(uint32_t* sink, int64_t iters, uint32_t seed) {
    uint32_t a[8], b[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + 1) + j * 0x9E3779B9u;
#pragma unroll
    for (int u = 0; u < 16; ++u) b[u] = (seed ^ (u * 0x85EBCA6Bu)) + blockIdx.x;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if constexpr (OP == 0) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0xF4;" : "+r"(a[j]) : "r"(b[u]), "r"(b[(u + 5) & 15]));
                } else if constexpr (OP == 1) {
                    asm volatile("popc.b32 %0, %0;" : "+r"(a[j]));
                } else {
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(b[u]));
                }
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) x ^= a[j];
    if (x == 0x12345678u) sink[0] = x;  // data-dependent, practically never true
}

// cfg5 bitmap: bit (row, item) set iff the top 32 bits of a counter-based
// hash of (seed, row, item) fall below p * 2^32.
__global__ void bernoulli_rows_kernel(unsigned long long* rows, int64_t n, int W, int m,
                                      uint32_t thresh, uint64_t key) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = n * W;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx / W;
        int w = (int)(idx - r * W);
        unsigned long long word = 0;
        uint64_t base = key ^ ((uint64_t)r * 0xD1B54A32D192ED03ull);
#pragma unroll 4
        for (int b = 0; b < 64; b += 2) {
            int item = w * 64 + b;
            uint64_t h = mix64(base + (uint64_t)(item >> 1) * 0x9E3779B97F4A7C15ull);
            if (item < m && (uint32_t)(h >> 32) < thresh) word |= 1ull << b;
            if (item + 1 < m && (uint32_t)h < thresh) word |= 1ull << (b + 1);
        }
        rows[idx] = word;
    }
}

}  // namespace dic

using namespace dic;

extern "C" int dic_probe_int_pipe(int op, int blocks, int threads, int64_t iters, uint32_t* sink,
                                  double* lane_ops, float* ms, void* stream) {
    DIC_REQUIRE(op >= 0 && op <= 2, "dic_probe_int_pipe: op must be 0 (LOP3), 1 (POPC), 2 (IADD)");
    DIC_REQUIRE(blocks >= 1 && threads >= 32 && threads <= 1024 && iters >= 1,
                "dic_probe_int_pipe: bad geometry");
    cudaStream_t s = as_stream(stream);
    cudaEvent_t e0, e1;
    DIC_CUDA(cudaEventCreate(&e0));
    DIC_CUDA(cudaEventCreate(&e1));
    DIC_CUDA(cudaEventRecord(e0, s));
    switch (op) {
        case 0: int_pipe_kernel<0><<<blocks, threads, 0, s>>>(sink, iters, 0x1234567u); ::dic::note_launch(); break;
        case 1: int_pipe_kernel<1><<<blocks, threads, 0, s>>>(sink, iters, 0x1234567u); ::dic::note_launch(); break;
        default: int_pipe_kernel<2><<<blocks, threads, 0, s>>>(sink, iters, 0x1234567u); ::dic::note_launch(); break;
    }
    DIC_CHECK_LAUNCH("int_pipe_kernel");
    DIC_CUDA(cudaEventRecord(e1, s));
    DIC_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    DIC_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms) *ms = t;
    if (lane_ops) *lane_ops = (double)blocks * threads * (double)iters * 16.0 * 8.0;
    return DIC_OK;
}

extern "C" int dic_synth_bernoulli_rows(int64_t n, int32_t m, double p, uint64_t seed, uint64_t* rows,
                                        void* stream) {
    DIC_REQUIRE(n >= 1 && m >= 1 && p >= 0.0 && p <= 1.0, "dic_synth_bernoulli_rows: bad n/m/p");
    const int W = (m + 63) / 64;
    double t = p * 4294967296.0;
    uint32_t thresh = t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
    uint64_t key = mix64(seed ^ 0x62657266ull);
    int64_t total = n * W;
    int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 32);
    bernoulli_rows_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<unsigned long long*>(rows), n, W, m, thresh, key); ::dic::note_launch();
    DIC_CHECK_LAUNCH("bernoulli_rows_kernel");
    return DIC_OK;
}
