// mmalab.cu — which tensor path can count the dense pair triangle?
//
// The pair wave (engine.py:165-168) is a Gram matrix X^T X of a 0/1 matrix per
// chunk.  Two tensor-core routes exist on sm_100a for it:
//   * the warp-level binary MMA  mma.sync.m16n8k256 .b1 AND.POPC  (operands
//     are the bit-sliced words themselves: no expansion), and
//   * tcgen05.mma kind::i8 (needs every bit expanded to a byte in shared memory).
// This harness measures the register-only issue rate of the warp-level MMAs
// (b1, s8 m16n8k32, f16 m16n8k16 for scale) per SM so the choice is measured,
// not guessed.  Tools only.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/lab/mmalab tools/lab/mmalab.cu
//   ./tools/lab/mmalab
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int ACC>
__global__ void __launch_bounds__(256) b1_kernel(int iters, int* out) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = (threadIdx.x + 1) * 0x9E3779B9u * (i + 1);
    for (int i = 0; i < 2; ++i) b[i] = (threadIdx.x + 7) * 0x85EBCA6Bu * (i + 3);
    int c[ACC][4];
    for (int j = 0; j < ACC; ++j)
        for (int i = 0; i < 4; ++i) c[j][i] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ACC; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
                "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int j = 0; j < ACC; ++j)
        for (int i = 0; i < 4; ++i) s += c[j][i];
    if (s == 0x12345678) out[0] = s;
}

template <int ACC>
__global__ void __launch_bounds__(256) s8_kernel(int iters, int* out) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = (threadIdx.x + 1) * 0x01010101u * (i + 1);
    for (int i = 0; i < 2; ++i) b[i] = (threadIdx.x + 7) * 0x01010101u * (i + 3);
    int c[ACC][4];
    for (int j = 0; j < ACC; ++j)
        for (int i = 0; i < 4; ++i) c[j][i] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ACC; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 "
                "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int j = 0; j < ACC; ++j)
        for (int i = 0; i < 4; ++i) s += c[j][i];
    if (s == 0x12345678) out[0] = s;
}

template <int ACC>
__global__ void __launch_bounds__(256) f16_kernel(int iters, int* out) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x3C003C00u;
    for (int i = 0; i < 2; ++i) b[i] = 0x3C003C00u;
    float c[ACC][4];
    for (int j = 0; j < ACC; ++j)
        for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ACC; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
                "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
    for (int j = 0; j < ACC; ++j)
        for (int i = 0; i < 4; ++i) s += c[j][i];
    if (s == 1234.5f) out[0] = (int)s;
}

// correctness of the b1 fragment mapping: A 16x256 bits, B 256x8 bits (as
// 8 rows of 256 bits), D[i][j] = popc(A_i & B_j)
__global__ void b1_check(const uint32_t* A /*[16][8]*/, const uint32_t* B /*[8][8]*/, int* D /*[16][8]*/) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    uint32_t a0 = A[g * 8 + t], a1 = A[(g + 8) * 8 + t], a2 = A[g * 8 + t + 4], a3 = A[(g + 8) * 8 + t + 4];
    uint32_t b0 = B[g * 8 + t], b1 = B[g * 8 + t + 4];
    int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    asm volatile(
        "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c0), "+r"(c1), "+r"(c2), "+r"(c3)
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    D[g * 8 + 2 * t] = c0;
    D[g * 8 + 2 * t + 1] = c1;
    D[(g + 8) * 8 + 2 * t] = c2;
    D[(g + 8) * 8 + 2 * t + 1] = c3;
}

template <class K>
static double run(K kern, int blocks, int threads, int iters, int* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(iters / 10, out);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int* out;
    cudaMalloc(&out, 4096);
    // mapping check
    {
        uint32_t hA[128], hB[64];
        uint64_t x = 0x1234567ull;
        for (auto& v : hA) v = (uint32_t)((x = x * 6364136223846793005ull + 1442695040888963407ull) >> 32);
        for (auto& v : hB) v = (uint32_t)((x = x * 6364136223846793005ull + 1442695040888963407ull) >> 32);
        uint32_t *dA, *dB;
        int* dD;
        cudaMalloc(&dA, sizeof(hA));
        cudaMalloc(&dB, sizeof(hB));
        cudaMalloc(&dD, 128 * 4);
        cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
        b1_check<<<1, 32>>>(dA, dB, dD);
        int hD[128];
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 8; ++j) {
                int s = 0;
                for (int w = 0; w < 8; ++w) s += __builtin_popcount(hA[i * 8 + w] & hB[j * 8 + w]);
                bad += s != hD[i * 8 + j];
            }
        printf("b1 fragment mapping (A word t/t+4 of item g, B word t/t+4 of item g): %s (%d mismatches)\n",
               bad ? "WRONG" : "ok", bad);
    }
    const double ghz = clk / 1e6;
    for (int wpb : {4, 8}) {
        for (int per_sm : {1, 2, 4}) {
            const int blocks = sms * per_sm, threads = wpb * 32;
            const int iters = 20000;
            const double warps = (double)blocks * wpb;
            double ms = run(b1_kernel<8>, blocks, threads, iters, out);
            double mma = warps * iters * 8;
            double bitmac = mma * 16 * 8 * 256;
            printf("b1  m16n8k256  warps/SM %2d: %.3f ms  %.3e bit-MAC/s  %.0f bit-MAC/clk/SM (@%.2f GHz max)\n",
                   wpb * per_sm, ms, bitmac / (ms * 1e-3), bitmac / (ms * 1e-3) / sms / (ghz * 1e9), ghz);
            ms = run(s8_kernel<8>, blocks, threads, iters, out);
            double mac = warps * iters * 8 * 16 * 8 * 32;
            printf("s8  m16n8k32   warps/SM %2d: %.3f ms  %.3e MAC/s  %.0f MAC/clk/SM\n", wpb * per_sm, ms,
                   mac / (ms * 1e-3), mac / (ms * 1e-3) / sms / (ghz * 1e9));
            ms = run(f16_kernel<8>, blocks, threads, iters, out);
            mac = warps * iters * 8 * 16 * 8 * 16;
            printf("f16 m16n8k16   warps/SM %2d: %.3f ms  %.3e MAC/s  %.0f MAC/clk/SM\n", wpb * per_sm, ms,
                   mac / (ms * 1e-3), mac / (ms * 1e-3) / sms / (ghz * 1e9));
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
