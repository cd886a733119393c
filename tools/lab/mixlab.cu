// mixlab.cu — register-only throughput of the pair-count instruction mixes
// (no shared memory): how close can LOP3 + POPC (+ IMAD) get to the 2
// lane-ops per pair-word roofline when nothing else competes for issue or
// the MIO queue?  Tools only.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lop3_maj(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lop3_and(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, 0, 0xC0;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t popc(uint32_t a) {
    uint32_t d;
    asm volatile("popc.b32 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// MIX 0: 8 AND + 8 CSA LOP3 + 4 POPC + 4 IMAD per 8 words (the kernel's)
// MIX 1: 8 AND + 8 POPC (no CSA)
// MIX 2: as 0 but the combine through IADD (compiler's choice)
template <int MIX>
__device__ __forceinline__ uint32_t step(const uint32_t (&a)[8], const uint32_t (&b)[8], uint32_t acc,
                                         uint32_t one) {
    if (MIX == 1) {
#pragma unroll
        for (int w = 0; w < 8; ++w) acc = imad(popc(lop3_and(a[w], b[w])), one, acc);
        return acc;
    }
    const uint32_t x0 = lop3_and(a[0], b[0]), x1 = lop3_and(a[1], b[1]), x2 = lop3_and(a[2], b[2]);
    const uint32_t x3 = lop3_and(a[3], b[3]), x4 = lop3_and(a[4], b[4]), x5 = lop3_and(a[5], b[5]);
    const uint32_t x6 = lop3_and(a[6], b[6]), x7 = lop3_and(a[7], b[7]);
    const uint32_t s1 = lop3_xor3(x0, x1, x2), c1 = lop3_maj(x0, x1, x2);
    const uint32_t s2 = lop3_xor3(x3, x4, x5), c2 = lop3_maj(x3, x4, x5);
    const uint32_t s3 = lop3_xor3(s1, s2, x6), c3 = lop3_maj(s1, s2, x6);
    const uint32_t t = lop3_xor3(c1, c2, c3), f = lop3_maj(c1, c2, c3);
    if (MIX == 2) return acc + popc(s3) + popc(x7) + 2u * popc(t) + 4u * popc(f);
    acc = imad(popc(s3), one, acc);
    acc = imad(popc(x7), one, acc);
    acc = imad(popc(t), 2u, acc);
    return imad(popc(f), 4u, acc);
}

// each thread: P independent pair chains over registers; the operands are
// rotated every iteration (one LOP3-free register move per word would be
// visible; instead the B words are XOR-perturbed once per 16 steps)
template <int MIX, int P>
__global__ void __launch_bounds__(256) mix_kernel(const uint32_t* in, uint32_t* out, int iters, uint32_t one) {
    uint32_t a[P][8], b[8];
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
        for (int w = 0; w < 8; ++w) a[p][w] = in[(threadIdx.x + p * 8 + w) & 1023];
#pragma unroll
    for (int w = 0; w < 8; ++w) b[w] = in[(threadIdx.x * 3 + w) & 1023];
    uint32_t acc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = step<MIX>(a[p], b, acc[p], one);
#pragma unroll
        for (int w = 0; w < 8; ++w) b[w] = imad(b[w], 0x9E3779B1u, one);
    }
    uint32_t s = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) s += acc[p];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MIX, int P>
void run(const char* name, const uint32_t* in, uint32_t* out, int nsm, int blocks_per_sm) {
    const int iters = 4000;
    const int grid = nsm * blocks_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        mix_kernel<MIX, P><<<grid, 256>>>(in, out, iters, 1u);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    // roofline ops: 2 lane-ops per pair-word, 8 words per step
    const double ops = 2.0 * 8 * P * (double)iters * grid * 256;
    printf("%-28s P=%2d blocks/SM %d: %.3f ms  %.3e lane-ops/s  (%.3f of 1.851e13)  err=%s\n", name, P,
           blocks_per_sm, best, ops / (best * 1e-3), ops / (best * 1e-3) / 1.851e13,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *in, *out;
    cudaMalloc(&in, 4096);
    cudaMalloc(&out, 4 * 148 * 8 * 256);
    uint32_t h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = 0x9E3779B9u * (i + 1);
    cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
    run<0, 16>("csa+imad", in, out, nsm, 3);
    run<0, 16>("csa+imad", in, out, nsm, 4);
    run<0, 8>("csa+imad", in, out, nsm, 4);
    run<0, 8>("csa+imad", in, out, nsm, 6);
    run<2, 16>("csa+iadd", in, out, nsm, 3);
    run<2, 8>("csa+iadd", in, out, nsm, 6);
    run<1, 16>("and+popc", in, out, nsm, 3);
    run<1, 8>("and+popc", in, out, nsm, 6);
    return 0;
}
