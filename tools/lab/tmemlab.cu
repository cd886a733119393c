// tmemlab.cu — is tensor memory a second operand store for integer bit logic?
// Measures tcgen05.ld (TMEM -> registers) throughput per SM, alone and
// running concurrently with shared-memory LDS.128 traffic, against LDS
// alone.  Tools only.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<1>(uint32_t taddr, uint32_t (&r)[1]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<2>(uint32_t taddr, uint32_t (&r)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// MODE 0: TMEM loads only (all warps); 1: LDS.128 only; 2: half the warps
// TMEM, half LDS; N = columns per tcgen05.ld, D = loads in flight per wait
template <int MODE, int N, int D>
__global__ void __launch_bounds__(512, 1) tmem_kernel(uint32_t* out, int iters, unsigned long long* cycles) {
    __shared__ uint32_t taddr_s;
    extern __shared__ __align__(16) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 16384; i += 512) reinterpret_cast<uint32_t*>(sm)[i] = i * 0x9E3779B9u;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = taddr_s + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    const bool use_tmem = MODE == 0 || (MODE == 2 && (warp & 4) == 0) || (MODE == 3 && warp >= 8);
    const unsigned long long t0 = clock64();
    if (use_tmem) {
        for (int it = 0; it < iters; ++it) {
            uint32_t r[D][N];
#pragma unroll
            for (int d = 0; d < D; ++d) tmem_ld<N>(tbase + (uint32_t)(((it * D + d) * N * 7) & (512 - N)), r[d]);
            tmem_wait_ld();
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int n = 0; n < N; ++n) acc ^= r[d][n];
        }
    } else {
        const uint4* base = reinterpret_cast<const uint4*>(sm);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int d = 0; d < D * N / 4; ++d) {
                // 8-lane groups read one contiguous 128 B row each (conflict-free)
                const uint4 v = base[(((it * 5 + d * 3 + (lane >> 3) * 11) & 127) * 8) + (lane & 7)];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
        }
    }
    const unsigned long long t1 = clock64();
    out[blockIdx.x * 512 + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int MODE, int N, int D>
void run(const char* name, int nsm, uint32_t* out, unsigned long long* cyc) {
    const int iters = 20000;
    auto k = tmem_kernel<MODE, N, D>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<nsm, 512, 65536>>>(out, 10, cyc);
    cudaEventRecord(e0);
    k<<<nsm, 512, 65536>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // bytes per SM per iteration: every warp moves 32 lanes x D x N x 4 B
    const double tmem_w = MODE == 0 ? 16 : ((MODE == 2 || MODE == 3) ? 8 : 0),
                 lds_w = MODE == 1 ? 16 : ((MODE == 2 || MODE == 3) ? 8 : 0);
    const double bytes = (tmem_w + lds_w) * 32.0 * D * N * 4 * iters;
    printf("%-26s N=%d D=%d  %.3f ms  %.1f B/clk/SM (tmem warps %g, lds warps %g)  err=%s\n", name, N, D, ms,
           bytes / (double)c, tmem_w, lds_w, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 4 * 512 * nsm);
    cudaMalloc(&cyc, 8 * nsm);
    run<1, 4, 4>("lds only", nsm, out, cyc);
    run<0, 1, 16>("tmem only x1", nsm, out, cyc);
    run<0, 1, 32>("tmem only x1", nsm, out, cyc);
    run<0, 2, 16>("tmem only x2", nsm, out, cyc);
    run<3, 1, 16>("8 tmem x1 + 8 lds warps", nsm, out, cyc);
    run<3, 1, 32>("8 tmem x1 + 8 lds warps", nsm, out, cyc);
    run<0, 1, 8>("tmem only x1", nsm, out, cyc);
    run<0, 4, 4>("tmem only x4", nsm, out, cyc);
    run<0, 8, 4>("tmem only x8", nsm, out, cyc);
    run<2, 4, 4>("half tmem x4 / half lds", nsm, out, cyc);
    run<2, 8, 4>("half tmem x8 / half lds", nsm, out, cyc);
    return 0;
}
