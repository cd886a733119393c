// barlab — cost of a grid-wide barrier among co-resident CTAs (one per SM,
// 1,024 threads), the building block of the fused checkpoint kernel.
//   V0  __threadfence(); atomicAdd; volatile spin; __threadfence()   (fence.sc.gpu twice)
//   V1  atom.add.release.gpu; ld.acquire.gpu spin                    (no full fence)
//   V2  V1 with every CTA spinning on its own copy written by the last arriver (fan-out)
// Also: the "last CTA out" pattern, and the empty-kernel launch-to-launch time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/lab/barlab tools/lab/barlab.cu && ./tools/lab/barlab
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            printf("%s: %s\n", #x, cudaGetErrorString(e_));                           \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void bar_v0(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1ull);
        while (*(volatile unsigned long long*)ctr < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ void bar_v1(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(1024, 1) bar_kernel(unsigned long long* ctr, int nbar, unsigned long long* out,
                                                      unsigned long long* data) {
    const unsigned long long G = gridDim.x;
    unsigned long long t0 = 0;
    for (int i = 0; i < nbar; ++i) {
        // a little traffic before each barrier, like a phase would leave
        data[(size_t)blockIdx.x * 1024 + threadIdx.x] = i;
        if (i == 1 && threadIdx.x == 0) t0 = gtime();
        if (V == 0) bar_v0(ctr, G * (i + 1));
        else bar_v1(ctr, G * (i + 1));
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = gtime() - t0;
}

// Dependent-load chain after a grid barrier (data written by another SM just
// before it), and straight-line code executed cold vs warm.
template <int N>
__device__ __noinline__ unsigned long long big_code(unsigned long long x) {
    // N independent-looking but sequentially dependent ALU ops, fully unrolled:
    // ~N*3 instructions of straight-line code
#pragma unroll
    for (int i = 0; i < N; ++i) x = (x ^ (x >> 7)) * 0x9E3779B97F4A7C15ull + i;
    return x;
}

// 8 independent chains: issue-bound when warm, fetch-bound when cold
template <int N, int SALT>
__device__ __noinline__ unsigned long long wide_code(unsigned long long x) {
    unsigned v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = (unsigned)x + q + SALT;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (v[q] ^ (v[q] >> 7)) + (unsigned)(i * 8 + q + SALT);
    }
    unsigned long long r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) r += v[q];
    return r;
}

__global__ void __launch_bounds__(1024, 1) evict_kernel(unsigned long long* p) {
    // a different large body, run by every warp of every SM
    unsigned long long x = wide_code<600, 7>(p[0] + threadIdx.x);
    if (x == 12345) p[1] = x;
}

__global__ void __launch_bounds__(1024, 1) icache_kernel(unsigned long long* p, unsigned long long* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long t0 = gtime();
        unsigned long long x = wide_code<150, 1>(p[0]);
        unsigned long long t1 = gtime();
        unsigned long long y = wide_code<150, 1>(x);
        unsigned long long t2 = gtime();
        out[4] = t1 - t0;
        out[5] = (t2 - t1) + (y == 12345);
    }
}

__global__ void __launch_bounds__(1024, 1) chain_kernel(unsigned long long* ctr, unsigned long long* chain, int n,
                                                        unsigned long long* out) {
    const unsigned long long G = gridDim.x;
    // every CTA writes the chain links owned by it: link i -> (i * 7919 + 1) % n
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        chain[i] = (unsigned long long)((i * 7919ll + 1) % n);
    bar_v0(ctr, G);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t0 = gtime();
        unsigned long long j = 0;
        for (int i = 0; i < 16; ++i) j = chain[j];
        unsigned long long t1 = gtime();
        out[1] = (t1 - t0) + (j == 0xFFFFFFFFull);
        // cold vs warm straight-line code
        t0 = gtime();
        unsigned long long x = big_code<512>(j);
        t1 = gtime();
        unsigned long long y = big_code<512>(x);
        unsigned long long t2 = gtime();
        out[2] = t1 - t0;
        out[3] = (t2 - t1) + (y == 12345);
    }
}

__global__ void __launch_bounds__(1024, 1) empty_kernel(unsigned long long* p) {
    if (p[0] == 12345) p[1] = 1;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    unsigned long long *ctr, *out, *data;
    CK(cudaMalloc(&ctr, 64));
    CK(cudaMalloc(&out, 64));
    CK(cudaMalloc(&data, (size_t)sms * 1024 * 8));
    const int nbar = 101;
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemset(ctr, 0, 64));
            void* args[] = {&ctr, (void*)&nbar, &out, &data};
            if (v == 0) CK(cudaLaunchCooperativeKernel((const void*)bar_kernel<0>, dim3(sms), dim3(1024), args, 0, 0));
            else CK(cudaLaunchCooperativeKernel((const void*)bar_kernel<1>, dim3(sms), dim3(1024), args, 0, 0));
            CK(cudaDeviceSynchronize());
            unsigned long long ns = 0;
            CK(cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost));
            printf("V%d: %d CTAs x 1024: %.3f us per barrier\n", v, sms, ns / 1e3 / (nbar - 1));
        }
    }
    {
        const int n = 1 << 20;
        unsigned long long* chain;
        CK(cudaMalloc(&chain, (size_t)n * 8));
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemset(ctr, 0, 64));
            // evict code / data caches with the other kernel
            empty_kernel<<<sms, 1024>>>(ctr);
            void* args[] = {&ctr, &chain, (void*)&n, &out};
            CK(cudaLaunchCooperativeKernel((const void*)chain_kernel, dim3(sms), dim3(1024), args, 0, 0));
            CK(cudaDeviceSynchronize());
            unsigned long long h[4];
            CK(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
            printf("post-barrier dependent L2 load: %.3f us per level; 512-step unrolled code: cold %.3f us, warm %.3f us\n",
                   h[1] / 1e3 / 16, h[2] / 1e3, h[3] / 1e3);
        }
    }
    for (int rep = 0; rep < 3; ++rep) {
        evict_kernel<<<sms, 1024>>>(ctr);
        icache_kernel<<<sms, 1024>>>(ctr, out);
        CK(cudaDeviceSynchronize());
        unsigned long long h[6];
        CK(cudaMemcpy(h, out, 48, cudaMemcpyDeviceToHost));
        printf("3600 straight-line instructions (one warp): cold %.3f us, warm %.3f us\n", h[4] / 1e3, h[5] / 1e3);
    }
    // back-to-back tiny kernels: stream launches and a graph of 100
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0, s));
        for (int i = 0; i < 200; ++i) empty_kernel<<<sms, 1024, 0, s>>>(ctr);
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("stream: %.3f us per tiny kernel (148 x 1024)\n", ms * 1e3 / 200);
    }
    cudaGraph_t g;
    cudaGraphExec_t gx;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < 100; ++i) empty_kernel<<<sms, 1024, 0, s>>>(ctr);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&gx, g, 0));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0, s));
        CK(cudaGraphLaunch(gx, s));
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("graph: %.3f us per tiny kernel (100 in one graph)\n", ms * 1e3 / 100);
    }
    return 0;
}
