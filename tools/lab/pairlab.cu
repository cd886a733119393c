// pairlab.cu — standalone timing lab for the dense pair-triangle kernel
// (csrc/pairs.cu).  Builds bit-sliced tiles of a cfg4-shaped chunk (m items,
// 100k rows, TW = 16), runs kernel variants, checks every variant's triangle
// against the first one and prints per-variant time, rate and the spread of
// per-CTA finish times.  Not part of the library; tools only.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -o pairlab tools/lab/pairlab.cu && ./pairlab [m] [rows]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lop3_maj(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lop3_and(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, 0, 0xC0;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// acc += sum_w popc(a_w & b_w), 8 words; MODE 0: IADD3 combine (current),
// 1: IMAD combine with a runtime 1 (moves the adds to the FMA pipe)
template <int MODE>
__device__ __forceinline__ uint32_t and_popc8(uint4 a0, uint4 a1, uint4 b0, uint4 b1, uint32_t acc, uint32_t one) {
    const uint32_t x0 = lop3_and(a0.x, b0.x), x1 = lop3_and(a0.y, b0.y), x2 = lop3_and(a0.z, b0.z);
    const uint32_t x3 = lop3_and(a0.w, b0.w), x4 = lop3_and(a1.x, b1.x), x5 = lop3_and(a1.y, b1.y);
    const uint32_t x6 = lop3_and(a1.z, b1.z), x7 = lop3_and(a1.w, b1.w);
    const uint32_t s1 = lop3_xor3(x0, x1, x2), c1 = lop3_maj(x0, x1, x2);
    const uint32_t s2 = lop3_xor3(x3, x4, x5), c2 = lop3_maj(x3, x4, x5);
    const uint32_t s3 = lop3_xor3(s1, s2, x6), c3 = lop3_maj(s1, s2, x6);
    const uint32_t t = lop3_xor3(c1, c2, c3), f = lop3_maj(c1, c2, c3);
    if (MODE == 0) return acc + __popc(s3) + __popc(x7) + 2u * __popc(t) + 4u * __popc(f);
    acc = imad(__popc(s3), one, acc);
    acc = imad(__popc(x7), one, acc);
    acc = imad(__popc(t), 2u, acc);
    return imad(__popc(f), 4u, acc);
}

constexpr int kBlk = 64;
constexpr int kThreads = 256;

__host__ __device__ inline int64_t tri_index(int64_t a, int64_t b, int64_t m) {
    return a * m - a * (a + 1) / 2 + (b - a - 1);
}
struct PB {
    int a0, b0, na, nb;
    bool diag;
};
__device__ __forceinline__ PB pair_block(int64_t bi, int nblk, int m) {
    int y = (int)bi, I = 0;
    while (y >= nblk - I) {
        y -= nblk - I;
        ++I;
    }
    PB p;
    p.a0 = I * kBlk;
    p.b0 = (I + y) * kBlk;
    p.na = min(kBlk, m - p.a0);
    p.nb = min(kBlk, m - p.b0);
    p.diag = y == 0;
    return p;
}

struct Geo {
    int64_t g_first, g_last;
    uint32_t first_mask, last_mask;
};
__device__ __forceinline__ uint32_t group_mask(const Geo& c, int64_t g) {
    uint32_t mk = (g < c.g_first || g > c.g_last) ? 0u : 0xFFFFFFFFu;
    if (g == c.g_first) mk &= c.first_mask;
    if (g == c.g_last) mk &= c.last_mask;
    return mk;
}

// the 4x4 register tile over one 8-word step; SKIP: warp-uniform skips of
// register groups with no valid pair (diagonal i > j; rows past na / nb)
template <int MODE, bool SKIP>
__device__ __forceinline__ void tile_step(const uint8_t* A, const uint8_t* B, int RB, int ta, int tb, int q,
                                          uint32_t (&cnt)[4][4], uint32_t one, uint32_t live) {
    uint4 av0[4], av1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        av0[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + q * 16);
        av1[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + q * 16 + 16);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 bv0 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + q * 16);
        const uint4 bv1 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + q * 16 + 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (SKIP && !((live >> (4 * i + j)) & 1u)) continue;
            cnt[i][j] = and_popc8<MODE>(av0[i], av1[i], bv0, bv1, cnt[i][j], one);
        }
    }
}

// V: 0 = reference structure (2 stages, __syncthreads per tile)
//    1 = STAGES-deep ring with per-stage empty barriers (no __syncthreads)
template <int TW, int MINB, int MODE, bool SKIP, int STAGES, bool RING>
__global__ void __launch_bounds__(kThreads, MINB)
    pair_kernel(const uint32_t* __restrict__ tids, int m, Geo geom, int64_t t_first, int64_t t_last, int nblk,
                unsigned long long* __restrict__ tri, uint32_t one, uint64_t* __restrict__ ctime) {
    constexpr int RW = TW + 4;
    constexpr int RB = RW * 4;
    constexpr uint32_t BLK = kBlk * RB;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 8;
    uint8_t* buf = smem + 128;
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x] = gtimer();

    const int64_t tile_words = (int64_t)m * RW;
    const int64_t nt = t_last - t_first + 1;
    const int64_t U = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const int64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;

    auto issue = [&](int64_t u, int s) {
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        const PB pb = pair_block(bi, nblk, m);
        const uint32_t ab = (uint32_t)pb.na * RB, bb = (uint32_t)pb.nb * RB;
        uint8_t* dst = buf + (size_t)s * 2 * BLK;
        const uint32_t* src = tids + t * tile_words;
        mbar_expect_tx(&full[s], ab + (pb.diag ? 0u : bb));
        bulk_g2s(dst, src + (int64_t)pb.a0 * RW, ab, &full[s]);
        if (!pb.diag) bulk_g2s(dst + BLK, src + (int64_t)pb.b0 * RW, bb, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kThreads / 32);
        }
        fence_mbar_init();
        for (int s = 0; s < STAGES && u0 + s < u1; ++s) issue(u0 + s, s);
    }
    __syncthreads();

    const int ta = threadIdx.x & 15, tb = threadIdx.x >> 4;
    const int lane = threadIdx.x & 31;
    uint32_t cnt[4][4];
    int64_t cur = -1;
    PB pb{0, 0, 0, 0, true};
    auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int a = pb.a0 + ta + 16 * i, b = pb.b0 + tb + 16 * j;
                if (a < b && b < m && cnt[i][j]) atomicAdd(tri + tri_index(a, b, m), (unsigned long long)cnt[i][j]);
            }
    };
    uint32_t live = 0xFFFFu;  // register groups (i, j) holding a valid pair: bit 4i+j
    for (int64_t u = u0; u < u1; ++u) {
        const int64_t it = u - u0;
        const int s = (int)(it % STAGES);
        const uint32_t ph = (uint32_t)((it / STAGES) & 1);
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        if (bi != cur) {
            if (cur >= 0) flush();
            cur = bi;
            pb = pair_block(bi, nblk, m);
            live = 0;
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j)
                    if (16 * i < pb.na && 16 * j < pb.nb && !(pb.diag && i > j)) live |= 1u << (4 * i + j);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) cnt[i][j] = 0;
        }
        mbar_wait(&full[s], ph);
        uint8_t* A = buf + (size_t)s * 2 * BLK;
        uint8_t* B = pb.diag ? A : A + BLK;
        if (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last) {
            const int rows = pb.diag ? pb.na : 2 * kBlk;
            for (int idx = threadIdx.x; idx < rows * RW; idx += kThreads) {
                const int r = idx / RW, slot = idx - r * RW;
                if (slot >= TW || (r < kBlk ? r >= pb.na : r - kBlk >= pb.nb)) continue;
                uint32_t* w = reinterpret_cast<uint32_t*>(A + (size_t)r * RB) + slot;
                *w &= group_mask(geom, t * TW + slot);
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < TW / 4; q += 2) {
            tile_step<MODE, SKIP>(A, B, RB, ta, tb, q, cnt, one, live);
        }
        if (!RING) {
            __syncthreads();
            if (threadIdx.x == 0 && u + STAGES < u1) {
                fence_proxy_async();
                issue(u + STAGES, s);
            }
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (threadIdx.x == 0 && u + STAGES < u1) {
                mbar_wait(&empty[s], ph);
                fence_proxy_async();
                issue(u + STAGES, s);
            }
        }
    }
    flush();
    if (threadIdx.x == 0 && ctime) {
        ctime[2 * blockIdx.x + 1] = gtimer();
    }
}


// compile-time diagonal specialisation: register groups i > j of a diagonal
// block hold no pair (a = ta + 16i >= 16i > tb + 16j), so they are not emitted
template <int MODE, bool DIAG>
__device__ __forceinline__ void tile_step_d(const uint8_t* A, const uint8_t* B, int RB, int ta, int tb, int q,
                                            uint32_t (&cnt)[4][4], uint32_t one) {
    uint4 av0[4], av1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        av0[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + q * 16);
        av1[i] = *reinterpret_cast<const uint4*>(A + (ta + 16 * i) * RB + q * 16 + 16);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 bv0 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + q * 16);
        const uint4 bv1 = *reinterpret_cast<const uint4*>(B + (tb + 16 * j) * RB + q * 16 + 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (DIAG && i > j) continue;
            cnt[i][j] = and_popc8<MODE>(av0[i], av1[i], bv0, bv1, cnt[i][j], one);
        }
    }
}

// Lockstep warp groups: one CTA per SM of G x 256 threads; step k hands unit
// u0 + kG + g to group g, every group consumes its unit of the same stage and
// the whole CTA syncs per step, so no group runs ahead or starves at the end.
template <int TW, int G, int MODE, bool DSPEC, int STAGES>
__global__ void __launch_bounds__(kThreads* G, 1)
    pair_kernel_grp(const uint32_t* __restrict__ tids, int m, Geo geom, int64_t t_first, int64_t t_last, int nblk,
                    unsigned long long* __restrict__ tri, uint32_t one, uint64_t* __restrict__ ctime) {
    constexpr int RW = TW + 4;
    constexpr int RB = RW * 4;
    constexpr uint32_t BLK = kBlk * RB;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint8_t* buf = smem + 128;
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x] = gtimer();
    const int64_t tile_words = (int64_t)m * RW;
    const int64_t nt = t_last - t_first + 1;
    const int64_t U = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const int64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;
    const int64_t steps = (u1 - u0 + G - 1) / G;
    auto issue = [&](int64_t k, int s) {
        uint32_t bytes = 0;
        for (int g = 0; g < G; ++g) {
            const int64_t u = u0 + k * G + g;
            if (u >= u1) break;
            const int64_t bi = u / nt;
            const PB pb = pair_block(bi, nblk, m);
            bytes += (uint32_t)pb.na * RB + (pb.diag ? 0u : (uint32_t)pb.nb * RB);
        }
        mbar_expect_tx(&full[s], bytes);
        for (int g = 0; g < G; ++g) {
            const int64_t u = u0 + k * G + g;
            if (u >= u1) break;
            const int64_t bi = u / nt;
            const int64_t t = t_first + (u - bi * nt);
            const PB pb = pair_block(bi, nblk, m);
            uint8_t* dst = buf + ((size_t)s * G + g) * 2 * BLK;
            const uint32_t* src = tids + t * tile_words;
            bulk_g2s(dst, src + (int64_t)pb.a0 * RW, (uint32_t)pb.na * RB, &full[s]);
            if (!pb.diag) bulk_g2s(dst + BLK, src + (int64_t)pb.b0 * RW, (uint32_t)pb.nb * RB, &full[s]);
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int s = 0; s < STAGES && s < steps; ++s) issue(s, s);
    }
    __syncthreads();
    const int grp = threadIdx.x / kThreads, tid = threadIdx.x % kThreads;
    const int ta = tid & 15, tb = tid >> 4;
    uint32_t cnt[4][4];
    int64_t cur = -1;
    PB pb{0, 0, 0, 0, true};
    auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int a = pb.a0 + ta + 16 * i, b = pb.b0 + tb + 16 * j;
                if (a < b && b < m && cnt[i][j]) atomicAdd(tri + tri_index(a, b, m), (unsigned long long)cnt[i][j]);
            }
    };
    for (int64_t k = 0; k < steps; ++k) {
        const int s = (int)(k % STAGES);
        const uint32_t ph = (uint32_t)((k / STAGES) & 1);
        const int64_t u = u0 + k * G + grp;
        const bool mine = u < u1;
        int64_t t = 0;
        if (mine) {
            const int64_t bi = u / nt;
            t = t_first + (u - bi * nt);
            if (bi != cur) {
                if (cur >= 0) flush();
                cur = bi;
                pb = pair_block(bi, nblk, m);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) cnt[i][j] = 0;
            }
        }
        mbar_wait(&full[s], ph);
        uint8_t* A = buf + ((size_t)s * G + grp) * 2 * BLK;
        uint8_t* B = pb.diag ? A : A + BLK;
        // any edge tile in this step: every thread evaluates the same predicate
        bool edge = false;
        for (int g = 0; g < G; ++g) {
            const int64_t v = u0 + k * G + g;
            if (v >= u1) break;
            const int64_t tv = t_first + (v - (v / nt) * nt);
            edge |= (tv * TW <= geom.g_first || tv * TW + TW - 1 >= geom.g_last);
        }
        if (edge) {
            if (mine && (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last)) {
                const int rows = pb.diag ? pb.na : 2 * kBlk;
                for (int idx = tid; idx < rows * RW; idx += kThreads) {
                    const int r = idx / RW, slot = idx - r * RW;
                    if (slot >= TW || (r < kBlk ? r >= pb.na : r - kBlk >= pb.nb)) continue;
                    uint32_t* w = reinterpret_cast<uint32_t*>(A + (size_t)r * RB) + slot;
                    *w &= group_mask(geom, t * TW + slot);
                }
            }
            __syncthreads();
        }
        if (mine) {
            if (DSPEC && pb.diag) {
#pragma unroll
                for (int q = 0; q < TW / 4; q += 2) tile_step_d<MODE, true>(A, B, RB, ta, tb, q, cnt, one);
            } else {
#pragma unroll
                for (int q = 0; q < TW / 4; q += 2) tile_step_d<MODE, false>(A, B, RB, ta, tb, q, cnt, one);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && k + STAGES < steps) {
            fence_proxy_async();
            issue(k + STAGES, s);
        }
    }
    if (cur >= 0) flush();
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x + 1] = gtimer();
}

// Dynamic grains: CTAs claim runs of GR units from a global counter (thread 0,
// when its issue cursor runs dry); the unit of each stage travels in smem.
// The first SF percent of the units are split statically (contiguous ranges,
// few flushes), the rest is claimed dynamically (tight tail).  Register tile
// TI x TJ per thread: a = ta + SA*i, b = tb + SB*j with SA = 64/TI,
// SB = 64/TJ; threads = SA * SB.
template <int MODE, bool DIAG, int TI, int TJ>
__device__ __forceinline__ void tile_step_g(const uint8_t* A, const uint8_t* B, int RB, int ta, int tb, int q,
                                            uint32_t (&cnt)[TI][TJ], uint32_t one) {
    constexpr int SA = 64 / TI, SB = 64 / TJ;
    uint4 av0[TI], av1[TI];
#pragma unroll
    for (int i = 0; i < TI; ++i) {
        av0[i] = *reinterpret_cast<const uint4*>(A + (ta + SA * i) * RB + q * 16);
        av1[i] = *reinterpret_cast<const uint4*>(A + (ta + SA * i) * RB + q * 16 + 16);
    }
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
        const uint4 bv0 = *reinterpret_cast<const uint4*>(B + (tb + SB * j) * RB + q * 16);
        const uint4 bv1 = *reinterpret_cast<const uint4*>(B + (tb + SB * j) * RB + q * 16 + 16);
#pragma unroll
        for (int i = 0; i < TI; ++i) {
            if (DIAG && SA * i >= SB * (j + 1)) continue;
            cnt[i][j] = and_popc8<MODE>(av0[i], av1[i], bv0, bv1, cnt[i][j], one);
        }
    }
}

template <int TW, int MINB, int MODE, bool DSPEC, int STAGES, int GR, int TI, int TJ, int SF>
__global__ void __launch_bounds__((64 / TI) * (64 / TJ), MINB)
    pair_kernel_dyn(const uint32_t* __restrict__ tids, int m, Geo geom, int64_t t_first, int64_t t_last, int nblk,
                    unsigned long long* __restrict__ tri, uint32_t one, uint64_t* __restrict__ ctime,
                    unsigned long long* __restrict__ ctr) {
    constexpr int NT = (64 / TI) * (64 / TJ);
    constexpr int SA = 64 / TI, SB = 64 / TJ;
    constexpr int RW = TW + 4;
    constexpr int RB = RW * 4;
    constexpr uint32_t BLK = kBlk * RB;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    int64_t* sunit = reinterpret_cast<int64_t*>(smem + 64);
    uint8_t* buf = smem + 128;
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x] = gtimer();
    const int64_t tile_words = (int64_t)m * RW;
    const int64_t nt = t_last - t_first + 1;
    const int64_t U = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const int64_t US = U * SF / 100;  // statically split prefix
    int64_t icur = US * blockIdx.x / gridDim.x, iend = US * (blockIdx.x + 1) / gridDim.x;
    auto next_unit = [&]() -> int64_t {
        if (icur == iend) {
            const int64_t g = (int64_t)atomicAdd(ctr, 1ull);
            icur = US + g * GR;
            iend = icur + GR < U ? icur + GR : U;
            if (icur >= U) {
                icur = iend = U;
                return -1;
            }
        }
        return icur++;
    };
    auto issue = [&](int64_t u, int s) {
        sunit[s] = u;
        if (u < 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
            return;
        }
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        const PB pb = pair_block(bi, nblk, m);
        const uint32_t ab = (uint32_t)pb.na * RB, bb = (uint32_t)pb.nb * RB;
        uint8_t* dst = buf + (size_t)s * 2 * BLK;
        const uint32_t* src = tids + t * tile_words;
        mbar_expect_tx(&full[s], ab + (pb.diag ? 0u : bb));
        bulk_g2s(dst, src + (int64_t)pb.a0 * RW, ab, &full[s]);
        if (!pb.diag) bulk_g2s(dst + BLK, src + (int64_t)pb.b0 * RW, bb, &full[s]);
    };
    bool done_issuing = false;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int s = 0; s < STAGES; ++s) {
            const int64_t u = done_issuing ? -1 : next_unit();
            if (u < 0) done_issuing = true;
            issue(u, s);
        }
    }
    __syncthreads();
    const int ta = threadIdx.x % SA, tb = threadIdx.x / SA;
    uint32_t cnt[TI][TJ];
    int64_t cur = -1;
    PB pb{0, 0, 0, 0, true};
    auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TJ; ++j) {
                const int a = pb.a0 + ta + SA * i, b = pb.b0 + tb + SB * j;
                if (a < b && b < m && cnt[i][j]) atomicAdd(tri + tri_index(a, b, m), (unsigned long long)cnt[i][j]);
            }
    };
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % STAGES);
        const uint32_t ph = (uint32_t)((k / STAGES) & 1);
        mbar_wait(&full[s], ph);
        const int64_t u = sunit[s];
        if (u < 0) break;
        const int64_t bi = u / nt;
        const int64_t t = t_first + (u - bi * nt);
        if (bi != cur) {
            if (cur >= 0) flush();
            cur = bi;
            pb = pair_block(bi, nblk, m);
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < TJ; ++j) cnt[i][j] = 0;
        }
        uint8_t* A = buf + (size_t)s * 2 * BLK;
        uint8_t* B = pb.diag ? A : A + BLK;
        if (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last) {
            const int rows = pb.diag ? pb.na : 2 * kBlk;
            for (int idx = threadIdx.x; idx < rows * RW; idx += NT) {
                const int r = idx / RW, slot = idx - r * RW;
                if (slot >= TW || (r < kBlk ? r >= pb.na : r - kBlk >= pb.nb)) continue;
                uint32_t* w = reinterpret_cast<uint32_t*>(A + (size_t)r * RB) + slot;
                *w &= group_mask(geom, t * TW + slot);
            }
            __syncthreads();
        }
        if (DSPEC && pb.diag) {
#pragma unroll
            for (int q = 0; q < TW / 4; q += 2) tile_step_g<MODE, true, TI, TJ>(A, B, RB, ta, tb, q, cnt, one);
        } else {
#pragma unroll
            for (int q = 0; q < TW / 4; q += 2) tile_step_g<MODE, false, TI, TJ>(A, B, RB, ta, tb, q, cnt, one);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_proxy_async();
            const int64_t nu = done_issuing ? -1 : next_unit();
            if (nu < 0) done_issuing = true;
            issue(nu, s);
        }
    }
    if (cur >= 0) flush();
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x + 1] = gtimer();
}

// v2: the producer decodes each unit once (block pair, tile, edge) into a
// per-stage descriptor in shared memory, so consumers do no 64-bit division;
// TPS units per stage (one barrier per TPS tiles); dynamic grains.
struct UnitDesc {
    int64_t bi;   // block pair (-1: no unit)
    int64_t t;    // tile
    int a0, b0, na, nb;
    int diag, edge;
};

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

template <int TW, int MINB, int MODE, int STAGES, int GR, int TPS, int SF, int Q = 0>
__global__ void __launch_bounds__(kThreads, MINB)
    pair_kernel_v2(const uint32_t* __restrict__ tids, int m, Geo geom, int64_t t_first, int64_t t_last, int nblk,
                   unsigned long long* __restrict__ tri, uint32_t one, uint64_t* __restrict__ ctime,
                   unsigned long long* __restrict__ ctr) {
    constexpr int RW = TW + 4;
    constexpr int RB = RW * 4;
    constexpr uint32_t BLK = kBlk * RB;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);                        // [STAGES]
    UnitDesc* desc = reinterpret_cast<UnitDesc*>(smem + 64);                   // [STAGES][TPS]
    uint8_t* buf = smem + 64 + ((STAGES * TPS * sizeof(UnitDesc) + 127) / 128) * 128;
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x] = gtimer();
    const int64_t tile_words = (int64_t)m * RW;
    const int64_t nt = t_last - t_first + 1;
    const int64_t U = (int64_t)nblk * (nblk + 1) / 2 * nt;
    const int64_t US = U * SF / 100;
    int64_t icur = Q ? 0 : US * blockIdx.x / gridDim.x, iend = Q ? 0 : US * (blockIdx.x + 1) / gridDim.x;
    bool dry = false;
    // Q = 1: the units are split into nsm contiguous ranges; the CTAs resident
    // on SM s claim GR units at a time from range s (ctr[s]), then steal
    // from the following ranges, so co-resident CTAs share one range
    const int nsm = Q ? (int)gridDim.x / MINB : 1;
    const int home = Q ? (int)(smid() % (uint32_t)nsm) : 0;
    int ridx = 0;
    auto next_unit_q = [&]() -> int64_t {
        if (dry) return -1;
        if (icur == iend) {
            for (;;) {
                if (ridx >= nsm) {
                    dry = true;
                    return -1;
                }
                const int r = (home + ridx) % nsm;
                const int64_t rb = U * r / nsm, re = U * (r + 1) / nsm;
                const int64_t g = (int64_t)atomicAdd(ctr + r, (unsigned long long)GR);
                if (rb + g < re) {
                    icur = rb + g;
                    iend = icur + GR < re ? icur + GR : re;
                    break;
                }
                ++ridx;
            }
        }
        return icur++;
    };
    auto next_unit = [&]() -> int64_t {
        if (Q) return next_unit_q();
        if (dry) return -1;
        if (icur == iend) {
            const int64_t g = (int64_t)atomicAdd(ctr, 1ull);
            icur = US + g * GR;
            iend = icur + GR < U ? icur + GR : U;
            if (icur >= U) {
                dry = true;
                return -1;
            }
        }
        return icur++;
    };
    // thread 0: fill stage s with up to TPS units; returns false when none
    auto issue = [&](int s) {
        uint32_t bytes = 0;
        UnitDesc* d = desc + s * TPS;
        int64_t us[TPS];
        for (int k = 0; k < TPS; ++k) {
            us[k] = next_unit();
            if (us[k] < 0) {
                d[k].bi = -1;
                continue;
            }
            const int64_t bi = us[k] / nt;
            const int64_t t = t_first + (us[k] - bi * nt);
            const PB pb = pair_block(bi, nblk, m);
            d[k].bi = bi;
            d[k].t = t;
            d[k].a0 = pb.a0;
            d[k].b0 = pb.b0;
            d[k].na = pb.na;
            d[k].nb = pb.nb;
            d[k].diag = pb.diag;
            d[k].edge = (t * TW <= geom.g_first || t * TW + TW - 1 >= geom.g_last);
            bytes += (uint32_t)pb.na * RB + (pb.diag ? 0u : (uint32_t)pb.nb * RB);
        }
        if (bytes == 0) {
            mbar_arrive(&full[s]);
            return;
        }
        mbar_expect_tx(&full[s], bytes);
        for (int k = 0; k < TPS; ++k) {
            if (us[k] < 0) continue;
            uint8_t* dst = buf + ((size_t)s * TPS + k) * 2 * BLK;
            const uint32_t* src = tids + d[k].t * tile_words;
            bulk_g2s(dst, src + (int64_t)d[k].a0 * RW, (uint32_t)d[k].na * RB, &full[s]);
            if (!d[k].diag) bulk_g2s(dst + BLK, src + (int64_t)d[k].b0 * RW, (uint32_t)d[k].nb * RB, &full[s]);
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int s = 0; s < STAGES; ++s) issue(s);
    }
    __syncthreads();
    const int ta = threadIdx.x & 15, tb = threadIdx.x >> 4;
    uint32_t cnt[4][4];
    int64_t cur = -1;
    int a0 = 0, b0 = 0;
    auto flush = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int a = a0 + ta + 16 * i, b = b0 + tb + 16 * j;
                if (a < b && b < m && cnt[i][j]) atomicAdd(tri + tri_index(a, b, m), (unsigned long long)cnt[i][j]);
            }
    };
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % STAGES);
        const uint32_t ph = (uint32_t)((k / STAGES) & 1);
        mbar_wait(&full[s], ph);
        const UnitDesc* d = desc + s * TPS;
        if (d[0].bi < 0) break;
        bool anyedge = false;
#pragma unroll
        for (int e = 0; e < TPS; ++e) anyedge |= (d[e].bi >= 0 && d[e].edge);
        if (anyedge) {
            for (int e = 0; e < TPS; ++e) {
                if (d[e].bi < 0 || !d[e].edge) continue;
                uint8_t* A = buf + ((size_t)s * TPS + e) * 2 * BLK;
                const int rows = d[e].diag ? d[e].na : 2 * kBlk;
                for (int idx = threadIdx.x; idx < rows * RW; idx += kThreads) {
                    const int r = idx / RW, slot = idx - r * RW;
                    if (slot >= TW || (r < kBlk ? r >= d[e].na : r - kBlk >= d[e].nb)) continue;
                    uint32_t* w = reinterpret_cast<uint32_t*>(A + (size_t)r * RB) + slot;
                    *w &= group_mask(geom, d[e].t * TW + slot);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int e = 0; e < TPS; ++e) {
            const int64_t bi = d[e].bi;
            if (bi < 0) break;
            const int diag = d[e].diag;
            if (bi != cur) {
                if (cur >= 0) flush();
                cur = bi;
                a0 = d[e].a0;
                b0 = d[e].b0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) cnt[i][j] = 0;
            }
            const uint8_t* A = buf + ((size_t)s * TPS + e) * 2 * BLK;
            const uint8_t* B = diag ? A : A + BLK;
            if (diag) {
#pragma unroll
                for (int q = 0; q < TW / 4; q += 2) tile_step_d<MODE, true>(A, B, RB, ta, tb, q, cnt, one);
            } else {
#pragma unroll
                for (int q = 0; q < TW / 4; q += 2) tile_step_d<MODE, false>(A, B, RB, ta, tb, q, cnt, one);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_proxy_async();
            issue(s);
        }
    }
    if (cur >= 0) flush();
    if (threadIdx.x == 0 && ctime) ctime[2 * blockIdx.x + 1] = gtimer();
}

struct Ctx {
    const uint32_t* tids;
    int m;
    Geo g;
    int64_t t_first, t_last;
    unsigned long long* tri;
    int64_t tri_len;
    std::vector<unsigned long long> ref;
    int reps;
    double ops;
    unsigned long long* ctr;
    int nsm;
};

template <class L>
float run(const char* name, Ctx& c, unsigned grid, int per_sm, L launch) {
    uint64_t* ctime;
    CK(cudaMalloc(&ctime, 16 * (size_t)grid));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < c.reps; ++r) {
        CK(cudaMemset(c.tri, 0, 8 * c.tri_len));
        CK(cudaMemset(c.ctr, 0, 8 * 1024));
        cudaEventRecord(e0);
        launch(ctime);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    std::vector<unsigned long long> h(c.tri_len);
    CK(cudaMemcpy(h.data(), c.tri, 8 * c.tri_len, cudaMemcpyDeviceToHost));
    bool ok = true;
    if (c.ref.empty())
        c.ref = h;
    else
        ok = (c.ref == h);
    std::vector<uint64_t> ct(2 * grid);
    CK(cudaMemcpy(ct.data(), ctime, 16 * (size_t)grid, cudaMemcpyDeviceToHost));
    uint64_t t0 = ~0ull;
    std::vector<double> ends;
    for (unsigned b = 0; b < grid; ++b) t0 = std::min(t0, ct[2 * b]);
    for (unsigned b = 0; b < grid; ++b) ends.push_back((ct[2 * b + 1] - t0) * 1e-3);
    std::sort(ends.begin(), ends.end());
    printf("%-34s grid %4u (%d/SM) %8.1f us  %.3e lane-ops/s (%.3f of 1.85e13)  CTA end p0 %.0f p10 %.0f p50 %.0f p90 %.0f max %.0f  %s\n",
           name, grid, per_sm, best * 1e3, c.ops / (best * 1e-3), c.ops / (best * 1e-3) / 1.851e13, ends[0],
           ends[grid / 10], ends[grid / 2], ends[grid * 9 / 10], ends.back(), ok ? "OK" : "MISMATCH");
    cudaFree(ctime);
    return best;
}

template <int TW, int MINB, int MODE, bool SKIP, int STAGES, bool RING>
void run_static(const char* name, Ctx& c) {
    auto kern = pair_kernel<TW, MINB, MODE, SKIP, STAGES, RING>;
    const size_t smem = 128 + (size_t)STAGES * 2 * kBlk * (TW + 4) * 4;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
    const int nblk = (c.m + kBlk - 1) / kBlk;
    const int64_t units = (int64_t)nblk * (nblk + 1) / 2 * (c.t_last - c.t_first + 1);
    const unsigned grid = (unsigned)std::min<int64_t>(units, (int64_t)per_sm * c.nsm);
    run(name, c, grid, per_sm, [&](uint64_t* ct) {
        kern<<<grid, kThreads, smem>>>(c.tids, c.m, c.g, c.t_first, c.t_last, nblk, c.tri, 1u, ct);
    });
}

template <int TW, int G, int MODE, bool DSPEC, int STAGES>
void run_grp(const char* name, Ctx& c) {
    auto kern = pair_kernel_grp<TW, G, MODE, DSPEC, STAGES>;
    const size_t smem = 128 + (size_t)STAGES * G * 2 * kBlk * (TW + 4) * 4;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads * G, smem));
    const int nblk = (c.m + kBlk - 1) / kBlk;
    const unsigned grid = (unsigned)(per_sm * c.nsm);
    run(name, c, grid, per_sm, [&](uint64_t* ct) {
        kern<<<grid, kThreads * G, smem>>>(c.tids, c.m, c.g, c.t_first, c.t_last, nblk, c.tri, 1u, ct);
    });
}

template <int TW, int MINB, int MODE, bool DSPEC, int STAGES, int GR, int TI = 4, int TJ = 4, int SF = 0>
void run_dyn(const char* name, Ctx& c) {
    auto kern = pair_kernel_dyn<TW, MINB, MODE, DSPEC, STAGES, GR, TI, TJ, SF>;
    constexpr int NT = (64 / TI) * (64 / TJ);
    const size_t smem = 128 + (size_t)STAGES * 2 * kBlk * (TW + 4) * 4;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    const int nblk = (c.m + kBlk - 1) / kBlk;
    const unsigned grid = (unsigned)(per_sm * c.nsm);
    run(name, c, grid, per_sm, [&](uint64_t* ct) {
        kern<<<grid, NT, smem>>>(c.tids, c.m, c.g, c.t_first, c.t_last, nblk, c.tri, 1u, ct, c.ctr);
    });
}

template <int TW, int MINB, int MODE, int STAGES, int GR, int TPS, int SF, int Q = 0>
void run_v2(const char* name, Ctx& c) {
    auto kern = pair_kernel_v2<TW, MINB, MODE, STAGES, GR, TPS, SF, Q>;
    const size_t smem = 64 + ((STAGES * TPS * sizeof(UnitDesc) + 127) / 128) * 128 +
                        (size_t)STAGES * TPS * 2 * kBlk * (TW + 4) * 4;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
    const int nblk = (c.m + kBlk - 1) / kBlk;
    const unsigned grid = (unsigned)(per_sm * c.nsm);
    run(name, c, grid, per_sm, [&](uint64_t* ct) {
        kern<<<grid, kThreads, smem>>>(c.tids, c.m, c.g, c.t_first, c.t_last, nblk, c.tri, 1u, ct, c.ctr);
    });
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 1000;
    const int64_t rows = argc > 2 ? atoll(argv[2]) : 100000;
    constexpr int TW = 16;
    const int64_t groups = (rows + 31) / 32;
    const int64_t nt = (groups + TW - 1) / TW;
    const int64_t words = nt * (int64_t)m * (TW + 4);
    std::vector<uint32_t> h(words, 0);
    uint64_t x = 0x1234567ull;
    auto rnd = [&]() {
        x += 0x9E3779B97F4A7C15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    for (int64_t t = 0; t < nt; ++t)
        for (int i = 0; i < m; ++i)
            for (int w = 0; w < TW; ++w) {
                uint64_t a = rnd(), b = rnd();
                h[(t * m + i) * (TW + 4) + w] = (uint32_t)(a & (a >> 32) & b & (b >> 32) & rnd());
            }
    Ctx c;
    uint32_t* d;
    CK(cudaMalloc(&d, 4 * words));
    CK(cudaMemcpy(d, h.data(), 4 * words, cudaMemcpyHostToDevice));
    c.tids = d;
    c.m = m;
    c.tri_len = (int64_t)m * (m - 1) / 2;
    CK(cudaMalloc(&c.tri, 8 * c.tri_len));
    CK(cudaMalloc(&c.ctr, 8 * 1024));
    const int64_t first = 37, last = rows - 1;
    c.g.g_first = first >> 5;
    c.g.g_last = last >> 5;
    c.g.first_mask = 0xFFFFFFFFu << (first & 31);
    const uint32_t lb = (uint32_t)(last & 31);
    c.g.last_mask = lb == 31 ? 0xFFFFFFFFu : ((1u << (lb + 1)) - 1u);
    c.t_first = c.g.g_first / TW;
    c.t_last = c.g.g_last / TW;
    c.ops = 2.0 * c.tri_len * ((last - first + 1) / 32.0);
    c.reps = 7;
    CK(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, 0));
    printf("m %d rows %lld tiles %lld pairs %lld; roofline ops %.3e\n", m, (long long)rows, (long long)nt,
           (long long)c.tri_len, c.ops);
    run_dyn<TW, 3, 1, true, 3, 2, 4, 4, 50>("t44 256thr minb3", c);
    run_dyn<TW, 4, 1, true, 3, 2, 4, 8, 50>("t48 128thr minb4", c);
    run_dyn<TW, 2, 1, true, 3, 2, 2, 4, 50>("t24 512thr minb2", c);
    run_dyn<TW, 2, 1, true, 3, 2, 4, 2, 50>("t42 512thr minb2", c);
    run_dyn<TW, 1, 1, true, 3, 2, 2, 2, 50>("t22 1024thr minb1", c);
    run_dyn<TW, 2, 1, true, 3, 2, 8, 4, 50>("t84 128thr minb2", c);
    return 0;
}
