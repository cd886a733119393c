// async.cuh — PTX helpers for mbarrier-tracked bulk async copies (the TMA
// engine's cp.async.bulk) and small bit-logic helpers shared by the counting
// kernels.
#pragma once

#include "common.cuh"

namespace dic {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
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

// acc + sum_w popc(a_w & b_w) over 8 words with a carry-save tree: 16 LOP3 +
// 4 POPC (7 terms -> ones/twos/fours, plus one leftover word).  The four
// weighted adds go through IMAD with a runtime 1 (`one`), i.e. onto the FMA
// pipe, which the pair kernel otherwise leaves idle, instead of IADD3 on the
// ALU pipe the LOP3s saturate
__device__ __forceinline__ uint32_t imad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t and_popc8_acc(uint4 a0, uint4 a1, uint4 b0, uint4 b1, uint32_t acc,
                                                  uint32_t one) {
    const uint32_t x0 = lop3_and(a0.x, b0.x), x1 = lop3_and(a0.y, b0.y), x2 = lop3_and(a0.z, b0.z);
    const uint32_t x3 = lop3_and(a0.w, b0.w), x4 = lop3_and(a1.x, b1.x), x5 = lop3_and(a1.y, b1.y);
    const uint32_t x6 = lop3_and(a1.z, b1.z), x7 = lop3_and(a1.w, b1.w);
    const uint32_t s1 = lop3_xor3(x0, x1, x2), c1 = lop3_maj(x0, x1, x2);
    const uint32_t s2 = lop3_xor3(x3, x4, x5), c2 = lop3_maj(x3, x4, x5);
    const uint32_t s3 = lop3_xor3(s1, s2, x6), c3 = lop3_maj(s1, s2, x6);
    const uint32_t t = lop3_xor3(c1, c2, c3), f = lop3_maj(c1, c2, c3);
    // (an IADD3 combine measured 1-3 % slower on a cfg4 chunk: tools/lab/pair_ab.sh)
    acc = imad_u32(__popc(s3), one, acc);
    acc = imad_u32(__popc(x7), one, acc);
    acc = imad_u32(__popc(t), 2u, acc);
    return imad_u32(__popc(f), 4u, acc);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t popc4(uint4 v) {
    return __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
}
__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) {
    return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w);
}

}  // namespace dic
