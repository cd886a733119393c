// containment.cu — the pattern containment matrix of DicMiner.transform
// (estimator.py:90-99): entry (j, p) says pattern p's items all occur in
// transaction j, i.e. (row_j & mask_p) == mask_p.
//
// On the bit-sliced tiles this is one AND per (pattern item, 32-row group):
// lane p of a warp owns pattern p of a 32-pattern block and walks the groups
// of one tile, AND-ing the words of its items (all in the same L2-resident
// tile image); the 32 row bits of the result are then either stored as one
// word (packed output, [G][P] words, consecutive lanes -> consecutive
// words) or spread over 32 bytes of the row-major bool matrix (consecutive
// lanes -> consecutive bytes of a row).  The dense form is bound by its n*P
// output bytes; the packed form by the item-word reads.
#include "common.cuh"

namespace dic {

template <bool DENSE>
__global__ void __launch_bounds__(256) containment_kernel(const uint32_t* __restrict__ tids, int64_t n, int32_t m,
                                                          const uint16_t* __restrict__ items,
                                                          const int64_t* __restrict__ offs, int64_t P,
                                                          uint8_t* __restrict__ dense, uint32_t* __restrict__ packed) {
    const int TW = tile_groups(m), RW = row_words(TW);
    const int64_t tiles = tile_count(n, m);
    const int64_t PB = (P + 31) / 32;
    const int64_t G = (n + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; u < tiles * PB; u += warps) {
        const int64_t t = u / PB, pb = u - t * PB;
        const int64_t p = pb * 32 + lane;
        const bool valid = p < P;
        int64_t kb = 0, ke = 0;
        bool possible = valid;
        if (valid) {
            kb = offs[p];
            ke = offs[p + 1];
            for (int64_t q = kb; q < ke; ++q) possible &= (int32_t)items[q] < m;  // item outside this universe
        }
        const uint32_t* tile = tids + t * (int64_t)m * RW;
        for (int gl = 0; gl < TW; ++gl) {
            const int64_t g = t * TW + gl;
            if (g >= G) break;
            uint32_t w = possible ? 0xFFFFFFFFu : 0u;
            if (possible)
                for (int64_t q = kb; q < ke; ++q) w &= __ldg(tile + (int64_t)items[q] * RW + gl);
            const int64_t r0 = g * 32;
            if (r0 + 32 > n) w &= (n - r0 >= 32) ? 0xFFFFFFFFu : ((1u << (uint32_t)(n - r0)) - 1u);
            if constexpr (DENSE) {
                if (valid) {
                    const int rows = n - r0 < 32 ? (int)(n - r0) : 32;
                    for (int r = 0; r < rows; ++r) dense[(r0 + r) * P + p] = (uint8_t)((w >> r) & 1u);
                }
            } else {
                if (valid) packed[g * P + p] = w;
            }
        }
    }
}

}  // namespace dic

using namespace dic;

static int containment_launch(const uint32_t* tids, int64_t n, int32_t m, const uint16_t* items, const int64_t* offs,
                              int64_t P, uint8_t* dense, uint32_t* packed, void* stream, const char* who) {
    DIC_REQUIRE(n >= 1 && m >= 1 && m <= 65535 && P >= 0 && tids && offs && (dense || packed),
                "%s: bad arguments (n=%lld, m=%d, P=%lld)", who, (long long)n, m, (long long)P);
    if (P == 0) return DIC_OK;
    const int64_t units = tile_count(n, m) * ((P + 31) / 32);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((units + 7) / 8, (int64_t)sm_count() * 16));
    cudaStream_t s = as_stream(stream);
    if (dense)
        containment_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(tids, n, m, items, offs, P, dense, nullptr);
    else
        containment_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(tids, n, m, items, offs, P, nullptr, packed);
    ::dic::note_launch();
    DIC_CHECK_LAUNCH("containment_kernel");
    return DIC_OK;
}

extern "C" int dic_containment(const uint32_t* tids, int64_t n, int32_t m, const uint16_t* items, const int64_t* offs,
                               int64_t P, uint8_t* out, void* stream) {
    return containment_launch(tids, n, m, items, offs, P, out, nullptr, stream, "dic_containment");
}

extern "C" int dic_containment_packed(const uint32_t* tids, int64_t n, int32_t m, const uint16_t* items,
                                      const int64_t* offs, int64_t P, uint32_t* out, void* stream) {
    return containment_launch(tids, n, m, items, offs, P, nullptr, out, stream, "dic_containment_packed");
}
