// abi.cu — library plumbing of the C ABI: version, thread-local error text,
// device queries, and the API-level candidate admission kernel
// (make_candidates' join + subset test, engine.py:320-369, on a host catalog).
#include "common.cuh"

#include <string.h>

namespace dic {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;

void note_launch() { __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED); }
void note_launches(long long n) { __atomic_fetch_add(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Keep freed stream-ordered allocations in the device pool (the default
// release threshold of 0 hands memory back to the driver at every sync,
// turning each engine's allocations into cudaMalloc calls).
void retain_pool() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done = true;
}

int sm_count() {
    static int cached = -1;
    if (cached < 0) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached = v;
    }
    return cached;
}

// ---------------------------------------------------------------------------
// admission
// ---------------------------------------------------------------------------
constexpr int32_t kEmptySlot = -1;

__global__ void set_clear_kernel(int32_t* ht, int64_t cap) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
         i += (int64_t)gridDim.x * blockDim.x)
        ht[i] = kEmptySlot;
}

__device__ __forceinline__ bool words_eq(const unsigned long long* a, const unsigned long long* b, int W) {
    for (int w = 0; w < W; ++w)
        if (a[w] != b[w]) return false;
    return true;
}

// Insert masks[i] (distinct by the caller's contract; duplicates are kept
// once) into the set.
__global__ void set_insert_kernel(int32_t* ht, uint64_t hmask, const unsigned long long* __restrict__ masks,
                                  int64_t K, int W) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const unsigned long long* mk = masks + i * W;
    uint64_t slot = hash_words(reinterpret_cast<const uint64_t*>(mk), W) & hmask;
    while (true) {
        int32_t prev = atomicCAS(ht + slot, kEmptySlot, (int32_t)i);
        if (prev == kEmptySlot || words_eq(masks + (int64_t)prev * W, mk, W)) return;
        slot = (slot + 1) & hmask;
    }
}

__device__ bool set_contains(const int32_t* ht, uint64_t hmask, const unsigned long long* masks, int W,
                             const unsigned long long* q) {
    uint64_t slot = hash_words(reinterpret_cast<const uint64_t*>(q), W) & hmask;
    while (true) {
        int32_t e = ht[slot];
        if (e == kEmptySlot) return false;
        if (words_eq(masks + (int64_t)e * W, q, W)) return true;
        slot = (slot + 1) & hmask;
    }
}

constexpr int kMaxAdmW = 64;  // masks up to 4096 items in the API-level kernel

__global__ void admission_kernel(const unsigned long long* __restrict__ src, int64_t S,
                                 const int32_t* __restrict__ level1, int64_t L, int W,
                                 const int32_t* known_ht, uint64_t kmask, const unsigned long long* known,
                                 const int32_t* box_ht, uint64_t bmask, const unsigned long long* boxes,
                                 uint8_t* __restrict__ admit) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S * L) return;
    int64_t s = t / L, j = t - s * L;
    int l = level1[j];
    unsigned long long cand[kMaxAdmW];
    for (int w = 0; w < W; ++w) cand[w] = src[s * W + w];
    uint8_t ok = 0;
    if (!((cand[l >> 6] >> (l & 63)) & 1ull)) {
        cand[l >> 6] |= 1ull << (l & 63);
        if (!set_contains(known_ht, kmask, known, W, cand)) {
            ok = 1;
            for (int w = 0; w < W && ok; ++w) {
                unsigned long long x = cand[w];
                while (x && ok) {
                    int b = __ffsll((long long)x) - 1;
                    x &= x - 1;
                    cand[w] ^= 1ull << b;
                    if (!set_contains(box_ht, bmask, boxes, W, cand)) ok = 0;
                    cand[w] ^= 1ull << b;
                }
            }
        }
    }
    admit[t] = ok;
}

static int64_t pow2_at_least(int64_t x) {
    int64_t c = 64;
    while (c < x) c <<= 1;
    return c;
}

}  // namespace dic

using namespace dic;

extern "C" int dic_abi_version(void) { return DIC_ABI_VERSION; }

extern "C" const char* dic_last_error(void) { return g_err; }

extern "C" int dic_device_sm_count(void) { return sm_count(); }

extern "C" int64_t dic_launch_count(void) { return (int64_t)__atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

extern "C" int dic_candidate_admission(const uint64_t* src_masks, int64_t S, const int32_t* level1, int64_t L,
                                       int32_t W, const uint64_t* known_masks, int64_t K,
                                       const uint64_t* box_masks, int64_t B, uint8_t* admit, void* stream) {
    DIC_REQUIRE(W >= 1 && W <= kMaxAdmW, "dic_candidate_admission: W=%d outside [1, %d]", W, kMaxAdmW);
    DIC_REQUIRE(S >= 0 && L >= 0 && K >= 0 && B >= 0, "dic_candidate_admission: negative size");
    if (S == 0 || L == 0) return DIC_OK;
    cudaStream_t s = as_stream(stream);
    int64_t kc = pow2_at_least(2 * K + 2), bc = pow2_at_least(2 * B + 2);
    int32_t *kht = nullptr, *bht = nullptr;
    DIC_CUDA(cudaMallocAsync((void**)&kht, kc * sizeof(int32_t), s));
    DIC_CUDA(cudaMallocAsync((void**)&bht, bc * sizeof(int32_t), s));
    set_clear_kernel<<<(unsigned)std::min<int64_t>((kc + 255) / 256, 4096), 256, 0, s>>>(kht, kc); ::dic::note_launch();
    set_clear_kernel<<<(unsigned)std::min<int64_t>((bc + 255) / 256, 4096), 256, 0, s>>>(bht, bc); ::dic::note_launch();
    auto* km = reinterpret_cast<const unsigned long long*>(known_masks);
    auto* bm = reinterpret_cast<const unsigned long long*>(box_masks);
    if (K > 0) set_insert_kernel<<<(unsigned)((K + 255) / 256), 256, 0, s>>>(kht, kc - 1, km, K, W); ::dic::note_launch();
    if (B > 0) set_insert_kernel<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(bht, bc - 1, bm, B, W); ::dic::note_launch();
    int64_t total = S * L;
    admission_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(src_masks), S, level1, L, W, kht, kc - 1, km, bht, bc - 1, bm,
        admit); ::dic::note_launch();
    DIC_CHECK_LAUNCH("admission_kernel");
    DIC_CUDA(cudaFreeAsync(kht, s));
    DIC_CUDA(cudaFreeAsync(bht, s));
    DIC_CUDA(cudaStreamSynchronize(s));
    return DIC_OK;
}
