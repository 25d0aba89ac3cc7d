// draw.cu — a1: the integer draws of Algorithm 1 step 2: the rotation
// g in 1..360 (|G| = 360, L284) and the sketch S (L102 "sample S_i"; L299
// interleaved minibatches; north_star "seeded uniform subset").  Counter-based
// SplitMix64 keyed by (seed, stream, iter, image) — DESIGN.md §2 R5.  Host and device
// versions below are bit-identical to each other and to the independent oracle.
#include <algorithm>
#include <vector>

#include "internal.h"
#include "sm64.h"

namespace skei {
namespace {

constexpr uint64_t kStreamRot = 1, kStreamSketch = 2;

__host__ __device__ inline uint32_t mulhi_below(uint64_t w, uint32_t n) {
#ifdef __CUDA_ARCH__
    return (uint32_t)__umul64hi(w, (uint64_t)n);
#else
    return (uint32_t)(((unsigned __int128)w * n) >> 64);
#endif
}

__host__ __device__ inline int draw_rotation(uint64_t seed, uint64_t iter, uint64_t image) {
    return 1 + (int)mulhi_below(sm64_out(sm64_key(seed, kStreamRot, iter, image), 0), 360u);
}

// One warp per drawn image (32-thread blocks).  The lanes compute the Fisher-Yates targets
// j_i = i + U(n_full - i) in parallel (each is a pure function of the word index), lane 0
// applies the m swaps in shared memory in order, and the chosen set is compacted with
// ballots, which emits it already sorted ascending (the same set as the host's sort).
__global__ void __launch_bounds__(32) k_draw(uint64_t seed, uint64_t iter, uint64_t image0,
                                             int shared, int n_full, int m, int mode,
                                             int32_t *g_out, int32_t *idx_out) {
    // let a programmatically serialized successor (the pass's rotate + pack, skei_pass_draw)
    // start now: it waits for this grid's completion before it reads the draw
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    extern __shared__ int sm[];
    int *perm = sm;           // [n_full]
    int *tgt = sm + n_full;   // [m]
    const int lane = threadIdx.x;
    const int b = blockIdx.x;
    const uint64_t image = shared ? ~0ULL : image0 + (uint64_t)b;
    int32_t *idx = idx_out + (size_t)b * m;
    if (lane == 0) g_out[b] = draw_rotation(seed, iter, image);
    const uint64_t ksk = sm64_key(seed, kStreamSketch, iter, image);
    if (mode == 0) {
        const int nb = n_full / m;
        const int base = (int)mulhi_below(sm64_out(ksk, 0), (uint32_t)nb);
        for (int k = lane; k < m; k += 32) idx[k] = base + k * nb;
        return;
    }
    for (int i = lane; i < n_full; i += 32) perm[i] = i;
    for (int i = lane; i < m; i += 32)
        tgt[i] = i + (int)mulhi_below(sm64_out(ksk, (uint64_t)i), (uint32_t)(n_full - i));
    __syncwarp();
    if (lane == 0) {
        for (int i = 0; i < m; ++i) {
            const int j = tgt[i];
            const int t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
    }
    __syncwarp();
    // collect the m chosen values, then mark them in a flag array (perm is reused)
    for (int i = lane; i < m; i += 32) {
        const int v = perm[i];
        tgt[i] = v;  // the chosen values (unsorted)
    }
    __syncwarp();
    for (int i = lane; i < n_full; i += 32) perm[i] = 0;
    __syncwarp();
    for (int i = lane; i < m; i += 32) perm[tgt[i]] = 1;
    __syncwarp();
    int carry = 0;
    for (int base = 0; base < n_full; base += 32) {
        const int i = base + lane;
        const int f = (i < n_full) ? perm[i] : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) idx[carry + __popc(bal & ((1u << lane) - 1u))] = i;
        carry += __popc(bal);
    }
}

}  // namespace

int host_draw(uint64_t seed, uint64_t iter, uint64_t image, int n_full, int m, int mode,
              int32_t *g, int32_t *idx) {
    *g = draw_rotation(seed, iter, image);
    const uint64_t ksk = sm64_key(seed, kStreamSketch, iter, image);
    if (mode == 0) {
        const int nb = n_full / m;
        const int base = (int)mulhi_below(sm64_out(ksk, 0), (uint32_t)nb);
        for (int k = 0; k < m; ++k) idx[k] = base + k * nb;
        return 0;
    }
    std::vector<int> perm(n_full);
    for (int i = 0; i < n_full; ++i) perm[i] = i;
    for (int i = 0; i < m; ++i) {
        int j = i + (int)mulhi_below(sm64_out(ksk, (uint64_t)i), (uint32_t)(n_full - i));
        std::swap(perm[i], perm[j]);
    }
    std::sort(perm.begin(), perm.begin() + m);
    for (int k = 0; k < m; ++k) idx[k] = perm[k];
    return 0;
}

cudaError_t launch_draw(uint64_t seed, uint64_t iter, uint64_t image0, int count, int shared,
                        int n_full, int m, int mode, int32_t *g, int32_t *idx, cudaStream_t s) {
    const size_t smem = (mode == 1) ? sizeof(int) * ((size_t)n_full + m) : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_draw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_draw<<<count, 32, smem, s>>>(seed, iter, image0, shared, n_full, m, mode, g, idx);
    return cudaGetLastError();
}

}  // namespace skei
