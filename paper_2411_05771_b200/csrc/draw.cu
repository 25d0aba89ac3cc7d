// draw.cu — a1: the integer draws of Algorithm 1 step 2: the rotation
// g in 1..360 (|G| = 360, L284) and the sketch S (L102 "sample S_i"; L299
// interleaved minibatches; north_star "seeded uniform subset").  Counter-based
// SplitMix64 keyed by (seed, stream, iter, image) — DESIGN.md §2 R5.  Host and device
// versions below are bit-identical to each other and to the independent oracle.
#include <algorithm>
#include <vector>

#include "internal.h"

namespace skei {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kStreamRot = 1, kStreamSketch = 2;

__host__ __device__ inline uint64_t sm64_finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// i-th output of the SplitMix64 stream whose state starts at `state`.
__host__ __device__ inline uint64_t sm64_out(uint64_t state, uint64_t i) {
    return sm64_finalize(state + (i + 1) * kGolden);
}

__host__ __device__ inline uint64_t sm64_key(uint64_t seed, uint64_t stream, uint64_t iter,
                                             uint64_t image) {
    uint64_t k = sm64_out(seed, 0) ^ stream;
    k = sm64_out(k, 0) ^ iter;
    k = sm64_out(k, 0) ^ image;
    return sm64_out(k, 0);
}

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

// One block per drawn image: thread 0 runs the partial Fisher-Yates swaps in shared
// memory, then the block compacts the chosen flags with a prefix scan, which emits the
// subset already sorted ascending.
__global__ void k_draw(uint64_t seed, uint64_t iter, uint64_t image0, int shared, int n_full,
                       int m, int mode, int32_t *g_out, int32_t *idx_out) {
    extern __shared__ int sm[];
    int *perm = sm;              // [n_full]
    int *flag = sm + n_full;     // [n_full]
    __shared__ int warp_tot[32];
    const int b = blockIdx.x;
    const uint64_t image = shared ? ~0ULL : image0 + (uint64_t)b;
    int32_t *idx = idx_out + (size_t)b * m;
    if (threadIdx.x == 0) g_out[b] = draw_rotation(seed, iter, image);
    const uint64_t ksk = sm64_key(seed, kStreamSketch, iter, image);
    if (mode == 0) {
        const int nb = n_full / m;
        const int base = (int)mulhi_below(sm64_out(ksk, 0), (uint32_t)nb);
        for (int k = threadIdx.x; k < m; k += blockDim.x) idx[k] = base + k * nb;
        return;
    }
    for (int i = threadIdx.x; i < n_full; i += blockDim.x) {
        perm[i] = i;
        flag[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < m; ++i) {
            int j = i + (int)mulhi_below(sm64_out(ksk, (uint64_t)i), (uint32_t)(n_full - i));
            int t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) flag[perm[i]] = 1;
    __syncthreads();
    // block-wide exclusive scan over flags, chunked by blockDim
    int carry = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < n_full; base += blockDim.x) {
        int i = base + threadIdx.x;
        int f = (i < n_full) ? flag[i] : 0;
        unsigned bal = __ballot_sync(0xffffffffu, f);
        int pre = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        int woff = 0, tot = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < wid) woff += warp_tot[w];
            tot += warp_tot[w];
        }
        if (f) idx[carry + woff + pre] = i;
        carry += tot;
        __syncthreads();
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
    const size_t smem = (mode == 1) ? sizeof(int) * 2 * (size_t)n_full : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_draw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_draw<<<count, 256, smem, s>>>(seed, iter, image0, shared, n_full, m, mode, g, idx);
    return cudaGetLastError();
}

}  // namespace skei
