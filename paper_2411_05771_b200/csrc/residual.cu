// residual.cu — a7: r = A_S x1 - y_S, mc = ||r||^2, ei = ||x2 - x3||^2 (the
// loss of Algorithm 1 step 6; Eq. 6; unnormalised squared norms, R15).
//
// HBM-bound streaming reductions.  Deterministic two-stage reduction, no atomics:
// stage 1 — each block reduces a fixed chunk (fp32 per thread, warp shuffles, fp32 block
// total) into ws; stage 2 — one warp per image sums the chunk partials in fixed order in
// fp64.  x2/x3 are streamed with float4 loads.
#include <algorithm>

#include "internal.h"

namespace skei {
namespace {

constexpr int kThreads = 256;
constexpr int kMcPerThread = 8;   // residual elements per thread per block
constexpr int kEiPerThread = 16;  // float4 groups per thread per block

__device__ inline float block_sum(float v) {
    __shared__ float wsum[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    float t = 0.f;
    if (threadIdx.x < 32) {
        t = threadIdx.x < kThreads / 32 ? wsum[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;  // valid in thread 0
}

// grid (chunks, B)
__global__ void __launch_bounds__(kThreads) k_mc_partial(const float *__restrict__ p1,
                                                         const float *__restrict__ y,
                                                         const int32_t *__restrict__ idx,
                                                         int m, int idx_stride, int n_det,
                                                         int n_full, float *r, float *part) {
    const int b = blockIdx.y;
    const long per_img = (long)m * n_det;
    const int32_t *ib = idx + (long)b * idx_stride;
    const float *pb = p1 + (long)b * per_img;
    const float *yb = y + (long)b * n_full * n_det;
    float *rb = r ? r + (long)b * per_img : nullptr;
    const long e0 = (long)blockIdx.x * kThreads * kMcPerThread;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < kMcPerThread; ++i) {
        const long e = e0 + (long)i * kThreads + threadIdx.x;
        if (e < per_img) {
            const int k = (int)(e / n_det);
            const int j = (int)(e - (long)k * n_det);
            const float d = pb[e] - __ldg(yb + (long)ib[k] * n_det + j);
            if (rb) rb[e] = d;
            acc = fmaf(d, d, acc);
        }
    }
    const float t = block_sum(acc);
    if (threadIdx.x == 0) part[(long)b * gridDim.x + blockIdx.x] = t;
}

__global__ void __launch_bounds__(kThreads) k_ei_partial(const float *__restrict__ x2,
                                                         const float *__restrict__ x3, long nn,
                                                         int vec, float *part) {
    const int b = blockIdx.y;
    const float *a = x2 + (long)b * nn;
    const float *c = x3 + (long)b * nn;
    const long g0 = (long)blockIdx.x * kThreads * kEiPerThread;  // float4 group index
    const long ngroups = vec ? nn / 4 : 0;  // float4 path needs 16-byte aligned rows
    float acc = 0.f;
#pragma unroll 4
    for (int i = 0; i < kEiPerThread; ++i) {
        const long g = g0 + (long)i * kThreads + threadIdx.x;
        if (g < ngroups) {
            const float4 u = __ldg(reinterpret_cast<const float4 *>(a) + g);
            const float4 v = __ldg(reinterpret_cast<const float4 *>(c) + g);
            const float d0 = u.x - v.x, d1 = u.y - v.y, d2 = u.z - v.z, d3 = u.w - v.w;
            acc = fmaf(d0, d0, acc);
            acc = fmaf(d1, d1, acc);
            acc = fmaf(d2, d2, acc);
            acc = fmaf(d3, d3, acc);
        }
    }
    if (blockIdx.x == gridDim.x - 1) {  // scalar tail (nn % 4)
        for (long e = ngroups * 4 + threadIdx.x; e < nn; e += kThreads) {
            const float d = a[e] - c[e];
            acc = fmaf(d, d, acc);
        }
    }
    const float t = block_sum(acc);
    if (threadIdx.x == 0) part[(long)b * gridDim.x + blockIdx.x] = t;
}

// one warp per image and per quantity
__global__ void k_final(const float *part, int nchunks, float *out) {
    const int b = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nchunks; i += 32) acc += (double)part[(long)b * nchunks + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) out[b] = (float)acc;
}

int mc_chunks(int m, int n_det) {
    const long per = (long)m * n_det;
    return (int)((per + kThreads * kMcPerThread - 1) / (kThreads * kMcPerThread));
}
int ei_chunks(int n) {
    const long groups = ((long)n * n) / 4;
    const long per = (long)kThreads * kEiPerThread;
    return (int)std::max<long>(1, (groups + per - 1) / per);
}

}  // namespace

size_t residual_ws_bytes(const skei_plan *plan, int B, int m) {
    return sizeof(float) * (size_t)B * (mc_chunks(m, plan->n_det) + ei_chunks(plan->n)) + 256;
}

cudaError_t launch_residual(const skei_plan *plan, const float *p1, const float *y,
                            const int32_t *idx, int m, int idx_stride, const float *x2,
                            const float *x3, int B, float *mc, float *ei, float *r, void *ws,
                            cudaStream_t s) {
    float *part_mc = (float *)ws;
    const int cm = mc_chunks(m, plan->n_det);
    float *part_ei = part_mc + (size_t)B * cm;
    const int ce = ei_chunks(plan->n);
    if (p1 && mc) {
        k_mc_partial<<<dim3(cm, B), kThreads, 0, s>>>(p1, y, idx, m, idx_stride, plan->n_det,
                                                       plan->n_full, r, part_mc);
        k_final<<<B, 32, 0, s>>>(part_mc, cm, mc);
    }
    if (x2 && x3 && ei) {
        const long nn = (long)plan->n * plan->n;
        const int vec = (nn % 4 == 0) && ((uintptr_t)x2 % 16 == 0) && ((uintptr_t)x3 % 16 == 0);
        k_ei_partial<<<dim3(ce, B), kThreads, 0, s>>>(x2, x3, nn, vec, part_ei);
        k_final<<<B, 32, 0, s>>>(part_ei, ce, ei);
    }
    return cudaGetLastError();
}

}  // namespace skei
