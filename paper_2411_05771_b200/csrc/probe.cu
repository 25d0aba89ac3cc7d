// probe.cu — diagnostic bandwidth probes: shared-memory reads (skei_smem_probe, the measured
// denominator of the gather roofline) and L2 reads (skei_l2_probe, SURVEY
// §2.6 M2: the bound of the forward's re-staging of packed blocks from L2).  Each thread issues LDS.128 over a
// 64 KB buffer with a lane-contiguous, conflict-free pattern (a quarter-warp reads 128
// contiguous bytes per wavefront), accumulating so the loads cannot be elided.
#include "internal.h"

namespace skei {
namespace {

constexpr int kProbeThreads = 1024;
constexpr int kProbeBuf = 2048;  // float4 elements = 32 KB

__global__ void __launch_bounds__(kProbeThreads) k_smem_probe(float *sink, int iters) {
    __shared__ float4 buf[kProbeBuf];
    for (int i = threadIdx.x; i < kProbeBuf; i += kProbeThreads)
        buf[i] = make_float4((float)i, 1.f, 2.f, 3.f);
    __syncthreads();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int base = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const float4 v = buf[(base + u * 64) & (kProbeBuf - 1)];  // 32 distinct slots
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        base += 7;
    }
    const float s = acc.x + acc.y + acc.z + acc.w;
    if (s == -1.f) sink[blockIdx.x] = s;  // never true; keeps the loads live
    if (threadIdx.x == 0) sink[blockIdx.x] = s;
}

// L2 read bandwidth: every CTA streams the whole `n4`-float4 buffer (sized well under the
// L2, so after the first sweep every load hits L2) with ld.global.cg (L1 bypassed), each
// CTA starting at its own offset so the slices spread over both L2 partitions.
__global__ void __launch_bounds__(1024) k_l2_probe(const float4 *__restrict__ buf, long n4,
                                                   int iters, float *sink) {
    float acc = 0.f;
    const long start = (long)blockIdx.x * (n4 / gridDim.x);
    for (int it = 0; it < iters; ++it) {
        for (long j = threadIdx.x; j < n4; j += 4L * blockDim.x) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                long k = start + j + (long)u * blockDim.x;  // < 3 n4
                k = k >= n4 ? k - n4 : k;
                k = k >= n4 ? k - n4 : k;
                v[u] = __ldcg(buf + k);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    }
    if (acc == -1.f || threadIdx.x == 0) sink[blockIdx.x] = acc;
}

}  // namespace

cudaError_t launch_l2_probe(const float *buf, long n_floats, float *sink, int blocks, int iters,
                            cudaStream_t s) {
    k_l2_probe<<<blocks, 1024, 0, s>>>(reinterpret_cast<const float4 *>(buf), n_floats / 4, iters,
                                       sink);
    return cudaGetLastError();
}

cudaError_t launch_smem_probe(float *sink, int blocks, int iters, cudaStream_t s) {
    k_smem_probe<<<blocks, kProbeThreads, 0, s>>>(sink, iters);
    return cudaGetLastError();
}

}  // namespace skei
