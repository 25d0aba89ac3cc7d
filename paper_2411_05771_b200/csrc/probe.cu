// probe.cu — diagnostic shared-memory read-bandwidth probe (skei_smem_probe): the measured
// denominator of the gather roofline.  Each thread issues LDS.128 over a
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

}  // namespace

cudaError_t launch_smem_probe(float *sink, int blocks, int iters, cudaStream_t s) {
    k_smem_probe<<<blocks, kProbeThreads, 0, s>>>(sink, iters);
    return cudaGetLastError();
}

}  // namespace skei
