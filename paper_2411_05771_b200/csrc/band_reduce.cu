// band_reduce.cu — the receive side of the reduce-scatter split.
//
// With the sketch's m angles split over `world` ranks, every operator of the pass after the
// rotation is a sum over angle shards (||Ax - y||^2 = sum_i ||S_i A x - S_i
// y||^2; L92: the sketch is a row subset), so x_fbp = sum_r (pi / 2m) A_{S_r}^T q_r and
// grad = sum_r 2 A_{S_r}^T r_r.  Each rank's backprojector stores its partial of output row
// band o straight into rank o's receive buffer (the adjoint kernel's reduce-scatter
// epilogue, radon_adj.cu out_at, P2P stores over NVLink); after a cross-rank barrier rank o
// holds the world partials of its band, [world][2][B][bmax][n], and this kernel sums them in
// slot (= rank) order — a fixed order, so the result is bitwise reproducible — into the
// band of x_fbp and grad, and accumulates the band's ei partial sum (x2 - x_fbp)^2.
//
// HBM-bound: per band element it reads 2 world floats and x2 and writes 2 floats; float4
// where the row width allows (n % 4 == 0), 256 threads, a grid of ~4 CTAs per SM per image.
// ei: per-CTA fp32 partials (fixed tree), summed per image in CTA order in fp64 by one warp.
#include "internal.h"

namespace skei {
namespace {

constexpr int kThreads = 256;
constexpr int kPerCta = kThreads * 4 * 4;  // band elements per CTA (4 float4 per thread)

template <bool V4>
__global__ void __launch_bounds__(kThreads) k_band_reduce(const float *__restrict__ recv,
                                                          int world, int B, int bmax, int n,
                                                          int row0, int rows,
                                                          const float *__restrict__ x2,
                                                          float *xfbp, float *grad,
                                                          float *part) {
    const int b = blockIdx.y;
    const long per = (long)rows * n;              // band elements of one image
    const long slot = 2L * B * bmax * n;           // one rank's slot
    const long jstride = (long)B * bmax * n;       // job 1 after job 0 within a slot
    const float *src = recv + (long)b * bmax * n;  // job 0, image b, slot 0
    const float *xb = x2 + (long)b * n * n + (long)row0 * n;
    float ei = 0.f;
    constexpr int W = V4 ? 4 : 1;
    const long e0 = (long)blockIdx.x * kPerCta;
    const long e1 = min(per, e0 + kPerCta);
    for (long e = e0 + (long)threadIdx.x * W; e < e1; e += (long)kThreads * W) {
        // band element e = (row e / n, column e % n): recv rows are n wide as well
        float f[W], g[W], x[W];
#pragma unroll
        for (int k = 0; k < W; ++k) f[k] = g[k] = 0.f;
        for (int s = 0; s < world; ++s) {  // slot (rank) order
            const float *p = src + s * slot + e;
            if constexpr (V4) {
                const float4 a = __ldcg(reinterpret_cast<const float4 *>(p));
                const float4 c = __ldcg(reinterpret_cast<const float4 *>(p + jstride));
                f[0] += a.x; f[1] += a.y; f[2] += a.z; f[3] += a.w;
                g[0] += c.x; g[1] += c.y; g[2] += c.z; g[3] += c.w;
            } else {
                f[0] += __ldcg(p);
                g[0] += __ldcg(p + jstride);
            }
        }
        if constexpr (V4) {
            const float4 xv = __ldg(reinterpret_cast<const float4 *>(xb + e));
            x[0] = xv.x; x[1] = xv.y; x[2] = xv.z; x[3] = xv.w;
            *reinterpret_cast<float4 *>(xfbp + (long)b * per + e) = make_float4(f[0], f[1], f[2], f[3]);
            *reinterpret_cast<float4 *>(grad + (long)b * per + e) = make_float4(g[0], g[1], g[2], g[3]);
        } else {
            x[0] = __ldg(xb + e);
            xfbp[(long)b * per + e] = f[0];
            grad[(long)b * per + e] = g[0];
        }
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const float d = x[k] - f[k];
            ei = fmaf(d, d, ei);
        }
    }
    __shared__ float s_red[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ei += __shfl_xor_sync(0xffffffffu, ei, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ei;
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = 0.f;
        for (int w = 0; w < kThreads / 32; ++w) v += s_red[w];
        part[(long)b * gridDim.x + blockIdx.x] = v;
    }
}

// ei[b] = sum of image b's CTA partials in CTA order (fp64), one warp per image
__global__ void __launch_bounds__(32) k_band_ei(const float *part, int nblk, float *ei) {
    const int b = blockIdx.x, lane = threadIdx.x;
    double s = 0.0;
    for (int i = lane; i < nblk; i += 32) s += (double)part[(long)b * nblk + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ei[b] = (float)s;
}

}  // namespace

size_t band_reduce_part_floats(int n, int rows) {
    return (size_t)(((long)rows * n + kPerCta - 1) / kPerCta);
}

cudaError_t launch_band_reduce(const float *recv, int world, int B, int bmax, int n, int row0,
                               int rows, const float *x2, float *xfbp, float *grad, float *ei,
                               float *part, cudaStream_t s) {
    const int nblk = (int)band_reduce_part_floats(n, rows);
    const dim3 grid((unsigned)nblk, (unsigned)B, 1);
    // float4 needs 16-byte aligned rows everywhere: n % 4 == 0 and aligned base pointers
    const bool v4 = n % 4 == 0 && ((uintptr_t)recv | (uintptr_t)x2 | (uintptr_t)xfbp |
                                   (uintptr_t)grad) % 16 == 0;
    if (v4)
        k_band_reduce<true><<<grid, kThreads, 0, s>>>(recv, world, B, bmax, n, row0, rows, x2,
                                                      xfbp, grad, part);
    else
        k_band_reduce<false><<<grid, kThreads, 0, s>>>(recv, world, B, bmax, n, row0, rows, x2,
                                                       xfbp, grad, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_band_ei<<<B, 32, 0, s>>>(part, nblk, ei);
    return cudaGetLastError();
}

}  // namespace skei
