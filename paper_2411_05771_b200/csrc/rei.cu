// rei.cu — the REI variant's simulated measurement noise (PAPER.md L104:
// the robust EI loss reconstructs from A_S x2 + simulated noise, x3 = F(A_S^+(A_S x2 + eps))).
// pn[b][k][j] = p[b][k][j] + sigma eps, eps ~ N(0, 1): Box-Muller (cos branch) on words 2s
// and 2s+1 (s = k n_det + j) of the counter-based SplitMix64 stream keyed by (seed, stream
// 5, iter, image0 + b) — DESIGN.md R23, the same generator the oracle implements
// independently; u = ((w >> 11) + 1/2) 2^-53, the transcendentals in fp64.
#include "internal.h"
#include "sm64.h"

namespace skei {
namespace {

__global__ void __launch_bounds__(256) k_rei_noise(const float *p, float *pn, int B, int m,
                                                    int n_det, float sigma, uint64_t seed,
                                                    uint64_t iter, uint64_t image0) {
    const int b = blockIdx.y;
    const uint64_t key = sm64_key(seed, kStreamReiNoise, iter, image0 + (uint64_t)b);
    const long per = (long)m * n_det;
    for (long s = blockIdx.x * (long)blockDim.x + threadIdx.x; s < per;
         s += (long)gridDim.x * blockDim.x) {
        const double u1 = ((double)(sm64_out(key, 2 * (uint64_t)s) >> 11) + 0.5) * 0x1p-53;
        const double u2 = ((double)(sm64_out(key, 2 * (uint64_t)s + 1) >> 11) + 0.5) * 0x1p-53;
        const double eps = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
        pn[(long)b * per + s] = p[(long)b * per + s] + (float)(sigma * eps);
    }
}

}  // namespace

cudaError_t launch_rei_noise(const float *p, float *pn, int B, int m, int n_det, float sigma,
                             uint64_t seed, uint64_t iter, uint64_t image0, int num_sms,
                             cudaStream_t s) {
    const long per = (long)m * n_det;
    long bx = (per + 255) / 256;
    const long cap = (long)num_sms * 8 / (B > 0 ? B : 1) + 1;
    if (bx > cap) bx = cap;
    dim3 grid((unsigned)bx, (unsigned)B, 1);
    k_rei_noise<<<grid, 256, 0, s>>>(p, pn, B, m, n_det, sigma, seed, iter, image0);
    return cudaGetLastError();
}

}  // namespace skei
