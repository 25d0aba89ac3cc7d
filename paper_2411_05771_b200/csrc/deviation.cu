// deviation.cu — the Theorem-1 sketching deviation (Theorem 1
// L258-L270 and its proof L575-L583): delta = ||A^T (S^T S - I) A||_2 for the
// sqrt(n_full/m)-scaled row-subsampling sketch of the sketched angles, by power iteration
// on the symmetric operator D v = (n_full/m) A_S^T A_S v - A^T A v.  The operator runs on
// the pass's kernels (packing, forward projector on the full and on the sketched angle
// set, backprojector with accumulate-into-base); this file holds the per-iteration
// normalisation: ||w||^2 per image in a fixed-order (deterministic) reduction, v = w / ||w||.
#include "internal.h"

namespace skei {
namespace {

constexpr int kRedThreads = 512;

// norm2[b] = sum_i w[b][i]^2 (fp64 accumulation, one CTA per image, fixed order)
__global__ void __launch_bounds__(kRedThreads) k_sumsq(const float *w, long per, double *norm2) {
    __shared__ double s[kRedThreads / 32];
    const float *wb = w + (long)blockIdx.x * per;
    double acc = 0.0;
    for (long i = threadIdx.x; i < per; i += kRedThreads) {
        const double v = (double)wb[i];
        acc = fma(v, v, acc);
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < kRedThreads / 32; ++k) t += s[k];
        norm2[blockIdx.x] = t;
    }
}

// v = w / ||w|| per image (v = w if ||w|| = 0); lambda[b] = ||w|| as fp32
__global__ void k_normalise(const float *w, float *v, long per, const double *norm2,
                            float *lambda) {
    const int b = blockIdx.y;
    const double nrm = sqrt(norm2[b]);
    const float inv = nrm > 0.0 ? (float)(1.0 / nrm) : 1.f;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < per;
         i += (long)gridDim.x * blockDim.x)
        v[(long)b * per + i] = w[(long)b * per + i] * inv;
    if (lambda && blockIdx.x == 0 && threadIdx.x == 0) lambda[b] = (float)nrm;
}

__global__ void k_iota(int32_t *a, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

}  // namespace

cudaError_t launch_sumsq(const float *w, int B, long per, double *norm2, cudaStream_t s) {
    k_sumsq<<<B, kRedThreads, 0, s>>>(w, per, norm2);
    return cudaGetLastError();
}

cudaError_t launch_normalise(const float *w, float *v, int B, long per, const double *norm2,
                             float *lambda, int num_sms, cudaStream_t s) {
    long bx = (per + 255) / 256;
    const long cap = (long)num_sms * 8 / (B > 0 ? B : 1) + 1;
    if (bx > cap) bx = cap;
    k_normalise<<<dim3((unsigned)bx, (unsigned)B), 256, 0, s>>>(w, v, per, norm2, lambda);
    return cudaGetLastError();
}

cudaError_t launch_iota(int32_t *a, int n, cudaStream_t s) {
    k_iota<<<(n + 255) / 256, 256, 0, s>>>(a, n);
    return cudaGetLastError();
}

}  // namespace skei
