// deviation.cu — the Theorem-1 sketching deviation (Theorem 1
// L258-L270 and its proof L575-L583): delta = ||A^T (S^T S - I) A||_2 for the
// sqrt(n_full/m)-scaled row-subsampling sketch of the sketched angles, by power iteration
// on the symmetric operator D v = (n_full/m) A_S^T A_S v - A^T A v.  The operator runs on
// the pass's kernels (packing, forward projector on the full and on the sketched angle
// set, backprojector with accumulate-into-base); this file holds the per-iteration
// normalisation: ||w||^2 per image in a fixed-order (deterministic) two-level reduction —
// chunk partials from a grid of CTAs, completed by every CTA of the normalisation — and
// v = w / ||w||.
#include "internal.h"

namespace skei {
namespace {

constexpr int kRedThreads = 256;

// chunks per image of the two-level fixed-order norm (<= kNormChunks)
inline int norm_chunks(long per) {
    const long c = (per + 4095) / 4096;
    return (int)(c < kNormChunks ? (c > 0 ? c : 1) : kNormChunks);
}

// part[b][c] = sum of w[b][i]^2 over chunk c (fp64 accumulation, fixed order): the
// first level of the per-image norm, a grid of (chunks x images) CTAs
__global__ void __launch_bounds__(kRedThreads) k_sumsq(const float *w, long per, int nch,
                                                       double *part) {
    __shared__ double s[kRedThreads / 32];
    const long len = (per + nch - 1) / nch;
    const long i0 = (long)blockIdx.x * len, i1 = min(per, i0 + len);
    const float *wb = w + (long)blockIdx.y * per;
    double acc = 0.0;
    for (long i = i0 + threadIdx.x; i < i1; i += kRedThreads) {
        const double v = (double)wb[i];
        acc = fma(v, v, acc);
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < kRedThreads / 32; ++k) t += s[k];
        part[(long)blockIdx.y * nch + blockIdx.x] = t;
    }
}

// v = w / ||w|| per image (v = w if ||w|| = 0); lambda[b] = ||w|| as fp32.  Every CTA
// first completes the image's norm from the chunk partials in one fixed order (identical
// in all CTAs: lane-strided sums, then a fixed shuffle tree).
__global__ void k_normalise(const float *w, float *v, long per, int nch, const double *part,
                            float *lambda) {
    __shared__ double s_n2;
    const int b = blockIdx.y;
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int c = threadIdx.x; c < nch; c += 32) t += part[(long)b * nch + c];
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (threadIdx.x == 0) s_n2 = t;
    }
    __syncthreads();
    const double nrm = sqrt(s_n2);
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

cudaError_t launch_sumsq(const float *w, int B, long per, double *part, cudaStream_t s) {
    const int nch = norm_chunks(per);
    k_sumsq<<<dim3((unsigned)nch, (unsigned)B), kRedThreads, 0, s>>>(w, per, nch, part);
    return cudaGetLastError();
}

cudaError_t launch_normalise(const float *w, float *v, int B, long per, const double *part,
                             float *lambda, int num_sms, cudaStream_t s) {
    long bx = (per + 255) / 256;
    const long cap = (long)num_sms * 8 / (B > 0 ? B : 1) + 1;
    if (bx > cap) bx = cap;
    k_normalise<<<dim3((unsigned)bx, (unsigned)B), 256, 0, s>>>(w, v, per, norm_chunks(per),
                                                                 part, lambda);
    return cudaGetLastError();
}

cudaError_t launch_iota(int32_t *a, int n, cudaStream_t s) {
    k_iota<<<(n + 255) / 256, 256, 0, s>>>(a, n);
    return cudaGetLastError();
}

}  // namespace skei
