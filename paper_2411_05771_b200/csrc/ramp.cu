// ramp.cu — a4: q = h2 (*) p row by row (doubled Ram-Lak kernel, R8), as the
// north_star's "batched zero-padded real FFT-multiply kernel".
//
// Two real rows are packed into one complex sequence z = p_a + i p_b, zero-padded to
// P >= 2 n_det - 1 (so the circular convolution equals the linear one on the first
// n_det outputs).  Because the spectrum R[k] is real and even,
// IFFT(R . FFT(z)) = (h2 (*) p_a) + i (h2 (*) p_b): no post-processing twiddles.  The
// FFT is an in-shared-memory Stockham autosort transform, radix-4 stages plus one
// radix-2 stage when log2 P is odd; twiddles and R come from fp64-derived plan tables.
#include "internal.h"

namespace skei {
namespace {

constexpr int kThreads = 256;

__device__ inline float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ inline float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ inline float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
__device__ inline float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }
__device__ inline float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }

// twiddle exp(-+2 pi i e / P) for 0 <= e < P from the half table tw[0, P/2)
__device__ inline float2 twiddle(const float2 *tw, int e, int half, bool inverse) {
    float2 w = e < half ? tw[e] : make_float2(-tw[e - half].x, -tw[e - half].y);
    if (inverse) w.y = -w.y;
    return w;
}

// One full complex FFT of length P = 2^logP in shared memory; returns the buffer that
// holds the result.
__device__ float2 *stockham(float2 *a, float2 *b, const float2 *tw, int P, int logP,
                            bool inverse) {
    const int half = P / 2;
    int Ns = 1;
    int s = 0;
    for (; s + 2 <= logP; s += 2) {  // radix-4 stages
        const int quarter = P / 4;
        const int tstep = P / (4 * Ns);
        for (int j = threadIdx.x; j < quarter; j += blockDim.x) {
            const int k = j & (Ns - 1);
            float2 v0 = a[j], v1 = a[j + quarter], v2 = a[j + 2 * quarter], v3 = a[j + 3 * quarter];
            if (Ns > 1) {
                v1 = cmul(v1, twiddle(tw, k * tstep, half, inverse));
                v2 = cmul(v2, twiddle(tw, 2 * k * tstep, half, inverse));
                v3 = cmul(v3, twiddle(tw, 3 * k * tstep, half, inverse));
            }
            const float2 s02 = cadd(v0, v2), d02 = csub(v0, v2);
            const float2 s13 = cadd(v1, v3), d13 = csub(v1, v3);
            const float2 r13 = inverse ? mul_pi(d13) : mul_mi(d13);
            const int d = (j - k) * 4 + k;
            b[d] = cadd(s02, s13);
            b[d + Ns] = cadd(d02, r13);
            b[d + 2 * Ns] = csub(s02, s13);
            b[d + 3 * Ns] = csub(d02, r13);
        }
        __syncthreads();
        float2 *t = a;
        a = b;
        b = t;
        Ns *= 4;
    }
    if (s < logP) {  // final radix-2 stage
        const int tstep = P / (2 * Ns);
        for (int j = threadIdx.x; j < half; j += blockDim.x) {
            const int k = j & (Ns - 1);
            const float2 v0 = a[j];
            const float2 v1 = cmul(a[j + half], twiddle(tw, k * tstep, half, inverse));
            const int d = (j - k) * 2 + k;
            b[d] = cadd(v0, v1);
            b[d + Ns] = csub(v0, v1);
        }
        __syncthreads();
        a = b;
    }
    return a;
}

__global__ void __launch_bounds__(kThreads) k_ramp(const float *__restrict__ p, float *q,
                                                   int rows, int n_det, int P, int logP,
                                                   const float2 *__restrict__ tw_g,
                                                   const float *__restrict__ R) {
    extern __shared__ float2 sm[];
    float2 *bufA = sm, *bufB = sm + P, *tw = sm + 2 * P;  // tw: [P/2]
    const int ra = 2 * blockIdx.x, rb = ra + 1;
    const bool has_b = rb < rows;
    for (int i = threadIdx.x; i < P / 2; i += blockDim.x) tw[i] = tw_g[i];
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        float xa = 0.f, xb = 0.f;
        if (i < n_det) {
            xa = p[(long)ra * n_det + i];
            if (has_b) xb = p[(long)rb * n_det + i];
        }
        bufA[i] = make_float2(xa, xb);
    }
    __syncthreads();
    float2 *z = stockham(bufA, bufB, tw, P, logP, false);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const float r = R[i];
        z[i] = make_float2(z[i].x * r, z[i].y * r);
    }
    __syncthreads();
    float2 *other = (z == bufA) ? bufB : bufA;
    z = stockham(z, other, tw, P, logP, true);
    for (int i = threadIdx.x; i < n_det; i += blockDim.x) {
        q[(long)ra * n_det + i] = z[i].x;
        if (has_b) q[(long)rb * n_det + i] = z[i].y;
    }
}

}  // namespace

cudaError_t launch_ramp(const skei_plan *plan, const float *p, float *q, int rows,
                        cudaStream_t s) {
    const int P = plan->fft_len;
    const size_t smem = sizeof(float2) * (2 * (size_t)P + P / 2);
    if (smem > 48 * 1024) {  // per-device attribute: set on every call (cheap)
        cudaError_t e =
            cudaFuncSetAttribute(k_ramp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int grid = (rows + 1) / 2;
    k_ramp<<<grid, kThreads, smem, s>>>(p, q, rows, plan->n_det, P, plan->log2_fft, plan->d_tw,
                                        plan->d_ramp);
    return cudaGetLastError();
}

}  // namespace skei
