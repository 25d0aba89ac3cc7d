// radon_adj.cu — a5/a8: x = scale * A_S^T p, the exact transpose of the pixel-driven
// projector (BASELINE.json north_star: "radon_adj is its exact transpose, a per-pixel
// gather over angles with the sketched angle table in shared memory").
//
// Design (DESIGN.md §5 "radon_adj"):
//   * one CTA = a 32x32 pixel tile x BB images that share one angle list (BB = 4 for a
//     per-pass sketch, 1 for per-image sketches) x one job (two jobs — FBP of q and the
//     gradient of r — share a launch);
//   * angles are processed in chunks of KC; for each angle the CTA stages the W-bin
//     detector window the tile projects onto, interleaved over the BB images
//     ([angle][bin][image], 16-byte rows for BB = 4), zero outside [0, n_det) so
//     dropped taps need no branch;
//   * each thread owns one column x 4 rows of the tile; per (pixel, angle) it forms
//     j + f = t - s_0 in split precision (fp64 tile base per angle, fp32 local offset
//     |.| < 48 px — DESIGN.md §5 "precision"), then 2 LDS.128 + 2*BB FFMA:
//     acc_b += (1-f) q_b[j] + f q_b[j+1];
//   * 8 lanes of a quarter-warp are 8 consecutive columns whose bins span <= 8
//     consecutive 16-byte slots, so the LDS.128s are bank-conflict-free.
// Work per (pixel, angle, image) = 2 taps, 8 bytes of shared-memory reads: this
// kernel is bound by shared-memory bandwidth (the "gather roofline").
#include "internal.h"

namespace skei {
namespace {

constexpr int kTile = 32;        // tile side (pixels)
constexpr int kRowsPerThread = 4;
constexpr int kThreads = 256;    // 32 columns x 8 row groups
constexpr int kKC = 32;          // angles per staged chunk
constexpr int kW = 48;           // staged bins per angle (>= 31*sqrt(2) + 3)

struct AdjArgs {
    AdjJob job[2];
    const int32_t *idx;
    int m, idx_stride, B, tiles_x;
    Geom g;
};

template <int BB>
struct Vec;
template <> struct Vec<1> { using T = float; };
template <> struct Vec<2> { using T = float2; };
template <> struct Vec<4> { using T = float4; };

template <int BB>
__device__ inline void load_bins(const float *base, float (&v)[BB]) {
    typename Vec<BB>::T t = *reinterpret_cast<const typename Vec<BB>::T *>(base);
    const float *pt = reinterpret_cast<const float *>(&t);
#pragma unroll
    for (int b = 0; b < BB; ++b) v[b] = pt[b];
}

template <int BB>
__global__ void __launch_bounds__(kThreads) k_radon_adj(AdjArgs a) {
    __shared__ __align__(16) float win[kKC * kW * BB];
    __shared__ float s_off[kKC], s_cos[kKC], s_sin[kKC];
    __shared__ int s_w0[kKC], s_slot[kKC];

    const AdjJob job = blockIdx.z ? a.job[1] : a.job[0];
    const int n = a.g.n, n_det = a.g.n_det;
    const int tile = blockIdx.x;
    const int tr0 = (tile / a.tiles_x) * kTile, tc0 = (tile % a.tiles_x) * kTile;
    const int b0 = blockIdx.y * BB;
    const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const long nn = (long)n * n;

    float acc[kRowsPerThread][BB];
#pragma unroll
    for (int i = 0; i < kRowsPerThread; ++i)
#pragma unroll
        for (int b = 0; b < BB; ++b) acc[i][b] = 0.f;

    for (int k0 = 0; k0 < a.m; k0 += kKC) {
        const int kc = min(kKC, a.m - k0);
        if (threadIdx.x < kc) {
            const int k = k0 + threadIdx.x;
            const double2 cs = a.g.trig[idx[k]];
            // jpos at the tile origin pixel (tr0, tc0), fp64
            const double J0 = a.g.hd + (tc0 - a.g.h) * cs.x + (a.g.h - tr0) * cs.y;
            const double jmin = J0 + fmin(0.0, (kTile - 1) * cs.x) + fmin(0.0, -(kTile - 1) * cs.y);
            const double w0 = floor(jmin);
            s_off[threadIdx.x] = (float)(J0 - w0);
            s_cos[threadIdx.x] = (float)cs.x;
            s_sin[threadIdx.x] = (float)cs.y;
            s_w0[threadIdx.x] = (int)w0;
            s_slot[threadIdx.x] = k;
        }
        __syncthreads();
        // stage windows: element e -> (angle t, bin w, image b), image fastest
        for (int e = threadIdx.x; e < kc * kW * BB; e += kThreads) {
            const int b = e % BB;
            const int w = (e / BB) % kW;
            const int t = e / (BB * kW);
            const int j = s_w0[t] + w;
            float v = 0.f;
            if (j >= 0 && j < n_det)
                v = __ldg(job.p + ((long)(b0 + b) * a.m + s_slot[t]) * n_det + j);
            win[e] = v;
        }
        __syncthreads();
#pragma unroll 2
        for (int t = 0; t < kc; ++t) {
            const float ct = s_cos[t], st = s_sin[t];
            const float base = fmaf((float)tx, ct, fmaf(-(float)ty, st, s_off[t]));
            const float step = -8.0f * st;
            const float *wt = win + t * kW * BB;
#pragma unroll
            for (int i = 0; i < kRowsPerThread; ++i) {
                float jr = fmaxf(fmaf((float)i, step, base), 0.f);
                const float fl = floorf(jr);
                const float f = jr - fl;
                const int j = min((int)fl, kW - 2);
                float q0[BB], q1[BB];
                load_bins<BB>(wt + j * BB, q0);
                load_bins<BB>(wt + (j + 1) * BB, q1);
                const float f0 = 1.f - f;
#pragma unroll
                for (int b = 0; b < BB; ++b) acc[i][b] = fmaf(f, q1[b], fmaf(f0, q0[b], acc[i][b]));
            }
        }
        __syncthreads();
    }
    const int c = tc0 + tx;
    if (c < n) {
#pragma unroll
        for (int i = 0; i < kRowsPerThread; ++i) {
            const int r = tr0 + ty + 8 * i;
            if (r < n) {
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    job.x[(long)(b0 + b) * nn + (long)r * n + c] = job.scale * acc[i][b];
            }
        }
    }
}

}  // namespace

cudaError_t launch_radon_adj(const skei_plan *plan, const AdjJob *jobs, int njobs, int B,
                             const int32_t *idx, int m, int idx_stride, cudaStream_t s) {
    AdjArgs a;
    a.job[0] = jobs[0];
    a.job[1] = njobs > 1 ? jobs[1] : jobs[0];
    a.idx = idx;
    a.m = m;
    a.idx_stride = idx_stride;
    a.B = B;
    a.g = geom_of(plan);
    a.tiles_x = (plan->n + kTile - 1) / kTile;
    const int bb = pick_bb(B, idx_stride);
    dim3 grid((unsigned)(a.tiles_x * a.tiles_x), (unsigned)(B / bb), (unsigned)njobs);
    switch (bb) {
        case 4: k_radon_adj<4><<<grid, kThreads, 0, s>>>(a); break;
        case 2: k_radon_adj<2><<<grid, kThreads, 0, s>>>(a); break;
        default: k_radon_adj<1><<<grid, kThreads, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

}  // namespace skei
