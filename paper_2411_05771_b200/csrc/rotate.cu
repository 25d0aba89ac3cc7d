// rotate.cu — a2: x2 = T_g x1 (EI group action of Eq. 4), bilinear,
// zero outside, about the image centre, counter-clockwise for g > 0 (R11), fused
// with the packing of the forward projector's input.
//
// k_rotate_pack: one CTA = an 8 x 32 pixel tile of BB images that share g (BB = the image
// group of the forward projector).  Each thread forms the fp64 source coordinates of one
// output pixel once and applies them to its BB images (4 taps each, read-only path).  It
// writes, as requested (cos g, sin g come from the plan's fp64 table of the 360 angles):
//   * the plain rotated image out[b][r][c]                          (skei_rotate's output)
//   * the row-packed copy  xr[grp][r / R][c][r % R][b]  (R = 32 / BB lines per block)
//   * the col-packed copy  xc[grp][c / R][r][c % R][b]
// i.e. the image cut into blocks of R lines, each block stored pixel-major with the R lines
// x BB images of one pixel in 128 contiguous bytes — the layout k_radon_fwd stages with one
// TMA bulk copy per block.  Pixels outside the image (the last block's
// padding lines) are written as zeros.  The identity job (g = 0, no taps) packs x1.
#include "internal.h"

namespace skei {
namespace {

constexpr int kTR = 8, kTC = 32;  // tile rows x columns

template <int BB>
__global__ void __launch_bounds__(kTR * kTC) k_rotate_pack(RotPackArgs a) {
    constexpr int R = 32 / BB;
    constexpr int kRow = kTC * BB + 4;  // padded tile row (floats): conflict-free pack reads
    __shared__ __align__(16) float tile[kTR * kRow];
    const RotPackJob job = blockIdx.z ? a.job[1] : a.job[0];
    const int n = a.n;
    const int tr = threadIdx.x / kTC, tc = threadIdx.x % kTC;
    const int r0 = blockIdx.x / a.tiles_c * kTR, c0 = blockIdx.x % a.tiles_c * kTC;
    const int r = r0 + tr, c = c0 + tc;
    const int b0 = blockIdx.y * BB;
    const long nn = (long)n * n;
    const bool inside = r < n && c < n;
    if (job.zero && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
        job.zero[0] = job.zero[1] = job.zero[2] = 0u;  // the pass's counters (fused
                                                        // reductions, forward work queue)

    float v[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) v[b] = 0.f;
    if (inside) {
        if (job.g == nullptr) {  // identity (pack x1)
#pragma unroll
            for (int b = 0; b < BB; ++b)
                if (b0 + b < a.B) v[b] = __ldg(job.x + (b0 + b) * nn + (long)r * n + c);
        } else {
            // fp64 source coordinates, once per pixel for a shared g (g_stride = 0) or per
            // image (g_stride = 1)
            const double h = (n - 1) * 0.5;
            const double u = c - h, w = h - r;
            int gprev = 0x7fffffff;
            float w00 = 0.f, w01 = 0.f, w10 = 0.f, w11 = 0.f;
            bool okr0 = false, okr1 = false, okc0 = false, okc1 = false;
            long o00 = 0;
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                if (b0 + b >= a.B) continue;
                const int gd = job.g[job.g_stride ? b0 + b : 0];
                if (gd != gprev) {
                    gprev = gd;
                    // (cos g, sin g) from the plan's fp64 table (exact at multiples of 90)
                    const double2 csg = a.rot[((gd % 360) + 360) % 360];
                    const double cg = csg.x, sg = csg.y;
                    const double us = u * cg + w * sg;
                    const double vs = -u * sg + w * cg;
                    const double cs = us + h, rs = h - vs;
                    const double r0d = floor(rs), c0d = floor(cs);
                    const float fa = (float)(rs - r0d), fb = (float)(cs - c0d);
                    const int ri = (int)r0d, ci = (int)c0d;
                    okr0 = ri >= 0 && ri < n;
                    okr1 = ri + 1 >= 0 && ri + 1 < n;
                    okc0 = ci >= 0 && ci < n;
                    okc1 = ci + 1 >= 0 && ci + 1 < n;
                    w00 = (1.f - fa) * (1.f - fb);
                    w01 = (1.f - fa) * fb;
                    w10 = fa * (1.f - fb);
                    w11 = fa * fb;
                    o00 = (long)ri * n + ci;
                }
                const float *xb = job.x + (b0 + b) * nn;
                float acc = 0.f;
                if (okr0 && okc0) acc = fmaf(w00, __ldg(xb + o00), acc);
                if (okr0 && okc1) acc = fmaf(w01, __ldg(xb + o00 + 1), acc);
                if (okr1 && okc0) acc = fmaf(w10, __ldg(xb + o00 + n), acc);
                if (okr1 && okc1) acc = fmaf(w11, __ldg(xb + o00 + n + 1), acc);
                v[b] = acc;
            }
        }
        if (job.out) {
#pragma unroll
            for (int b = 0; b < BB; ++b)
                if (b0 + b < a.B) job.out[(b0 + b) * nn + (long)r * n + c] = v[b];
        }
    }
    if (!job.xr && !job.xc) return;
    {
        float *tp = tile + tr * kRow + tc * BB;
        if constexpr (BB == 4) {
            *reinterpret_cast<float4 *>(tp) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int b = 0; b < BB; ++b) tp[b] = v[b];
        }
    }
    __syncthreads();
    const long grp_stride = (long)a.nblk * n * 32;  // floats per image group per class
    const int e = threadIdx.x;                    // 256 threads, one float each per pass
    if (job.xr) {
        // row-packed: for each tile column c, the tile's rows are consecutive line slots of
        // their block (R >= 8: one block, 8 x BB contiguous floats)
        float *dst = job.xr + blockIdx.y * grp_stride;
        for (int q = e; q < kTC * kTR * BB; q += kTR * kTC) {
            const int b = q % BB, l = (q / BB) % kTR, cc = q / (BB * kTR);
            const int row = r0 + l;
            if (c0 + cc < n)
                dst[((long)(row / R) * n + c0 + cc) * 32 + (row % R) * BB + b] =
                    tile[l * kRow + cc * BB + b];
        }
    }
    if (job.xc) {
        // col-packed: block c/R holds columns [R*(c/R), +R); rows r0..r0+7 of the tile are
        // contiguous pixel entries of 32 floats, of which this tile fills columns c0..c0+31
        float *dst = job.xc + blockIdx.y * grp_stride;
        for (int q = e; q < kTR * kTC * BB; q += kTR * kTC) {
            const int b = q % BB, cc = (q / BB) % kTC, l = q / (BB * kTC);
            const int col = c0 + cc, row = r0 + l;
            if (row < n && col < a.nblk * R) dst[((long)(col / R) * n + row) * 32 + (col % R) * BB + b] = tile[l * kRow + cc * BB + b];
        }
    }
}

}  // namespace

size_t pack_floats(const skei_plan *plan, int B, int bb) {
    const int R = 32 / bb;
    const long nblk = (plan->n + R - 1) / R;
    return (size_t)((B + bb - 1) / bb) * nblk * plan->n * 32;
}

cudaError_t launch_rotate_pack(const skei_plan *plan, const RotPackJob *jobs, int njobs, int B,
                               int bb, cudaStream_t s) {
    RotPackArgs a;
    a.job[0] = jobs[0];
    a.job[1] = njobs > 1 ? jobs[1] : jobs[0];
    a.n = plan->n;
    a.B = B;
    a.rot = plan->d_rot;
    const int R = 32 / bb;
    a.nblk = (plan->n + R - 1) / R;
    a.tiles_c = (plan->n + kTC - 1) / kTC;
    // rows: cover whole packed blocks (multiples of R) so padding lines are zero-filled
    const int rows = a.nblk * R;
    const int tiles_r = (rows + kTR - 1) / kTR;
    dim3 grid((unsigned)(tiles_r * a.tiles_c), (unsigned)((B + bb - 1) / bb), (unsigned)njobs);
    switch (bb) {
        case 4: k_rotate_pack<4><<<grid, kTR * kTC, 0, s>>>(a); break;
        case 2: k_rotate_pack<2><<<grid, kTR * kTC, 0, s>>>(a); break;
        default: k_rotate_pack<1><<<grid, kTR * kTC, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_rotate(const skei_plan *plan, const float *x, float *out, int B,
                          const int32_t *g, int g_stride, cudaStream_t s) {
    RotPackJob j{x, out, g, g_stride, nullptr, nullptr, nullptr};
    const int bb = B % 4 == 0 ? 4 : (B % 2 == 0 ? 2 : 1);
    return launch_rotate_pack(plan, &j, 1, B, bb, s);
}

}  // namespace skei
