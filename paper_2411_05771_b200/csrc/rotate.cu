// rotate.cu — a2: x2 = T_g x1 (EI group action of Eq. 4), bilinear,
// zero outside, about the image centre, counter-clockwise for g > 0 (R11).
//
// HBM-bound (8 bytes moved per output pixel, 4 taps).  Source coordinates are formed in
// fp64 once per output pixel and reused for every image sharing the same g; the four
// taps are read through the read-only path (neighbouring threads touch neighbouring
// source pixels, so L1 absorbs the 4x reuse).
#include "internal.h"

namespace skei {
namespace {

__device__ inline void cossin_deg(int g, double *c, double *s) {
    int gm = ((g % 360) + 360) % 360;
    if (gm == 0) { *c = 1.0; *s = 0.0; return; }
    if (gm == 90) { *c = 0.0; *s = 1.0; return; }
    if (gm == 180) { *c = -1.0; *s = 0.0; return; }
    if (gm == 270) { *c = 0.0; *s = -1.0; return; }
    sincospi((double)gm / 180.0, s, c);
}

// grid: x over pixels (256 per block), y over image groups of `ipb` images.
__global__ void __launch_bounds__(256) k_rotate(const float *__restrict__ x,
                                                float *__restrict__ out, int n, int B,
                                                const int32_t *__restrict__ gdeg, int g_stride,
                                                int ipb) {
    const long npix = (long)n * n;
    const long pix = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= npix) return;
    const int r = (int)(pix / n), c = (int)(pix - (long)r * n);
    const int b0 = blockIdx.y * ipb;
    const int b1 = min(B, b0 + ipb);
    const double h = (n - 1) * 0.5;
    double cg, sg;
    cossin_deg(gdeg[g_stride ? b0 : 0], &cg, &sg);
    const double u = c - h, v = h - r;
    const double us = u * cg + v * sg;
    const double vs = -u * sg + v * cg;
    const double cs = us + h, rs = h - vs;
    const double r0d = floor(rs), c0d = floor(cs);
    const float a = (float)(rs - r0d), bb = (float)(cs - c0d);
    const int r0 = (int)r0d, c0 = (int)c0d;
    const bool ok00 = r0 >= 0 && r0 < n && c0 >= 0 && c0 < n;
    const bool ok01 = r0 >= 0 && r0 < n && c0 + 1 >= 0 && c0 + 1 < n;
    const bool ok10 = r0 + 1 >= 0 && r0 + 1 < n && c0 >= 0 && c0 < n;
    const bool ok11 = r0 + 1 >= 0 && r0 + 1 < n && c0 + 1 >= 0 && c0 + 1 < n;
    const float w00 = (1.f - a) * (1.f - bb), w01 = (1.f - a) * bb;
    const float w10 = a * (1.f - bb), w11 = a * bb;
    const long o00 = (long)r0 * n + c0;
    for (int b = b0; b < b1; ++b) {
        const float *xb = x + (long)b * npix;
        float acc = 0.f;
        if (ok00) acc = fmaf(w00, __ldg(xb + o00), acc);
        if (ok01) acc = fmaf(w01, __ldg(xb + o00 + 1), acc);
        if (ok10) acc = fmaf(w10, __ldg(xb + o00 + n), acc);
        if (ok11) acc = fmaf(w11, __ldg(xb + o00 + n + 1), acc);
        out[(long)b * npix + pix] = acc;
    }
}

}  // namespace

cudaError_t launch_rotate(const skei_plan *plan, const float *x, float *out, int B,
                          const int32_t *g, int g_stride, cudaStream_t s) {
    const int n = plan->n;
    const long npix = (long)n * n;
    const int ipb = g_stride ? 1 : 8;
    dim3 grid((unsigned)((npix + 255) / 256), (unsigned)((B + ipb - 1) / ipb));
    k_rotate<<<grid, 256, 0, s>>>(x, out, n, B, g, g_stride, ipb);
    return cudaGetLastError();
}

}  // namespace skei
