// rotate.cu — a2: x2 = T_g x1 (EI group action of Eq. 4), bilinear,
// zero outside, about the image centre, counter-clockwise for g > 0 (R11), fused
// with the packing of the forward projector's input.
//
// k_rotate_pack: one CTA = a 32 x 32 pixel tile of BB images (BB = the image group of the
// forward projector), a thread per column and 4 rows.  Source coordinates in split precision: the tile origin's source
// position in fp64 (cos g, sin g from the plan's fp64 table of the 360 angles, exact at
// multiples of 90) plus an fp32 offset of <= 40 px per pixel, then 4 bilinear taps per
// image through the read-only path.  It writes, as requested:
//   * the plain rotated image out[b][r][c]                          (skei_rotate's output)
//   * the row-packed copy  xr[grp][r / R][c][r % R][b]  (R = 32 / BB lines per block)
//   * the col-packed copy  xc[grp][c / R][r][c % R][b]
// i.e. the image cut into blocks of R lines, each block stored pixel-major with the R lines
// x BB images of one pixel in 128 contiguous bytes — the layout k_radon_fwd stages with one
// TMA bulk copy per block.  Pixels outside the image (the last block's
// padding lines) are written as zeros.  The identity job (g = 0, no taps) packs x1.  With a
// shared g the BB images share one set of taps per pixel; for |sin g| > |cos g| a warp's
// lanes take 32 rows of one column (taps stay within a few cache lines).  A shared g on a
// group of 4 instead stages the tile's source footprint (<= 47 x 47 pixels, zero outside the
// image) in shared memory, 4 images interleaved per pixel, so each tap is one LDS.128 with
// no bounds predicates (same weights and FMA order).  Behind the pass's
// own draw kernel (skei_pass_draw) the launch is programmatically serialised: only the
// rotation job waits (griddepcontrol.wait) for g.
#include "internal.h"

namespace skei {
namespace {

constexpr int kT = 32;          // tile side (pixels)
constexpr int kThreads = 256;   // 32 columns x 8 row groups; a thread owns 4 rows
// staged rotation (shared g, groups of 4): the tile's source footprint, <= 31 (|cos| + |sin|)
// + 2 taps + 2 guard pixels <= 47 per side, staged as [row][col][image] with an odd pixel
// pitch (16-byte slots: a quarter-warp's bilinear taps spread over the bank groups)
constexpr int kSrc = 48, kSrcPitch = 49;
constexpr int kStageF = kSrc * kSrcPitch * 4;
#ifndef SKEI_ROT_MINB
#define SKEI_ROT_MINB 5  // CTAs per SM the rotate + pack kernel's registers must allow (A/B knob)
#endif
#ifndef SKEI_ROT_STAGED
#define SKEI_ROT_STAGED 1  // shared-g rotations of groups of 4 via the staged footprint (A/B knob)
#endif

struct RotOrigin {
    int bc, br;      // integer part of the tile origin's source column / row
    float fc, fr;    // fractional parts
    float cg, sg;    // cos g, sin g
};

template <int BB>
struct VecT;
template <> struct VecT<1> { using T = float; };
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<4> { using T = float4; };

// XM: the identity job packs ascale * (x - xm) (a separate instantiation, so the pass's
// rotation + packing is compiled without it)
template <int BB, bool XM>
__global__ void __launch_bounds__(kThreads, SKEI_ROT_MINB) k_rotate_pack(RotPackArgs a) {
    constexpr int R = 32 / BB;
    using V = typename VecT<BB>::T;
    constexpr int kRow = kT * BB + 4;  // padded tile row (floats)
    // the output tile (packing) — overlaid, in the staged rotation, on the source footprint
    constexpr int kSmemF = kStageF > kT * kRow ? kStageF : kT * kRow;
    __shared__ __align__(16) float smraw[kSmemF];
    float *const tile = smraw;
    __shared__ RotOrigin sRot[BB];
    const RotPackJob job = blockIdx.z ? a.job[1] : a.job[0];
    const int n = a.n;
    const int tc = threadIdx.x & 31, tr = threadIdx.x >> 5;
    const int r0 = blockIdx.x / a.tiles_c * kT, c0 = blockIdx.x % a.tiles_c * kT;
    const int b0 = blockIdx.y * BB;
    const long nn = (long)n * n;
    if (job.zero && blockIdx.x == 0 && blockIdx.y == 0)  // the pass's counters (fused
        for (int t = threadIdx.x; t < kPassCounters; t += blockDim.x) job.zero[t] = 0u;  // reductions, forward split units)
    // launched programmatically behind the pass's own k_draw (skei_pass_draw): only the
    // rotation job reads the draw (g), so only its blocks wait for the draw grid; the
    // packing of x1 runs while the draw is still in flight
    if (a.pdl && job.g != nullptr) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (job.g != nullptr && threadIdx.x < BB && b0 + (int)threadIdx.x < a.B) {
        // source position of the tile origin (r0, c0) for image b0 + threadIdx.x, in fp64:
        // c' = h + (c0 - h) cos g + (h - r0) sin g,  r' = h + (c0 - h) sin g - (h - r0) cos g
        const int gd = job.g[job.g_stride ? b0 + threadIdx.x : 0];
        const double2 csg = a.rot[((gd % 360) + 360) % 360];  // exact at multiples of 90
        const double h = (n - 1) * 0.5, u = c0 - h, w = h - r0;
        const double cs = h + u * csg.x + w * csg.y;
        const double rs = h + u * csg.y - w * csg.x;
        const double fc = floor(cs), fr = floor(rs);
        sRot[threadIdx.x] = RotOrigin{(int)fc, (int)fr, (float)(cs - fc), (float)(rs - fr),
                                      (float)csg.x, (float)csg.y};
    }
    __syncthreads();

    // Rotations nearer a quarter turn (|sin g| > |cos g|) map a warp's 32 lanes to 32 rows
    // of one tile column: consecutive source positions then step by |cos g| < |sin g| rows
    // (instead of |sin g| per column), so a warp's bilinear taps stay within a few cache
    // lines; the plain output is then written from the staged tile (coalesced)
    const bool staged = SKEI_ROT_STAGED && BB == 4 && !XM && job.g != nullptr && job.g_stride == 0;
    const bool swp = !staged && job.g != nullptr && fabsf(sRot[0].sg) > fabsf(sRot[0].cg);
    if (staged) {
        // ---- staged rotation: the source footprint of the output tile, zero outside the
        // image, is copied once (coalesced rows, 4 images interleaved per pixel); every
        // bilinear tap is then one LDS.128 for the 4 images, with no bounds predicates.
        // Same weights, same FMA order as the direct path (outside taps add w * 0).
        const RotOrigin o = sRot[0];
        const float e = 31.f;
        const float cmn = o.fc + fminf(0.f, e * o.cg) + fminf(0.f, -e * o.sg);
        const float rmn = o.fr + fminf(0.f, e * o.sg) + fminf(0.f, e * o.cg);
        const int clo = o.bc + (int)floorf(cmn) - 1, rlo = o.br + (int)floorf(rmn) - 1;
        // every load of the footprint is issued before the first store (9 x 4 in flight per
        // thread instead of 4: the loop was 9 serialised DRAM round trips)
        constexpr int kIt = (kSrc * kSrc + kThreads - 1) / kThreads;
        float4 t[kIt];
#pragma unroll
        for (int q = 0; q < kIt; ++q) {
            const int it = threadIdx.x + q * kThreads;
            const int i = it / kSrc, j = it - i * kSrc;
            const int r = rlo + i, c = clo + j;
            t[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (it < kSrc * kSrc && r >= 0 && r < n && c >= 0 && c < n) {
                const float *xp = job.x + (long)b0 * nn + (long)r * n + c;
                t[q].x = __ldg(xp);
                if (b0 + 1 < a.B) t[q].y = __ldg(xp + nn);
                if (b0 + 2 < a.B) t[q].z = __ldg(xp + 2 * nn);
                if (b0 + 3 < a.B) t[q].w = __ldg(xp + 3 * nn);
            }
        }
#pragma unroll
        for (int q = 0; q < kIt; ++q) {
            const int it = threadIdx.x + q * kThreads;
            const int i = it / kSrc, j = it - i * kSrc;
            if (it < kSrc * kSrc) *reinterpret_cast<float4 *>(smraw + (i * kSrcPitch + j) * 4) = t[q];
        }
        __syncthreads();
        float4 res[kT / 8];
#pragma unroll
        for (int i = 0; i < kT / 8; ++i) {
            const int rr = tr + 8 * i, cc = tc;
            const float dr = (float)rr, dc = (float)cc;
            const float cl = o.fc + fmaf(dc, o.cg, -dr * o.sg);
            const float rl = o.fr + fmaf(dc, o.sg, dr * o.cg);
            const float flc = floorf(cl), flr = floorf(rl);
            const float fb = cl - flc, fa = rl - flr;
            const int ci = o.bc + (int)flc - clo, ri = o.br + (int)flr - rlo;
            SKEI_DCHECK(ci >= 0 && ci + 1 < kSrc && ri >= 0 && ri + 1 < kSrc, "rotation footprint");
            const float *sp = smraw + (ri * kSrcPitch + ci) * 4;
            const float4 x00 = *reinterpret_cast<const float4 *>(sp);
            const float4 x01 = *reinterpret_cast<const float4 *>(sp + 4);
            const float4 x10 = *reinterpret_cast<const float4 *>(sp + kSrcPitch * 4);
            const float4 x11 = *reinterpret_cast<const float4 *>(sp + kSrcPitch * 4 + 4);
            const float w00 = (1.f - fa) * (1.f - fb), w01 = (1.f - fa) * fb;
            const float w10 = fa * (1.f - fb), w11 = fa * fb;
            float4 v;
            v.x = fmaf(w11, x11.x, fmaf(w10, x10.x, fmaf(w01, x01.x, fmaf(w00, x00.x, 0.f))));
            v.y = fmaf(w11, x11.y, fmaf(w10, x10.y, fmaf(w01, x01.y, fmaf(w00, x00.y, 0.f))));
            v.z = fmaf(w11, x11.z, fmaf(w10, x10.z, fmaf(w01, x01.z, fmaf(w00, x00.z, 0.f))));
            v.w = fmaf(w11, x11.w, fmaf(w10, x10.w, fmaf(w01, x01.w, fmaf(w00, x00.w, 0.f))));
            const int r = r0 + rr, c = c0 + cc;
            if (r >= n || c >= n) v = make_float4(0.f, 0.f, 0.f, 0.f);
            res[i] = v;
            if (job.out && r < n && c < n) {
                const long o2 = (long)b0 * nn + (long)r * n + c;
                job.out[o2] = v.x;
                if (b0 + 1 < a.B) job.out[o2 + nn] = v.y;
                if (b0 + 2 < a.B) job.out[o2 + 2 * nn] = v.z;
                if (b0 + 3 < a.B) job.out[o2 + 3 * nn] = v.w;
            }
        }
        __syncthreads();  // footprint reads done: the tile overlays it
#pragma unroll
        for (int i = 0; i < kT / 8; ++i)
            *reinterpret_cast<float4 *>(tile + (tr + 8 * i) * kRow + tc * BB) = res[i];
    } else if (job.g == nullptr && !XM) {
        // identity (pack x1): all 4 x BB loads in flight before the tile stores
        float v[kT / 8][BB];
#pragma unroll
        for (int i = 0; i < kT / 8; ++i) {
            const int r = r0 + tr + 8 * i, c = c0 + tc;
#pragma unroll
            for (int b = 0; b < BB; ++b)
                v[i][b] = (r < n && c < n && b0 + b < a.B) ? __ldg(job.x + (b0 + b) * nn + (long)r * n + c) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < kT / 8; ++i) {
            V t;
            float *tp = reinterpret_cast<float *>(&t);
#pragma unroll
            for (int b = 0; b < BB; ++b) tp[b] = v[i][b];
            *reinterpret_cast<V *>(tile + (tr + 8 * i) * kRow + tc * BB) = t;
        }
    } else {
#pragma unroll
    for (int i = 0; i < kT / 8; ++i) {
        const int rr = swp ? tc : tr + 8 * i, r = r0 + rr;
        const int cc = swp ? tr + 8 * i : tc, c = c0 + cc;
        float v[BB];
#pragma unroll
        for (int b = 0; b < BB; ++b) v[b] = 0.f;
        if (r < n && c < n) {
            if (job.g == nullptr) {  // identity (pack x1)
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    if (b0 + b < a.B) v[b] = __ldg(job.x + (b0 + b) * nn + (long)r * n + c);
                if (XM && job.xm) {  // d = ascale (x - xm) (the EI gradient's 2 (x2 - x3))
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        if (b0 + b < a.B)
                            v[b] = job.ascale * (v[b] - __ldg(job.xm + (b0 + b) * nn + (long)r * n + c));
                }
            } else {
                // split-precision source coordinates: the tile origin's source position
                // (fp64, sRot) plus an fp32 offset of at most 2 x 32 pixels
                const float dr = (float)rr, dc = (float)cc;
                float fa = 0.f, fb = 0.f;
                int ci = 0, ri = 0;
                bool okr0 = false, okr1 = false, okc0 = false, okc1 = false;
#pragma unroll
                for (int b = 0; b < BB; ++b) {
                    if (b0 + b >= a.B) continue;
                    if (b == 0 || job.g_stride) {  // a shared g: the BB images share the taps
                        const RotOrigin o = sRot[job.g_stride ? b : 0];
                        const float cl = o.fc + fmaf(dc, o.cg, -dr * o.sg);
                        const float rl = o.fr + fmaf(dc, o.sg, dr * o.cg);
                        const float flc = floorf(cl), flr = floorf(rl);
                        fb = cl - flc;
                        fa = rl - flr;
                        ci = o.bc + (int)flc;
                        ri = o.br + (int)flr;
                        okr0 = ri >= 0 && ri < n;
                        okr1 = ri + 1 >= 0 && ri + 1 < n;
                        okc0 = ci >= 0 && ci < n;
                        okc1 = ci + 1 >= 0 && ci + 1 < n;
                    }
                    const float *xb = job.x + (b0 + b) * nn + (long)ri * n + ci;
                    float acc = 0.f;
                    if (okr0 && okc0) acc = fmaf((1.f - fa) * (1.f - fb), __ldg(xb), acc);
                    if (okr0 && okc1) acc = fmaf((1.f - fa) * fb, __ldg(xb + 1), acc);
                    if (okr1 && okc0) acc = fmaf(fa * (1.f - fb), __ldg(xb + n), acc);
                    if (okr1 && okc1) acc = fmaf(fa * fb, __ldg(xb + n + 1), acc);
                    v[b] = acc;
                }
            }
            if (job.out && !swp) {
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    if (b0 + b < a.B) job.out[(b0 + b) * nn + (long)r * n + c] = v[b];
            }
        }
        V t;
        float *tp = reinterpret_cast<float *>(&t);
#pragma unroll
        for (int b = 0; b < BB; ++b) tp[b] = v[b];
        *reinterpret_cast<V *>(tile + rr * kRow + cc * BB) = t;
    }
    }
    const bool late_out = swp && job.out;
    if (!job.xr && !job.xc && !late_out) return;
    __syncthreads();
    if (late_out) {  // plain output of a transposed-mapping tile, row by row
        const int c = c0 + tc;
#pragma unroll
        for (int i = 0; i < kT / 8; ++i) {
            const int rr = tr + 8 * i, r = r0 + rr;
            if (r >= n || c >= n) continue;
            const V t = *reinterpret_cast<const V *>(tile + rr * kRow + tc * BB);
            const float *tp = reinterpret_cast<const float *>(&t);
#pragma unroll
            for (int b = 0; b < BB; ++b)
                if (b0 + b < a.B) job.out[(b0 + b) * nn + (long)r * n + c] = tp[b];
        }
    }
    if (BB == 1 && a.fuse) {
        // job-fused layout (one image, its two jobs x1 / x2 as the two slots of a group of
        // 2): blocks of 16 lines, [block][pixel][line][slot], this job's slot = blockIdx.z
        constexpr int RF = 16;
        const long grp = (long)blockIdx.y * a.nblk * n * 32;
        const int lim = a.nblk * RF, slot = blockIdx.z;
        if (job.xr)
            for (int it = threadIdx.x; it < kT * kT; it += kThreads) {
                const int rl = it % RF, rest = it / RF;
                const int cc = rest % kT, rr = rest / kT * RF + rl;
                const int r = r0 + rr, cg = c0 + cc;
                if (r < lim && cg < n)
                    job.xr[grp + ((long)(r / RF) * n + cg) * 32 + (r % RF) * 2 + slot] = tile[rr * kRow + cc];
            }
        if (job.xc)
            for (int it = threadIdx.x; it < kT * kT; it += kThreads) {
                const int cl = it % RF, rest = it / RF;
                const int rr = rest % kT, cc = rest / kT * RF + cl;
                const int r = r0 + rr, cg = c0 + cc;
                if (r < n && cg < lim)
                    job.xc[grp + ((long)(cg / RF) * n + r) * 32 + (cg % RF) * 2 + slot] = tile[rr * kRow + cc];
            }
        return;
    }
    const long grp = (long)blockIdx.y * a.nblk * n * 32;  // floats per image group per class
    const int lim = a.nblk * R;                            // packed lines (incl. zero padding)
    if (R == 8 && r0 + kT <= lim && c0 + kT <= n && r0 + kT <= n && c0 + kT <= lim) {
        // interior tile (BB = 4): for a fixed block of 8 lines the tile's 32 pixels x 8 lines
        // are 4 KB of contiguous packed output, so thread t stores the 16-byte slot t of each
        // of the 4 blocks (pixel t / 8, line t % 8): one LDS.128 + one STG.128 per slot, the
        // addresses one add apart (no per-slot index arithmetic or bounds checks)
        const int px = threadIdx.x >> 3, ln = threadIdx.x & 7;
        if (job.xr) {  // row blocks r0 / 8 + rb: pixel = column c0 + px, line = row rb * 8 + ln
            V *dst = reinterpret_cast<V *>(job.xr + grp + ((long)(r0 >> 3) * n + c0) * 32) + threadIdx.x;
            const float *src = tile + ln * kRow + px * BB;
#pragma unroll
            for (int rb = 0; rb < kT / 8; ++rb)
                dst[(long)rb * n * 8] = *reinterpret_cast<const V *>(src + rb * 8 * kRow);
        }
        if (job.xc) {  // column blocks c0 / 8 + cb: pixel = row r0 + px, line = column cb * 8 + ln
            V *dst = reinterpret_cast<V *>(job.xc + grp + ((long)(c0 >> 3) * n + r0) * 32) + threadIdx.x;
            const float *src = tile + px * kRow + ln * BB;
#pragma unroll
            for (int cb = 0; cb < kT / 8; ++cb)
                dst[(long)cb * n * 8] = *reinterpret_cast<const V *>(src + cb * 8 * BB);
        }
        return;
    }
    // each item is one pixel-line slot of BB floats (16 / 8 / 4 bytes); consecutive threads
    // take consecutive slots of a packed 128-byte pixel column
    if (job.xr) {  // row-packed: block r / R, pixel c, line r % R
        for (int it = threadIdx.x; it < kT * kT; it += kThreads) {
            const int rl = it % R, rest = it / R;
            const int cc = rest % kT, rb = rest / kT;  // rows rb*R .. +R-1 of the tile
            const int rr = rb * R + rl;
            if (rr >= kT) continue;
            const int r = r0 + rr, cg = c0 + cc;
            if (r < lim && cg < n)
                *reinterpret_cast<V *>(job.xr + grp + ((long)(r / R) * n + cg) * 32 + (r % R) * BB) =
                    *reinterpret_cast<const V *>(tile + rr * kRow + cc * BB);
        }
    }
    if (job.xc) {  // col-packed: block c / R, pixel r, line c % R
        for (int it = threadIdx.x; it < kT * kT; it += kThreads) {
            const int cl = it % R, rest = it / R;
            const int rr = rest % kT, cb = rest / kT;
            const int cc = cb * R + cl;
            if (cc >= kT) continue;
            const int r = r0 + rr, cg = c0 + cc;
            if (r < n && cg < lim)
                *reinterpret_cast<V *>(job.xc + grp + ((long)(cg / R) * n + r) * 32 + (cg % R) * BB) =
                    *reinterpret_cast<const V *>(tile + rr * kRow + cc * BB);
        }
    }
}

// k_rotate_adj: out = T_g^T y, the transpose of the rotation, as a
// GATHER (no atomics): input pixel p = (rp, cp) receives w * y[o] from every output pixel
// o whose source position (r', c') has p among its 4 bilinear neighbours, with w the
// bilinear weight o gives p.  Those o lie in the image of the square |r' - rp| < 1,
// |c' - cp| < 1 under the inverse rotation, whose bounding box has half-width
// |cos g| + |sin g| <= sqrt 2: a 4 x 4 candidate window around p's inverse image.  Source
// positions in split precision as in k_rotate_pack: a reference output pixel near the
// tile's inverse image has its source position in fp64 (integer part + fp32 fraction), each
// candidate adds an fp32 offset of <= ~50 px (exact at quarter turns); the weight is
// nonzero only if p is one of the candidate's neighbours.  One thread per pixel and 4 rows,
// the BB images of a group share the weights when g is shared.
struct AdjRef {
    int ro, co;      // the reference output pixel
    int ri, ci;      // integer parts of its source position (r', c')
    float rf, cf;    // fractional parts
    float cg, sg;    // cos g, sin g
    float uo0, vo0;  // inverse image of the tile origin pixel, relative to (ro, co)
};
template <int BB>
__global__ void __launch_bounds__(kThreads) k_rotate_adj(const float *y, float *out, int n, int B,
                                                         const int32_t *g, int g_stride,
                                                         const double2 *rot, int tiles_c) {
    __shared__ AdjRef sref;
    const int tc = threadIdx.x & 31, tr = threadIdx.x >> 5;
    const int r0 = blockIdx.x / tiles_c * kT, c0 = blockIdx.x % tiles_c * kT;
    const int b0 = blockIdx.y * BB;
    const long nn = (long)n * n;
    const int c = c0 + tc;
    const int nimg = g_stride ? 1 : BB;  // images sharing one rotation per weight pass
#pragma unroll 1
    for (int bs = 0; bs < BB; bs += nimg) {
        if (b0 + bs >= B) break;
        if (threadIdx.x == 0) {
            const int gd = g[g_stride ? b0 + bs : 0];
            const double2 csg = rot[((gd % 360) + 360) % 360];  // exact at multiples of 90
            const double cg = csg.x, sg = csg.y, h = (n - 1) * 0.5;
            // inverse image of the tile origin pixel (r0, c0): the reference output pixel
            const double up = c0 - h, vp = h - r0;
            const double uo = up * cg - vp * sg, vo = up * sg + vp * cg;
            AdjRef rf;
            rf.co = (int)floor(uo + h);
            rf.ro = (int)floor(h - vo);
            // its source position (the forward definition), split
            const double u = rf.co - h, v = h - rf.ro;
            const double cs = u * cg + v * sg + h, rs = h - (-u * sg + v * cg);
            const double fcs = floor(cs), frs = floor(rs);
            rf.ci = (int)fcs;
            rf.ri = (int)frs;
            rf.cf = (float)(cs - fcs);
            rf.rf = (float)(rs - frs);
            rf.cg = (float)cg;
            rf.sg = (float)sg;
            rf.uo0 = (float)(uo + h - rf.co);  // column of the tile origin's inverse image
            rf.vo0 = (float)(h - vo - rf.ro);  // row
            sref = rf;
        }
        __syncthreads();
        const AdjRef rf = sref;
        const float wbox = fabsf(rf.cg) + fabsf(rf.sg);
#pragma unroll 1
        for (int i = 0; i < kT / 8; ++i) {
            const int rr = tr + 8 * i, r = r0 + rr;
            if (r >= n || c >= n) continue;
            // p's inverse image relative to the reference: origin's + the rotated offset
            const float dpc = (float)tc, dpr = (float)rr;
            const float ocf = rf.uo0 + fmaf(dpc, rf.cg, dpr * rf.sg);   // d u_o / d c = cos, d u_o / d r = sin
            const float orf = rf.vo0 + fmaf(-dpc, rf.sg, dpr * rf.cg);  // d r_o / d c = -sin, d r_o / d r = cos
            const int ocmin = rf.co + (int)floorf(ocf - wbox), ormin = rf.ro + (int)floorf(orf - wbox);
            float acc[BB];
#pragma unroll
            for (int b = 0; b < BB; ++b) acc[b] = 0.f;
#pragma unroll
            for (int dr = 0; dr < 4; ++dr) {
                const int ro = ormin + dr;
                if (ro < 0 || ro >= n) continue;
#pragma unroll
                for (int dc = 0; dc < 4; ++dc) {
                    const int co = ocmin + dc;
                    if (co < 0 || co >= n) continue;
                    // source position of output pixel (ro, co): reference + fp32 offset
                    const float oc = (float)(co - rf.co), orr = (float)(ro - rf.ro);
                    const float cl = rf.cf + fmaf(oc, rf.cg, -orr * rf.sg);
                    const float rl = rf.rf + fmaf(oc, rf.sg, orr * rf.cg);
                    const float flc = floorf(cl), flr = floorf(rl);
                    const int er = r - (rf.ri + (int)flr), ec = c - (rf.ci + (int)flc);
                    if (er < 0 || er > 1 || ec < 0 || ec > 1) continue;
                    const float a = rl - flr, bb = cl - flc;
                    const float w = (er ? a : 1.f - a) * (ec ? bb : 1.f - bb);
                    const long oo = (long)ro * n + co;
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        if (b < nimg && b0 + bs + b < B)
                            acc[b] = fmaf(w, __ldg(y + (b0 + bs + b) * nn + oo), acc[b]);
                }
            }
#pragma unroll
            for (int b = 0; b < BB; ++b)
                if (b < nimg && b0 + bs + b < B) out[(b0 + bs + b) * nn + (long)r * n + c] = acc[b];
        }
        __syncthreads();  // sref is rewritten by the next image's pass
    }
}

}  // namespace

cudaError_t launch_rotate_adj(const skei_plan *plan, const float *y, float *out, int B,
                              const int32_t *g, int g_stride, cudaStream_t s) {
    const int n = plan->n;
    const int tiles_c = (n + kT - 1) / kT;
    const int bb = g_stride ? 1 : (B % 4 == 0 ? 4 : (B % 2 == 0 ? 2 : 1));
    dim3 grid((unsigned)(tiles_c * tiles_c), (unsigned)((B + bb - 1) / bb), 1);
    switch (bb) {
        case 4: k_rotate_adj<4><<<grid, kThreads, 0, s>>>(y, out, n, B, g, g_stride, plan->d_rot, tiles_c); break;
        case 2: k_rotate_adj<2><<<grid, kThreads, 0, s>>>(y, out, n, B, g, g_stride, plan->d_rot, tiles_c); break;
        default: k_rotate_adj<1><<<grid, kThreads, 0, s>>>(y, out, n, B, g, g_stride, plan->d_rot, tiles_c); break;
    }
    return cudaGetLastError();
}

size_t pack_floats(const skei_plan *plan, int B, int bb) {
    const int R = 32 / bb;
    const long nblk = (plan->n + R - 1) / R;
    return (size_t)((B + bb - 1) / bb) * nblk * plan->n * 32;
}

cudaError_t launch_rotate_pack(const skei_plan *plan, const RotPackJob *jobs, int njobs, int B,
                               int bb, cudaStream_t s, bool pdl, bool fuse) {
    if (fuse && (bb != 1 || njobs != 2)) return cudaErrorInvalidValue;
    RotPackArgs a;
    a.pdl = pdl ? 1 : 0;
    a.fuse = fuse ? 1 : 0;
    a.job[0] = jobs[0];
    a.job[1] = njobs > 1 ? jobs[1] : jobs[0];
    a.n = plan->n;
    a.B = B;
    a.rot = plan->d_rot;
    const int R = fuse ? 16 : 32 / bb;  // lines per packed block (fused: 2 slots per line)
    a.nblk = (plan->n + R - 1) / R;
    // tiles cover the image and every packed line (incl. the zero padding lines)
    const int side = a.nblk * R > plan->n ? a.nblk * R : plan->n;
    a.tiles_c = (side + kT - 1) / kT;
    dim3 grid((unsigned)(a.tiles_c * a.tiles_c), (unsigned)((B + bb - 1) / bb), (unsigned)njobs);
    const bool xm = a.job[0].xm || (njobs > 1 && a.job[1].xm);
    // pdl: programmatic stream serialization (the kernel may start once the previous grid,
    // the pass's k_draw, has triggered; the rotation job waits for its completion)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
#define SKEI_ROTPACK(BBV)                                                       \
    do {                                                                        \
        cudaError_t e_ = xm ? cudaLaunchKernelEx(&cfg, k_rotate_pack<BBV, true>, a)  \
                            : cudaLaunchKernelEx(&cfg, k_rotate_pack<BBV, false>, a); \
        if (e_ != cudaSuccess) return e_;                                       \
    } while (0)
    switch (bb) {
        case 4: SKEI_ROTPACK(4); break;
        case 2: SKEI_ROTPACK(2); break;
        default: SKEI_ROTPACK(1); break;
    }
#undef SKEI_ROTPACK
    return cudaGetLastError();
}

cudaError_t launch_rotate(const skei_plan *plan, const float *x, float *out, int B,
                          const int32_t *g, int g_stride, cudaStream_t s) {
    RotPackJob j{x, out, g, g_stride, nullptr, nullptr, nullptr};
    const int bb = B % 4 == 0 ? 4 : (B % 2 == 0 ? 2 : 1);
    return launch_rotate_pack(plan, &j, 1, B, bb, s);
}

}  // namespace skei
