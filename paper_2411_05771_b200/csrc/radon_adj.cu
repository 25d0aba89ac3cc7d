// radon_adj.cu — a5/a8: x = scale * A_S^T p, the exact transpose of the pixel-driven
// projector (BASELINE.json north_star: "radon_adj is its exact transpose, a per-pixel
// gather over angles with the sketched angle table in shared memory").
//
// Design (DESIGN.md §7 "k_radon_adj"):
//   * One CTA = a 32 x 16 pixel tile x BB images sharing one angle list x all jobs of the
//     launch (the pass runs the FBP of q and the MC gradient of r as two jobs: they share
//     the geometry, so it is computed once for 2*BB images); 256 threads, 4 CTAs per SM.
//   * Each thread owns one pair of horizontally adjacent pixels (c, c+1) of one row.  The
//     detector positions t and t + cos(th) of a pair lie within one 3-bin window [j, j+3),
//     so a pair reads 3 bins per job (not 4) and interpolates each pixel with the 3 hat
//     weights max(0, 1 - |t - j - k|) (one of which is 0).
//   * Angles are processed in chunks of KC.  For each angle the CTA stages the W-bin detector
//     window of the tile, interleaved [bin][image] (one LDS.128 = a bin of 4 images), zero
//     outside [0, n_det) so dropped taps need no branch; double-buffered.  In the fused pass
//     (BULK) each window is one bulk copy from interleaved zero-padded copies of q and r that
//     warp 0 issues two chunks ahead (one barrier per chunk); standalone calls stage them
//     from the plain sinograms with cp.async.
//   * Bank-conflict-free gathers: the 8 lanes of a shared-memory phase are 8 consecutive rows
//     of one pixel column pair; their bins move by |sin th| <= 1 per row, so they span <= 8
//     consecutive 16-byte slots (distinct banks, equal slots broadcast).
//   * Positions in split precision: the fp64 tile-origin position per angle plus an fp32
//     local offset < 40 px.
//   * Optional fused epilogue (skei_pass with the identity network): ei partial sums
//     sum (x2 - x_fbp)^2 per tile and image, reduced in fixed order by the last CTA.
// Work per (pixel, angle, image) = 2 taps; per pixel pair and angle 3 LDS.BB per job.
//   * k_radon_adj_quad (below): the same with FOUR adjacent pixels per thread (one 5-bin
//     window per angle and job serves them; 32 x 32 tiles) — used wherever its grid fills a
//     wave, and for the job-fused groups; the pair kernel serves the small grids.
#include <type_traits>

#include "internal.h"
#include "tma.h"

namespace skei {
namespace {

constexpr int kTileW = 32;     // tile width (columns)
constexpr int kTileH = 16;     // tile height (rows)
constexpr int kThreads = 256;  // 8 warps: warp = 8 rows x 8 columns (4 pixel pairs)
constexpr int kPairs = 1;      // pixel pairs per thread
constexpr int kKC = 12;        // angles per staged chunk (2 buffers x 2 jobs fit 48 KB)
constexpr int kW = 40;         // staged bins per angle (>= sqrt(31^2 + 15^2) + 3)
constexpr int kTab = 256;      // m <= kTab: the whole per-angle table is built up front

struct AdjArgs {
    AdjJob job[2];
    const int32_t *idx;
    int m, idx_stride, B, tiles_x, tiles_y;
    int row0, row1;  // output rows [row0, row1) (a row band; [0, n) for whole images); the
                     // outputs (and base) are [B][row1 - row0][n], x2 of the fused ei [B][n][n]
    Geom g;
    // fused ei epilogue (job 0 = FBP): x2 [B][n][n], partials [B][ntiles], counter, ei [B]
    const float *ei_x2;
    float *ei_part;
    unsigned *ei_ctr;
    float *ei_out;
    AdjRs rs;  // reduce-scatter epilogue (rs.world > 0): outputs go to the row owners' slots
};

// where output (job jx, image img, row r, column c) is stored: the job's [B][row1 - row0][n]
// output, or with the reduce-scatter epilogue the slot of r's band owner (P2P)
__device__ __forceinline__ float *out_at(const AdjArgs &a, float *x, int jx, int img, int r,
                                         int c, long &ox) {
    const int n = a.g.n;
    if (a.rs.world == 0) {
        ox = (long)img * (a.row1 - a.row0) * n + (long)(r - a.row0) * n + c;
        return x;
    }
    const int q = n / a.rs.world, rem = n - q * a.rs.world;
    const int o = r < rem * (q + 1) ? r / (q + 1) : rem + (r - rem * (q + 1)) / q;
    const int start = o * q + min(o, rem);
    ox = ((long)(jx * a.B + img) * a.rs.bmax + (r - start)) * n + c;
    return a.rs.peer[o];
}

template <int BB>
struct Vec;
template <> struct Vec<1> { using T = float; };
template <> struct Vec<2> { using T = float2; };
template <> struct Vec<4> { using T = float4; };

template <int BB>
__device__ __forceinline__ void load_bins(const float *base, float (&v)[BB]) {
    typename Vec<BB>::T t = *reinterpret_cast<const typename Vec<BB>::T *>(base);
    const float *pt = reinterpret_cast<const float *>(&t);
#pragma unroll
    for (int b = 0; b < BB; ++b) v[b] = pt[b];
}

__device__ __forceinline__ void cp_async4(float *smem, const float *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// acc += w0 q0 + w1 q1 + w2 q2 over BB images (in that order), as packed fp32x2 FMAs
// (bitwise the same as the scalar fmaf chain)
template <int BB>
__device__ __forceinline__ void tap3(float (&acc)[BB], float w0, float w1, float w2,
                                     const float (&q0)[BB], const float (&q1)[BB],
                                     const float (&q2)[BB]) {
    if constexpr (BB == 1) {
        acc[0] = fmaf(w2, q2[0], fmaf(w1, q1[0], fmaf(w0, q0[0], acc[0])));
    } else {
#pragma unroll
        for (int b = 0; b < BB; b += 2) {
            float2 r = make_float2(acc[b], acc[b + 1]);
            r = __ffma2_rn(make_float2(w0, w0), make_float2(q0[b], q0[b + 1]), r);
            r = __ffma2_rn(make_float2(w1, w1), make_float2(q1[b], q1[b + 1]), r);
            r = __ffma2_rn(make_float2(w2, w2), make_float2(q2[b], q2[b + 1]), r);
            acc[b] = r.x;
            acc[b + 1] = r.y;
        }
    }
}

// hat weights of a position u in [0, 2] against bins 0, 1, 2
__device__ __forceinline__ void hat3(float u, float &w0, float &w1, float &w2) {
    w0 = fmaxf(0.f, 1.f - u);
    w1 = 1.f - fabsf(u - 1.f);
    w2 = fmaxf(0.f, u - 1.f);
}

// BULK: every job's windows are bulk copies from its interleaved padded sinogram (BB = 4).
// FUSED (BB = 2, NJ = 1, BULK): one image per CTA, its two jobs (q -> x_fbp, r -> grad) are
// the group's two slots, staged from the fused interleaved rows [b][k][pad + j][2] (window
// origins even, so every copy is 16-byte aligned); slot b writes job b's output.
template <int BB, int NJ, bool BULK, bool FUSED = false>
__global__ void __launch_bounds__(kThreads, 4) k_radon_adj(AdjArgs a) {
    __shared__ __align__(128) float win[2][NJ][kKC * kW * BB];
    // per-angle table: entry k of the sketch at [k] when m <= kTab (built once, by all
    // threads), else entry t of chunk ch at [(ch & 1) * kKC + t] (built per chunk)
    __shared__ float s_off[kTab], s_cos[kTab], s_sin[kTab];
    __shared__ int s_w0[kTab];
    __shared__ float s_red[kThreads / 32][BB];
    __shared__ bool s_last;
    __shared__ __align__(8) uint64_t full[2];  // BULK: window copies of each buffer landed

    const int n = a.g.n, n_det = a.g.n_det;
    const int tile = blockIdx.x;
    const int tr0 = a.row0 + (tile / a.tiles_x) * kTileH, tc0 = (tile % a.tiles_x) * kTileW;
    const int b0 = FUSED ? blockIdx.y : blockIdx.y * BB;  // first image (fused: the image)
    const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp w: rows 8*(w/2) .. +7, pixel pairs 8*(w%2) .. +7; lane: row (lane % 8), pairs
    // (lane / 8) and (lane / 8) + 4 — the 8 lanes of a quarter-warp are 8 consecutive rows
    // of one pair
    const int ry = 8 * (warp & 1) + (lane & 7);
    const int pc0 = 4 * (warp >> 1) + (lane >> 3);  // pair index 0..15
    const long nn = (long)n * n;

    float acc[NJ][kPairs][2][BB];  // [job][pair][pixel][image]
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int p = 0; p < kPairs; ++p)
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int b = 0; b < BB; ++b) acc[j][p][q][b] = 0.f;

    const int nchunks = (a.m + kKC - 1) / kKC;
    if constexpr (BULK) {
        if (threadIdx.x == 0) {
            mbar_init(&full[0], 1);
            mbar_init(&full[1], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }
    const bool full_tab = a.m <= kTab;
    // table entry of sketch angle k at slot e: window origin, fp64 -> split precision
    auto entry = [&](int k, int e) {
        const double2 cs = a.g.trig[idx[k]];
        // detector position of the tile origin pixel (tr0, tc0), fp64
        const double J0 = a.g.hd + (tc0 - a.g.h) * cs.x + (a.g.h - tr0) * cs.y;
        const double jmin = J0 + fmin(0.0, (kTileW - 1) * cs.x) + fmin(0.0, -(kTileH - 1) * cs.y);
        // (fused rows: an even origin, so the 8-byte bins of a window start 16-byte aligned)
        const double w0 = FUSED ? 2.0 * floor(0.5 * jmin) : floor(jmin);
        s_off[e] = (float)(J0 - w0);
        s_cos[e] = (float)cs.x;
        s_sin[e] = (float)cs.y;
        s_w0[e] = (int)w0;
    };
    // table slot of chunk ch's first angle
    auto tbase = [&](int ch) { return full_tab ? ch * kKC : (ch & 1) * kKC; };
    // per-angle table of chunk ch (threads < kKC; nothing to do for a whole-sketch table)
    auto table = [&](int ch) {
        const int k0 = ch * kKC;
        const int kc = min(kKC, a.m - k0);
        if (!full_tab && threadIdx.x < kc) entry(k0 + threadIdx.x, tbase(ch) + threadIdx.x);
    };
    if (full_tab) {  // the whole table up front: one dependent-load latency per CTA
        for (int k = threadIdx.x; k < a.m; k += kThreads) entry(k, k);
        __syncthreads();
    }
    // bulk path (thread 0): one bulk copy per (angle, job): kW bins x BB images, 16 B per bin,
    // from the interleaved padded sinogram (in bounds for any window origin >= -kAdjPad; the
    // pads supply the zeros outside [0, n_det)); completion on full[bf]
    auto issue_bulk = [&](int ch, int bf) {
        const int k0 = ch * kKC;
        const int kc = min(kKC, a.m - k0);
        constexpr unsigned bytes = kW * BB * sizeof(float);
        fence_proxy_async();  // earlier generic reads of this buffer -> async-proxy writes
        mbar_expect_tx(&full[bf], bytes * kc * NJ);
        const long wp = FUSED ? (long)((a.g.n_det + 2 * kAdjPad + 1) & ~1) : a.g.n_det + 2 * kAdjPad;
        for (int t = 0; t < kc; ++t) {
            const long row = ((long)blockIdx.y * a.m + k0 + t) * wp + kAdjPad + s_w0[tbase(ch) + t];
            SKEI_DCHECK(s_w0[tbase(ch) + t] >= -kAdjPad &&
                            kAdjPad + s_w0[tbase(ch) + t] + kW <= wp,
                        "backprojector window inside the padded row");
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
                bulk_g2s(&win[bf][jj][t * kW * BB], a.job[jj].pi + row * BB, bytes, &full[bf]);
        }
    };
    // plain path (all threads): table, then element-wise cp.async, zero outside [0, n_det)
    auto stage = [&](int ch, int bf) {
        const int k0 = ch * kKC;
        const int kc = min(kKC, a.m - k0);
        table(ch);
        __syncthreads();  // window origins visible
        // element e -> (angle t, bin w, image b), image fastest
        for (int e = threadIdx.x; e < kc * kW * BB; e += kThreads) {
            const int b = e % BB;
            const int w = (e / BB) % kW;
            const int t = e / (BB * kW);
            const int jb = s_w0[tbase(ch) + t] + w;
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                float *dst = &win[bf][jj][e];
                if (jb >= 0 && jb < n_det)
                    cp_async4(dst, a.job[jj].p + ((long)(b0 + b) * a.m + k0 + t) * n_det + jb);
                else
                    *dst = 0.f;
            }
        }
        cp_async_commit();
    };
    // warp 0 prepares chunk ch in buffer bf: its lanes write the table, lane 0 (after the
    // warp barrier) issues the copies; the other warps see the table through the mbarrier
    // (arrive.release by lane 0, try_wait.acquire by the consumers)
    auto produce = [&](int ch, int bf) {
        if (warp == 0) {
            table(ch);
            __syncwarp();
            if (lane == 0) issue_bulk(ch, bf);
        }
    };

    if constexpr (BULK) {
        produce(0, 0);
        if (nchunks > 1) produce(1, 1);
    } else {
        stage(0, 0);
    }
    for (int ch = 0; ch < nchunks; ++ch) {
        const int bf = ch & 1;
        if constexpr (BULK) {
            mbar_wait(&full[bf], (unsigned)((ch >> 1) & 1));
        } else {
            if (ch + 1 < nchunks) stage(ch + 1, bf ^ 1);
            if (ch + 1 < nchunks)
                cp_async_wait<1>();
            else
                cp_async_wait<0>();
            __syncthreads();
        }
        const int kc = min(kKC, a.m - ch * kKC);
        const int tb = tbase(ch);
#pragma unroll 2
        for (int t = 0; t < kc; ++t) {
            const float ct = s_cos[tb + t], st = s_sin[tb + t];
            // position of pixel (ry, 2 pc) relative to the window origin
            const float rowb = fmaf(-(float)ry, st, s_off[tb + t]);
#pragma unroll
            for (int p = 0; p < kPairs; ++p) {
                const int c = 2 * (pc0 + 16 * p);
                const float t1 = fmaf((float)c, ct, rowb);
                const float t2 = t1 + ct;
                const float lo = fmaxf(fminf(t1, t2), 0.f);
                const float jf = floorf(lo);
                const int j = min((int)jf, kW - 3);
                const float u1 = t1 - (float)j, u2 = t2 - (float)j;
                float w10, w11, w12, w20, w21, w22;
                hat3(u1, w10, w11, w12);
                hat3(u2, w20, w21, w22);
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) {
                    const float *wt = &win[bf][jj][(t * kW + j) * BB];
                    float q0[BB], q1[BB], q2[BB];
                    load_bins<BB>(wt, q0);
                    load_bins<BB>(wt + BB, q1);
                    load_bins<BB>(wt + 2 * BB, q2);
                    tap3<BB>(acc[jj][p][0], w10, w11, w12, q0, q1, q2);
                    tap3<BB>(acc[jj][p][1], w20, w21, w22, q0, q1, q2);
                }
            }
        }
        __syncthreads();  // buffer bf (and its table) is free for chunk ch + 2
        if constexpr (BULK) {
            if (ch + 2 < nchunks) produce(ch + 2, bf);
        }
    }

    // ---- epilogue: scale and store; optional fused ei partials (job 0 = FBP)
    const int r = tr0 + ry;
    float eacc[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) eacc[b] = 0.f;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
#pragma unroll
        for (int p = 0; p < kPairs; ++p) {
            const int c = tc0 + 2 * (pc0 + 16 * p);
            if (r >= a.row1) continue;
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                // the output of (job jj, image slot b); fused: job b of image b0
                const AdjJob &jo = a.job[FUSED ? b : jj];
                const int img = FUSED ? b0 : b0 + b;
                const float sc = jo.scale;
                const long o = (long)img * nn + (long)r * n + c;  // in a whole image
                long ox;
                float *const dst = out_at(a, jo.x, FUSED ? b : jj, img, r, c, ox);
                float v0 = sc * acc[jj][p][0][b], v1 = sc * acc[jj][p][1][b];
                if (jo.base) {  // x = base + scale A^T p
                    if (c < n) v0 += __ldg(jo.base + ox);
                    if (c + 1 < n) v1 += __ldg(jo.base + ox + 1);
                }
                if (c + 1 < n && ((ox & 1) == 0)) {
                    *reinterpret_cast<float2 *>(dst + ox) = make_float2(v0, v1);
                } else {
                    if (c < n) dst[ox] = v0;
                    if (c + 1 < n) dst[ox + 1] = v1;
                }
                if (jj == 0 && (!FUSED || b == 0) && a.ei_x2) {
                    if (c < n) {
                        const float d = __ldg(a.ei_x2 + o) - v0;
                        eacc[b] = fmaf(d, d, eacc[b]);
                    }
                    if (c + 1 < n) {
                        const float d = __ldg(a.ei_x2 + o + 1) - v1;
                        eacc[b] = fmaf(d, d, eacc[b]);
                    }
                }
            }
        }
    }
    if (!a.ei_x2) return;
    // deterministic per-tile partial per image, then the last CTA sums the tiles in order
#pragma unroll
    for (int b = 0; b < BB; ++b) {
        float v = eacc[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_red[warp][b] = v;
    }
    __syncthreads();
    const int ntiles = gridDim.x;
    if (threadIdx.x < (FUSED ? 1 : BB)) {
        float v = 0.f;
        for (int w = 0; w < kThreads / 32; ++w) v += s_red[w][threadIdx.x];
        a.ei_part[(long)(b0 + threadIdx.x) * ntiles + tile] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned total = gridDim.x * gridDim.y;
        s_last = atomicAdd(a.ei_ctr, 1u) == total - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // the last CTA: ei[b] = sum over tiles in tile order, fp64, one warp per image
    for (int b = warp; b < a.B; b += kThreads / 32) {
        double s = 0.0;
        for (int i = lane; i < ntiles; i += 32) s += (double)__ldcg(a.ei_part + (long)b * ntiles + i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) a.ei_out[b] = (float)s;
    }
    if (threadIdx.x == 0) *a.ei_ctr = 0u;  // ready for the next launch
}

// ---- quad variant (bulk staging only): each thread owns FOUR horizontally adjacent pixels
// of one row.  Their positions t_k = t_0 + k cos(th) span 3 |cos th| <= 3 bins, so the quad
// reads one 5-bin window per (angle, job) — 5 LDS for 4 pixels instead of 6 for two pairs.
// Pixel i in "canonical" order (i = 0 the pixel with the lowest position: k = i for
// cos >= 0, k = 3 - i for cos < 0) lies at u_i = u + i |cos| from the window origin
// (u in [0, 1)), so its 3 candidate bins start at a per-angle offset o_i with
// o_i in [i |cos| - 1, i |cos|]: o = (0,0,0,0) for |cos| <= 1/3, (0,0,0,1) for <= 1/2,
// (0,0,1,1) for <= 2/3, else (0,0,1,2) — warp-uniform, so each (pattern, sign) is its own
// compiled body (static register indexing).  The lanes of a quarter-warp are 8 consecutive
// rows of one quad column (conflict-free, as the pair kernel).  Tile 32 x 32, 256 threads.
constexpr int kQTileH = 32;  // quad tile height (rows); width kTileW
constexpr int kQW = 48;      // staged bins per angle (>= 31 sqrt 2 + 4)
#ifndef SKEI_ADJQ_KC
#define SKEI_ADJQ_KC 12
#endif
#ifndef SKEI_ADJQ_NB
#define SKEI_ADJQ_NB 2
#endif
constexpr int kQKC = SKEI_ADJQ_KC;  // angles per staged chunk
constexpr int kQNB = SKEI_ADJQ_NB;  // staged chunks in flight (bulk staging)
#ifndef SKEI_ADJQ_MINB
#define SKEI_ADJQ_MINB 3     // CTAs per SM the quad kernel is compiled for
#endif
#ifndef SKEI_ADJQ_MINB_FUSED
#define SKEI_ADJQ_MINB_FUSED 4  // ... for job-fused groups (8 accumulators per thread)
#endif
#ifndef SKEI_ADJQ_FUSED
#define SKEI_ADJQ_FUSED 1    // job-fused groups use the quad kernel (A/B knob)
#endif
#ifndef SKEI_ADJQ_NOBAR
#define SKEI_ADJQ_NOBAR 1    // quad kernel, bulk + full table: last warp refills, no chunk barrier
#endif
#ifndef SKEI_ADJQ_UNROLL
#define SKEI_ADJQ_UNROLL 1   // angles unrolled in the quad kernel's loop
#endif
constexpr int kQUnroll = SKEI_ADJQ_UNROLL;

template <int BB, int NJ, bool BULK, bool FUSED>
__global__ void __launch_bounds__(kThreads, FUSED ? SKEI_ADJQ_MINB_FUSED : SKEI_ADJQ_MINB)
    k_radon_adj_quad(AdjArgs a) {
    // window buffers: kQNB with bulk staging (refilled by the last warp out), 2 otherwise
    constexpr int NB = BULK ? kQNB : 2;
    __shared__ __align__(128) float win[NB][NJ][kQKC * kQW * BB];
    __shared__ float s_off[kTab], s_cos[kTab], s_sin[kTab];
    __shared__ int s_w0[kTab], s_pat[kTab];
    __shared__ float s_red[kThreads / 32][BB];
    __shared__ bool s_last;
    __shared__ __align__(8) uint64_t full[NB];
    __shared__ unsigned s_done[NB];  // warps finished with each buffer (monotonic; SKEI_ADJQ_NOBAR)

    const int n = a.g.n, n_det = a.g.n_det;
    const int tile = blockIdx.x;
    const int tr0 = a.row0 + (tile / a.tiles_x) * kQTileH, tc0 = (tile % a.tiles_x) * kTileW;
    const int b0 = FUSED ? blockIdx.y : blockIdx.y * BB;
    const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp w: rows 8 (w & 3) .. +7, quad columns 4 (w >> 2) .. +3; a quarter-warp = 8 rows
    const int ry = 8 * (warp & 3) + (lane & 7);
    const int qc = 4 * (warp >> 2) + (lane >> 3);  // quad index 0..7
    const long nn = (long)n * n;

    float acc[NJ][4][BB];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int b = 0; b < BB; ++b) acc[j][q][b] = 0.f;

    const int nchunks = (a.m + kQKC - 1) / kQKC;
    if (BULK && threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(&full[i], 1);
            s_done[i] = 0u;
        }
        fence_mbar_init();
    }
    const bool full_tab = a.m <= kTab;
    auto entry = [&](int k, int e) {
        const double2 cs = a.g.trig[idx[k]];
        const double J0 = a.g.hd + (tc0 - a.g.h) * cs.x + (a.g.h - tr0) * cs.y;
        const double jmin = J0 + fmin(0.0, (kTileW - 1) * cs.x) + fmin(0.0, -(kQTileH - 1) * cs.y);
        const double w0 = FUSED ? 2.0 * floor(0.5 * jmin) : floor(jmin);
        s_off[e] = (float)(J0 - w0);
        const float cf = (float)cs.x, ac = fabsf(cf);
        s_cos[e] = cf;
        s_sin[e] = (float)cs.y;
        s_w0[e] = (int)w0;
        const int pat = ac <= (1.f / 3.f) ? 0 : ac <= 0.5f ? 1 : ac <= (2.f / 3.f) ? 2 : 3;
        s_pat[e] = pat | (cf < 0.f ? 4 : 0);
    };
    auto tbase = [&](int ch) { return full_tab ? ch * kQKC : (ch % NB) * kQKC; };
    auto table = [&](int ch) {
        const int k0 = ch * kQKC;
        const int kc = min(kQKC, a.m - k0);
        if (!full_tab && threadIdx.x < kc) entry(k0 + threadIdx.x, tbase(ch) + threadIdx.x);
    };
    if (full_tab)
        for (int k = threadIdx.x; k < a.m; k += kThreads) entry(k, k);
    __syncthreads();
    auto issue_bulk = [&](int ch, int bf) {
        const int k0 = ch * kQKC;
        const int kc = min(kQKC, a.m - k0);
        constexpr unsigned bytes = kQW * BB * sizeof(float);
        fence_proxy_async();
        mbar_expect_tx(&full[bf], bytes * kc * NJ);
        const long wp = FUSED ? (long)((a.g.n_det + 2 * kAdjPad + 1) & ~1) : a.g.n_det + 2 * kAdjPad;
        for (int t = 0; t < kc; ++t) {
            const long row = ((long)blockIdx.y * a.m + k0 + t) * wp + kAdjPad + s_w0[tbase(ch) + t];
            SKEI_DCHECK(s_w0[tbase(ch) + t] >= -kAdjPad && kAdjPad + s_w0[tbase(ch) + t] + kQW <= wp,
                        "quad backprojector window inside the padded row");
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
                bulk_g2s(&win[bf][jj][t * kQW * BB], a.job[jj].pi + row * BB, bytes, &full[bf]);
        }
    };
    auto produce = [&](int ch, int bf) {
        if (warp == 0) {
            table(ch);
            __syncwarp();
            if (lane == 0) issue_bulk(ch, bf);
        }
    };
    // plain path (standalone calls: all threads): table, then element-wise cp.async from the
    // plain sinograms, zero outside [0, n_det) — the same window contents as the bulk copies
    auto stage = [&](int ch, int bf) {
        const int k0 = ch * kQKC;
        const int kc = min(kQKC, a.m - k0);
        table(ch);
        __syncthreads();  // window origins visible
        for (int e = threadIdx.x; e < kc * kQW * BB; e += kThreads) {
            const int b = e % BB;
            const int w = (e / BB) % kQW;
            const int t = e / (BB * kQW);
            const int jb = s_w0[tbase(ch) + t] + w;
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                float *dst = &win[bf][jj][e];
                if (jb >= 0 && jb < n_det)
                    cp_async4(dst, a.job[jj].p + ((long)(b0 + b) * a.m + k0 + t) * n_det + jb);
                else
                    *dst = 0.f;
            }
        }
        cp_async_commit();
    };
    if constexpr (BULK) {
        for (int c = 0; c < NB && c < nchunks; ++c) produce(c, c);
    } else {
        stage(0, 0);
    }

    // one angle: the quad's 5-bin window per job, canonical pixel i -> pixel k
    auto angle = [&](auto pat_tag, auto neg_tag, const float *w_base, float u, float ac) {
        constexpr int P = decltype(pat_tag)::value;
        constexpr bool NEG = decltype(neg_tag)::value;
        constexpr int o1 = 0, o2 = P >= 2 ? 1 : 0, o3 = P == 0 ? 0 : P == 3 ? 2 : 1;
        constexpr int oo[4] = {0, o1, o2, o3};
        float w[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) hat3(fmaf((float)i, ac, u) - (float)oo[i], w[i][0], w[i][1], w[i][2]);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const float *wt = w_base + jj * (kQKC * kQW * BB);
            float q[5][BB];
#pragma unroll
            for (int e = 0; e < 5; ++e) load_bins<BB>(wt + e * BB, q[e]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = NEG ? 3 - i : i;
                tap3<BB>(acc[jj][k], w[i][0], w[i][1], w[i][2], q[oo[i]], q[oo[i] + 1], q[oo[i] + 2]);
            }
        }
    };
    for (int ch = 0; ch < nchunks; ++ch) {
        const int bf = ch % NB;
        if constexpr (BULK) {
            mbar_wait(&full[bf], (unsigned)((ch / NB) & 1));
        } else {
            if (ch + 1 < nchunks) stage(ch + 1, bf ^ 1);
            if (ch + 1 < nchunks)
                cp_async_wait<1>();
            else
                cp_async_wait<0>();
            __syncthreads();
        }
        const int kc = min(kQKC, a.m - ch * kQKC);
        const int tb = tbase(ch);
#pragma unroll kQUnroll
        for (int t = 0; t < kc; ++t) {
            const float ct = s_cos[tb + t], st = s_sin[tb + t];
            const int pt = s_pat[tb + t];
            const float rowb = fmaf(-(float)ry, st, s_off[tb + t]);
            const float t0 = fmaf((float)(4 * qc), ct, rowb);
            const float tlow = (pt & 4) ? fmaf(3.f, ct, t0) : t0;  // the lowest of the 4
            const float jf = floorf(fmaxf(tlow, 0.f));
            const int j = min((int)jf, kQW - 5);
            const float u = tlow - (float)j;
            const float ac = fabsf(ct);
            const float *wb = &win[bf][0][(t * kQW + j) * BB];
            using I0 = std::integral_constant<int, 0>;
            using I1 = std::integral_constant<int, 1>;
            using I2 = std::integral_constant<int, 2>;
            using I3 = std::integral_constant<int, 3>;
            switch (pt) {
                case 0: angle(I0{}, std::false_type{}, wb, u, ac); break;
                case 1: angle(I1{}, std::false_type{}, wb, u, ac); break;
                case 2: angle(I2{}, std::false_type{}, wb, u, ac); break;
                case 3: angle(I3{}, std::false_type{}, wb, u, ac); break;
                case 4: angle(I0{}, std::true_type{}, wb, u, ac); break;
                case 5: angle(I1{}, std::true_type{}, wb, u, ac); break;
                case 6: angle(I2{}, std::true_type{}, wb, u, ac); break;
                default: angle(I3{}, std::true_type{}, wb, u, ac); break;
            }
        }
        if (BULK && SKEI_ADJQ_NOBAR && full_tab) {
            // no block-wide barrier per chunk: the last warp out of buffer bf refills it with
            // chunk ch + 2 (the angle table is complete up front, so a refill is only the bulk
            // copies), so warps drift up to a chunk apart instead of meeting every 12 angles
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();  // this warp's reads of the buffer are complete
                const unsigned old = atomicAdd(&s_done[bf], 1u);
                if (old == (unsigned)(kThreads / 32) * (unsigned)(ch / NB + 1) - 1u && ch + NB < nchunks) {
                    if constexpr (BULK) issue_bulk(ch + NB, bf);
                }
            }
        } else {
            __syncthreads();  // buffer bf (and its table) is free for chunk ch + NB
            if constexpr (BULK) {
                if (ch + NB < nchunks) produce(ch + NB, bf);
            }
        }
    }

    // ---- epilogue: scale and store; optional fused ei partials (job 0 = FBP)
    const int r = tr0 + ry;
    float eacc[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) eacc[b] = 0.f;
    const int c = tc0 + 4 * qc;
    if (r < a.row1) {
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                const AdjJob &jo = a.job[FUSED ? b : jj];
                const int img = FUSED ? b0 : b0 + b;
                const float sc = jo.scale;
                const long o = (long)img * nn + (long)r * n + c;
                long ox;
                float *const dst = out_at(a, jo.x, FUSED ? b : jj, img, r, c, ox);
                float v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = sc * acc[jj][k][b];
                if (jo.base) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (c + k < n) v[k] += __ldg(jo.base + ox + k);
                }
                if (c + 3 < n && ((ox & 3) == 0)) {
                    *reinterpret_cast<float4 *>(dst + ox) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (c + k < n) dst[ox + k] = v[k];
                }
                if (jj == 0 && (!FUSED || b == 0) && a.ei_x2) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (c + k < n) {
                            const float d = __ldg(a.ei_x2 + o + k) - v[k];
                            eacc[b] = fmaf(d, d, eacc[b]);
                        }
                }
            }
        }
    }
    if (!a.ei_x2) return;
#pragma unroll
    for (int b = 0; b < BB; ++b) {
        float v = eacc[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_red[warp][b] = v;
    }
    __syncthreads();
    const int ntiles = gridDim.x;
    if (threadIdx.x < (FUSED ? 1 : BB)) {
        float v = 0.f;
        for (int w = 0; w < kThreads / 32; ++w) v += s_red[w][threadIdx.x];
        a.ei_part[(long)(b0 + threadIdx.x) * ntiles + tile] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned total = gridDim.x * gridDim.y;
        s_last = atomicAdd(a.ei_ctr, 1u) == total - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int b = warp; b < a.B; b += kThreads / 32) {
        double sd = 0.0;
        for (int i = lane; i < ntiles; i += 32) sd += (double)__ldcg(a.ei_part + (long)b * ntiles + i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
        if (lane == 0) a.ei_out[b] = (float)sd;
    }
    if (threadIdx.x == 0) *a.ei_ctr = 0u;
}

#ifndef SKEI_ADJ_QUAD
#define SKEI_ADJ_QUAD 1  // bulk-staged backprojections use the quad kernel (A/B knob)
#endif

// the quad kernel's grid: 32 x 32 tiles (a.tiles_y is recomputed for its tile height)
template <int BB, int NJ, bool BULK, bool FUSED>
cudaError_t launch_quad(AdjArgs a, int ngroups, cudaStream_t s) {
    a.tiles_y = (a.row1 - a.row0 + kQTileH - 1) / kQTileH;
    dim3 grid((unsigned)(a.tiles_x * a.tiles_y), (unsigned)ngroups, 1);
    k_radon_adj_quad<BB, NJ, BULK, FUSED><<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fused(const AdjArgs &a, int B, cudaStream_t s) {
    if (SKEI_ADJQ_FUSED) return launch_quad<2, 1, true, true>(a, B, s);
    // job-fused groups: the quad kernel compiled for 4 CTAs per SM (64 registers; 8
    // accumulators per thread): cfg4 2618 -> 2369 us, cfg5 250 -> 236 us against the pair
    // kernel (at 3 CTAs per SM it was slower: 2644 / 268 us)
    dim3 grid((unsigned)(a.tiles_x * a.tiles_y), (unsigned)B, 1);
    k_radon_adj<2, 1, true, true><<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int BB>
cudaError_t launch_bb(const AdjArgs &a, int njobs, int B, cudaStream_t s, bool quad) {
    dim3 grid((unsigned)(a.tiles_x * a.tiles_y), (unsigned)(B / BB), 1);
    // bulk-copy staging needs 16-byte bins (BB = 4) and interleaved sources for every job
    constexpr bool kB4 = BB == 4;  // (the bulk variants are only instantiated for BB = 4)
    const bool bulk = kB4 && a.job[0].pi && (njobs == 1 || a.job[1].pi);
    if (quad) {
        if (bulk) {
            if constexpr (kB4)
                return njobs == 2 ? launch_quad<4, 2, true, false>(a, B / BB, s)
                                  : launch_quad<4, 1, true, false>(a, B / BB, s);
        }
        return njobs == 2 ? launch_quad<BB, 2, false, false>(a, B / BB, s)
                          : launch_quad<BB, 1, false, false>(a, B / BB, s);
    }
    if (njobs == 2) {
        if (bulk)
            k_radon_adj<BB, 2, kB4><<<grid, kThreads, 0, s>>>(a);
        else
            k_radon_adj<BB, 2, false><<<grid, kThreads, 0, s>>>(a);
    } else {
        if (bulk)
            k_radon_adj<BB, 1, kB4><<<grid, kThreads, 0, s>>>(a);
        else
            k_radon_adj<BB, 1, false><<<grid, kThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace

size_t adj_ei_part_floats(const skei_plan *plan, int B) {
    const int tx = (plan->n + kTileW - 1) / kTileW, ty = (plan->n + kTileH - 1) / kTileH;
    return (size_t)B * tx * ty;
}

cudaError_t launch_radon_adj(const skei_plan *plan, const AdjJob *jobs, int njobs, int B,
                             const int32_t *idx, int m, int idx_stride, cudaStream_t s,
                             const AdjEi *ei, int row0, int rows, bool fused,
                             const AdjRs *rs) {
    if (fused && (njobs != 2 || !jobs[0].pi)) return cudaErrorInvalidValue;
    // the reduce-scatter epilogue: whole images, no base addend, no fused ei
    if (rs && (rs->world < 1 || rs->world > kMaxRsPeers || row0 > 0 || rows >= 0 || ei ||
               jobs[0].base || (njobs > 1 && jobs[1].base)))
        return cudaErrorInvalidValue;
    AdjArgs a;
    if (rs) a.rs = *rs;
    a.job[0] = jobs[0];
    a.job[1] = njobs > 1 ? jobs[1] : jobs[0];
    a.idx = idx;
    a.m = m;
    a.idx_stride = idx_stride;
    a.B = B;
    a.g = geom_of(plan);
    a.row0 = row0 < 0 ? 0 : row0;
    a.row1 = rows < 0 ? plan->n : a.row0 + rows;
    a.tiles_x = (plan->n + kTileW - 1) / kTileW;
    a.tiles_y = (a.row1 - a.row0 + kTileH - 1) / kTileH;
    a.ei_x2 = ei ? ei->x2 : nullptr;
    a.ei_part = ei ? ei->part : nullptr;
    a.ei_ctr = ei ? ei->ctr : nullptr;
    a.ei_out = ei ? ei->out : nullptr;
    if (fused) return launch_fused(a, B, s);
    const int bb = pick_bb(B, idx_stride);
    // the quad kernel (32 x 32 tiles, 3 CTAs per SM) when its grid fills at least one wave;
    // smaller problems (cfg2: 128 quad CTAs) keep the pair kernel's 2x finer grid
    const long quad_ctas = (long)a.tiles_x * ((a.row1 - a.row0 + kQTileH - 1) / kQTileH) * (B / bb);
    const bool quad = SKEI_ADJ_QUAD && quad_ctas >= 3L * plan->num_sms;
    switch (bb) {
        case 4: return launch_bb<4>(a, njobs, B, s, quad);
        case 2: return launch_bb<2>(a, njobs, B, s, quad);
        default: return launch_bb<1>(a, njobs, B, s, quad);
    }
}

}  // namespace skei
