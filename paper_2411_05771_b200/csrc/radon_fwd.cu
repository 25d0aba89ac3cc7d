// radon_fwd.cu — a3: p = A_S x, the pixel-driven projector with linear detector
// interpolation, A[th, s] = sum_p x_p max(0, 1 - |x_p cos th + y_p sin th - s|/ds)
// (BASELINE.json north_star), "organised as a per-(angle, detector-strip) gather so no
// global atomics are needed".
//
// Design (DESIGN.md §5 "radon_fwd"):
//   * Angles split into two classes by an exact integer test on the angle index:
//     row class (|cos| >= |sin|: 4i <= n_full or 4i >= 3 n_full) marches over image rows,
//     column class marches over image columns.  Along a line the pixel positions map to
//     the detector with slope beta (|beta| >= 1/sqrt 2), so every (bin, line) pair has at
//     most 3 candidate pixels: the first integer above a* - 1/|beta| and the next two,
//     where a* is the line position that projects exactly onto the bin centre.
//   * One CTA = (class, group of K angles of that class, batch group of BB images that
//     share the angle list, quarter of the lines).  The four line-quarters of a work
//     unit form a thread-block cluster: each CTA streams its quarter of the image through
//     shared memory in blocks of R lines (cp.async), interleaved [line][pixel][image] so
//     one LDS.128 fetches a candidate pixel of 4 images, and accumulates its partial
//     projection in registers; at the end the partials are summed across the cluster
//     through distributed shared memory in fixed rank order (deterministic, no atomics).
//   * Work items: warp task = (angle, 32 consecutive bins); a warp owns up to 6 tasks,
//     lane = bin.  Per (task, line): a* from an fp64 per-block base plus an fp32 local
//     offset (split precision), 3 hat weights, 3 LDS.BB, 3*BB FFMA.
//   * A task skips a line block when none of its 32 bins sees the block (warp vote).
#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace skei {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxT = 6;     // tasks per warp
constexpr int kS = 4;        // line split = cluster size
constexpr int kKMax = 16;    // angles per CTA
constexpr int kPadL = 4;     // zero pixels left of each staged line (right pad >= 5)

struct FwdArgs {
    FwdJob job[2];
    const int32_t *idx;
    int m, idx_stride, B;
    int K;       // angles per CTA
    int chunks;  // ceil(n_det / 32)
    int pitch;   // staged pixels per line (>= n + 9, = 1 mod 8 for conflict-free staging)
    Geom g;
};

__device__ inline void cp_async4(float *smem, const float *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ inline void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int BB>
struct Px;
template <> struct Px<1> { using T = float; };
template <> struct Px<2> { using T = float2; };
template <> struct Px<4> { using T = float4; };

template <int BB>
__device__ inline void ld_px(const float *p, float (&v)[BB]) {
    const typename Px<BB>::T t = *reinterpret_cast<const typename Px<BB>::T *>(p);
    const float *pt = reinterpret_cast<const float *>(&t);
#pragma unroll
    for (int b = 0; b < BB; ++b) v[b] = pt[b];
}

template <int BB>
__global__ void __cluster_dims__(kS, 1, 1) __launch_bounds__(kThreads, 3)
    k_radon_fwd(FwdArgs a) {
    constexpr int R = 32 / BB;  // lines per staged block (R * BB = 32 floats per pixel column)
    extern __shared__ __align__(16) float stage[];  // [R][pitch][BB]; partials at the end
    __shared__ double sP0[kKMax], sPj[kKMax], sPl[kKMax];
    __shared__ float sAbsB[kKMax], sSec[kKMax], sPlf[kKMax];
    __shared__ int sSlot[kKMax];
    __shared__ int sCount;

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int unit = blockIdx.x / kS;
    const int cls = unit & 1, grp = unit >> 1;
    const FwdJob job = blockIdx.z ? a.job[1] : a.job[0];
    const int b0 = blockIdx.y * BB;
    const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);
    const int n = a.g.n, n_det = a.g.n_det, n_full = a.g.n_full;
    const int pitch = a.pitch;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int K = a.K;

    // ---- 1. the grp-th group of K angles of class cls, in sketch-slot order
    if (threadIdx.x < 32) {
        int seen = 0;
        for (int base = 0; base < a.m; base += 32) {
            const int k = base + lane;
            bool in = false;
            if (k < a.m) {
                const int i = idx[k];
                const bool row_class = (4 * i <= n_full) || (4 * i >= 3 * n_full);
                in = (cls == 0) ? row_class : !row_class;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            const int pre = seen + __popc(bal & ((1u << lane) - 1u));
            if (in && pre >= grp * K && pre < grp * K + K) sSlot[pre - grp * K] = k;
            seen += __popc(bal);
        }
        if (lane == 0) sCount = max(0, min(K, seen - grp * K));
    }
    __syncthreads();
    const int kcnt = sCount;
    if (kcnt == 0) return;  // same decision in every CTA of the cluster (depends on unit only)

    // ---- 2. per-angle line geometry in fp64: a*(j, l) = P0 + j Pj + l Pl
    if (threadIdx.x < kcnt) {
        const double2 cs = a.g.trig[idx[sSlot[threadIdx.x]]];
        const double c = cs.x, s = cs.y, h = a.g.h, hd = a.g.hd;
        double P0, Pj, Pl, ab;
        if (cls == 0) {  // lines = rows r, along = columns: c* = h + (j - hd - (h - r) s)/c
            P0 = h - (hd + h * s) / c;
            Pj = 1.0 / c;
            Pl = s / c;
            ab = fabs(c);
        } else {  // lines = columns c, along = rows: r* = h + (hd - j + (c - h) cos)/sin
            P0 = h + (hd - h * c) / s;
            Pj = -1.0 / s;
            Pl = c / s;
            ab = fabs(s);
        }
        sP0[threadIdx.x] = P0;
        sPj[threadIdx.x] = Pj;
        sPl[threadIdx.x] = Pl;
        sAbsB[threadIdx.x] = (float)ab;
        sSec[threadIdx.x] = (float)(1.0 / ab);
        sPlf[threadIdx.x] = (float)Pl;
    }
    // zero pads: positions [0, kPadL) and [kPadL + n, pitch) of every staged line
    for (int e = threadIdx.x; e < R * (pitch - n) * BB; e += kThreads) {
        const int b = e % BB;
        const int q = (e / BB) % (pitch - n);
        const int l = e / (BB * (pitch - n));
        const int pos = q < kPadL ? q : n + q;
        stage[(l * pitch + pos) * BB + b] = 0.f;
    }
    __syncthreads();

    // ---- 3. tasks of this thread
    int tk[kMaxT], tj[kMaxT];
    bool tvalid[kMaxT];
    float tab[kMaxT], tsec[kMaxT], tplf[kMaxT];
    float acc[kMaxT][BB];
#pragma unroll
    for (int t = 0; t < kMaxT; ++t) {
        const int task = warp + kWarps * t;
        tk[t] = task / a.chunks;
        tj[t] = (task % a.chunks) * 32 + lane;
        tvalid[t] = tk[t] < kcnt;
        const int kk = tvalid[t] ? tk[t] : 0;
        tab[t] = sAbsB[kk];
        tsec[t] = sSec[kk];
        tplf[t] = sPlf[kk];
#pragma unroll
        for (int b = 0; b < BB; ++b) acc[t][b] = 0.f;
    }

    const int lines_per = (n + kS - 1) / kS;
    const int L0 = rank * lines_per, L1 = min(n, L0 + lines_per);
    const long nn = (long)n * n;
    const float *xb = job.x + (long)b0 * nn;

    for (int lb = L0; lb < L1; lb += R) {
        const int nl = min(R, L1 - lb);
        // ---- stage R lines (source lines clamped into the image; extra lines unused)
        if (cls == 0) {
#pragma unroll 1
            for (int l = 0; l < R; ++l) {
                const int row = min(lb + l, n - 1);
                for (int e = threadIdx.x; e < n * BB; e += kThreads) {
                    const int b = e % BB, c = e / BB;
                    cp_async4(stage + (l * pitch + kPadL + c) * BB + b,
                              xb + (long)b * nn + (long)row * n + c);
                }
            }
        } else {
            for (int e = threadIdx.x; e < n * R * BB; e += kThreads) {
                const int b = e % BB, l = (e / BB) % R, r = e / (BB * R);
                const int col = min(lb + l, n - 1);
                cp_async4(stage + (l * pitch + kPadL + r) * BB + b,
                          xb + (long)b * nn + (long)r * n + col);
            }
        }
        cp_async_wait_all();
        __syncthreads();

        // ---- per-task base of this block (fp64) and warp-level activity
        int tbase[kMaxT];
        float tfrac[kMaxT];
        bool tact[kMaxT];
#pragma unroll
        for (int t = 0; t < kMaxT; ++t) {
            tbase[t] = 0;
            tfrac[t] = 0.f;
            tact[t] = false;
            if (tvalid[t]) {  // warp-uniform
                const int k = tk[t];
                const double ad = sP0[k] + (double)tj[t] * sPj[k] + (double)lb * sPl[k];
                const double fl = floor(ad);
                tbase[t] = (int)fl;
                tfrac[t] = (float)(ad - fl);
                const double ae = ad + (double)(nl - 1) * sPl[k];
                const double lo = fmin(ad, ae), hi = fmax(ad, ae);
                const bool act = tj[t] < n_det && hi + tsec[t] > 0.0 && lo - tsec[t] < n - 1.0;
                tact[t] = __any_sync(0xffffffffu, act);
            }
        }
        // Two-level accumulation: the R lines of this block are summed into blk, which is
        // then added to the running total (keeps fp32 rounding at ~1e-7 of the total).
#pragma unroll
        for (int t = 0; t < kMaxT; ++t) {
            if (!tact[t]) continue;
            float blk[BB];
#pragma unroll
            for (int b = 0; b < BB; ++b) blk[b] = 0.f;
#pragma unroll 2
            for (int l = 0; l < nl; ++l) {
                const float *srow = stage + (l * pitch + kPadL) * BB;
                const float lf = (float)l;
                {
                    const float apos = fmaf(lf, tplf[t], tfrac[t]);
                    const float cf = floorf(apos - tsec[t]) + 1.f;
                    int ci = tbase[t] + (int)cf;
                    ci = min(max(ci, -3), n);
                    const float d0 = (cf - apos) * tab[t];
                    const float d1 = d0 + tab[t], d2 = d1 + tab[t];
                    const float w0 = fmaxf(0.f, 1.f - fabsf(d0));
                    const float w1 = fmaxf(0.f, 1.f - fabsf(d1));
                    const float w2 = fmaxf(0.f, 1.f - fabsf(d2));
                    const float *px = srow + ci * BB;
                    float v0[BB], v1[BB], v2[BB];
                    ld_px<BB>(px, v0);
                    ld_px<BB>(px + BB, v1);
                    ld_px<BB>(px + 2 * BB, v2);
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        blk[b] = fmaf(w2, v2[b], fmaf(w1, v1[b], fmaf(w0, v0[b], blk[b])));
                }
            }
#pragma unroll
            for (int b = 0; b < BB; ++b) acc[t][b] += blk[b];
        }
        __syncthreads();
    }

    // ---- 4. partials -> shared memory, then fixed-order sum across the cluster (DSMEM)
    float *part = stage;  // [kcnt][n_det][BB]
#pragma unroll
    for (int t = 0; t < kMaxT; ++t) {
        if (tvalid[t] && tj[t] < n_det) {
#pragma unroll
            for (int b = 0; b < BB; ++b) part[((long)tk[t] * n_det + tj[t]) * BB + b] = acc[t][b];
        }
    }
    cluster.sync();
    const int T = kcnt * n_det * BB;
    const int per = (T + kS - 1) / kS;
    const int o0 = rank * per, o1 = min(T, o0 + per);
    const float *rp[kS];
#pragma unroll
    for (int q = 0; q < kS; ++q) rp[q] = cluster.map_shared_rank(part, q);
    const long img_stride = (long)a.m * n_det;
    for (int o = o0 + threadIdx.x; o < o1; o += kThreads) {
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < kS; ++q) s += rp[q][o];
        const int b = o % BB;
        const int kj = o / BB;
        const int k = kj / n_det, j = kj - k * n_det;
        job.p[(long)(b0 + b) * img_stride + (long)sSlot[k] * n_det + j] = s;
    }
    cluster.sync();
}

template <int BB>
cudaError_t launch_bb(const FwdArgs &a, int njobs, cudaStream_t s) {
    constexpr int R = 32 / BB;
    const size_t stage_f = (size_t)R * a.pitch * BB;
    const size_t part_f = (size_t)a.K * a.g.n_det * BB;
    const size_t smem = sizeof(float) * (stage_f > part_f ? stage_f : part_f);
    cudaError_t e = cudaFuncSetAttribute(k_radon_fwd<BB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ngroups = (a.m + a.K - 1) / a.K;  // per class, worst case
    dim3 grid((unsigned)(kS * 2 * ngroups), (unsigned)(a.B / BB), (unsigned)njobs);
    k_radon_fwd<BB><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_radon_fwd(const skei_plan *plan, const FwdJob *jobs, int njobs, int B,
                             const int32_t *idx, int m, int idx_stride, cudaStream_t s) {
    FwdArgs a;
    a.job[0] = jobs[0];
    a.job[1] = njobs > 1 ? jobs[1] : jobs[0];
    a.idx = idx;
    a.m = m;
    a.idx_stride = idx_stride;
    a.B = B;
    a.g = geom_of(plan);
    a.chunks = (plan->n_det + 31) / 32;
    a.K = (kWarps * kMaxT) / a.chunks;
    if (a.K < 1) return cudaErrorInvalidValue;  // n_det > 48*32 bins not supported
    if (a.K > kKMax) a.K = kKMax;
    int pitch = plan->n + 9;
    while (pitch % 8 != 1) ++pitch;
    a.pitch = pitch;
    const int bb = pick_bb(B, idx_stride);
    switch (bb) {
        case 4: return launch_bb<4>(a, njobs, s);
        case 2: return launch_bb<2>(a, njobs, s);
        default: return launch_bb<1>(a, njobs, s);
    }
}

}  // namespace skei
