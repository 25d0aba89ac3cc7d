// radon_fwd.cu — a3: p = A_S x, the pixel-driven projector with linear detector
// interpolation, A[th, s] = sum_p x_p max(0, 1 - |x_p cos th + y_p sin th - s|/ds)
// (BASELINE.json north_star; R1-R4 in DESIGN.md), "organised as a per-(angle,
// detector-strip) gather so no global atomics are needed".
//
// Design (DESIGN.md §7 "k_radon_fwd"):
//   * Angles are split by an exact integer test on the angle index into the row class
//     (|cos| >= |sin|: 4i <= n_full or 4i >= 3 n_full; lines = image rows) and the column
//     class (lines = image columns).  Along a line the pixel index maps to the detector
//     with slope beta (|beta| >= 1/sqrt 2), so each (bin, line) pair has at most 3 candidate
//     pixels: the first integer above a* - 1/|beta| and the next two, where a* is the line
//     position that projects exactly onto the bin centre.
//   * Input is the packed copy written by k_rotate_pack (rotate.cu): per image group and
//     class, blocks of R = 32/BB lines stored [pixel][line][image] — 128 contiguous bytes
//     per pixel — so a whole block is ONE TMA bulk copy (cp.async.bulk + mbarrier,
//     double-buffered, issued by one thread: no staging instructions, no registers) and one
//     LDS.BB fetches a candidate pixel of BB images.
//   * Work unit = (job, group of BB images sharing the sketch, class, group of K angles);
//     the S CTAs of a thread-block cluster (S chosen at launch to fill the waves) split the
//     unit's lines.  Staged pixels are reused by all K angles of the unit.
//   * Bank-conflict-free gathers: lane L processes the lines of a block in the skewed
//     order l = (L + s) mod R.  The lanes of one shared-memory phase (8 lanes for LDS.128,
//     16 for LDS.64, 32 for LDS.32) then read R distinct line slots, i.e. distinct banks,
//     whatever pixel each lane's bin needs (a lane-per-bin layout gives 2-way conflicts at
//     every angle with |beta| < 1 because 8 bins span more than 8 pixels).
//   * 1024 threads (64 registers each), one CTA per SM.  Task = (angle, 32 consecutive
//     bins), lane = bin; the K x chunks tasks are dealt round-robin to the 32 warps (each
//     warp gets a mix of angles, whose footprints differ); a thread owns up to kMaxT tasks
//     and keeps BB accumulators per task in registers: K = 32 kMaxT / chunks angles.
//   * Decoupled pipeline: no per-block barrier.  The last warp to finish a staged block
//     (shared-memory counter) refills its buffer with the block nbuf ahead, so warps drift
//     up to nbuf - 1 blocks apart and per-block load imbalance averages out.
//   * Per (bin, line): a* from an fp64 per-block base plus an fp32 offset < R (split
//     precision), 3 hat weights, 3 LDS.BB (the third skipped when its weight
//     is 0), 3*BB FFMA.  The R lines of a block are summed into a partial before it is
//     added to the running total (two-level summation).  A chunk skips a block none of its
//     32 bins sees.
//   * End: per-CTA partial projections -> shared memory -> fixed-rank-order sum across the
//     cluster through distributed shared memory (deterministic, no atomics) -> p.
#include <cooperative_groups.h>

#include "internal.h"

namespace skei {
namespace {

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxT = 6;    // 32-bin chunks per thread (registers left for load pipelining)
constexpr int kKMax = 32;   // angles per CTA
constexpr int kPadL = 4;    // zero pixel columns left of the line data
constexpr int kPadR = 4;    // ... and right of it (candidates reach n + 2)
constexpr int kColF = 32;   // floats per staged pixel column (R * BB)

struct FwdArgs {
    FwdJob job[2];
    const int32_t *idx;
    int m, idx_stride, B;
    int K;       // angles per CTA: K * chunks <= kWarps * kMaxT tasks
    int chunks;  // ceil(n_det / 32)
    int nblk;    // packed blocks per image group (ceil(n / R))
    int nbuf;    // staging buffers (2 = double-buffered)
    Geom g;
};

// ---- TMA bulk copy + mbarrier (sm_90+ async proxy), inline PTX
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    // try_wait with a suspend-time hint: a waiting warp sleeps in hardware until the phase
    // completes (or the hint expires) instead of spinning on issue slots other warps need
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// One packed block (n pixel columns of 128 B) -> the interior of a staging buffer.
__device__ __forceinline__ void issue_block(float *buf, const float *src, int n, uint64_t *bar) {
    const unsigned bytes = (unsigned)n * 128u;
    mbar_expect_tx(bar, bytes);
    constexpr unsigned kPiece = 32768u;
    for (unsigned off = 0; off < bytes; off += kPiece) {
        const unsigned len = bytes - off < kPiece ? bytes - off : kPiece;
        bulk_g2s(reinterpret_cast<char *>(buf) + off, reinterpret_cast<const char *>(src) + off, len, bar);
    }
}

template <int BB>
struct Px;
template <> struct Px<1> { using T = float; };
template <> struct Px<2> { using T = float2; };
template <> struct Px<4> { using T = float4; };

template <int BB>
__device__ __forceinline__ void ld_px(const float *p, float (&v)[BB]) {
    const typename Px<BB>::T t = *reinterpret_cast<const typename Px<BB>::T *>(p);
    const float *pt = reinterpret_cast<const float *>(&t);
#pragma unroll
    for (int b = 0; b < BB; ++b) v[b] = pt[b];
}

template <int BB>
__global__ void __launch_bounds__(kThreads, 1) k_radon_fwd(FwdArgs a) {
    constexpr int R = kColF / BB;
    extern __shared__ __align__(128) float smem[];  // nbuf x [n + pads][R][BB]; partials at end
    __shared__ __align__(8) uint64_t full[3];
    __shared__ int done[3];  // warps that finished each buffer (monotonic)
    __shared__ double sP0[kKMax], sPj[kKMax], sPl[kKMax];
    __shared__ float sAbsB[kKMax], sSec[kKMax], sPlf[kKMax];
    __shared__ int sSlot[kKMax];
    __shared__ int sCount;

    cg::cluster_group cluster = cg::this_cluster();
    const int S = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int unit = blockIdx.x / S;
    const int cls = unit & 1, grp = unit >> 1;
    const FwdJob job = blockIdx.z ? a.job[1] : a.job[0];
    const int b0 = blockIdx.y * BB;
    const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);
    const int n = a.g.n, n_det = a.g.n_det, n_full = a.g.n_full;
    const int K = a.K;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

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
    // zero pad columns of every buffer (never written by the bulk copies)
    const int stage_f = (n + kPadL + kPadR) * kColF;
    for (int e = threadIdx.x; e < a.nbuf * (kPadL + kPadR) * kColF; e += kThreads) {
        const int bi = e / ((kPadL + kPadR) * kColF);
        const int e2 = e - bi * (kPadL + kPadR) * kColF;
        const int q = e2 / kColF, w = e2 - q * kColF;
        const int col = q < kPadL ? q : kPadL + n + (q - kPadL);
        smem[bi * stage_f + col * kColF + w] = 0.f;
    }
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&full[2], 1);
        done[0] = done[1] = done[2] = 0;
        fence_mbar_init();
    }
    __syncthreads();

    // this CTA's lines: whole packed blocks
    const int blocks_per = (a.nblk + S - 1) / S;
    const int blk0 = min(a.nblk, rank * blocks_per), blk1 = min(a.nblk, blk0 + blocks_per);
    const int nb = blk1 - blk0;
    const float *xsrc = (cls ? job.xc : job.xr) + (long)blockIdx.y * a.nblk * n * kColF;
    // TMA pipeline: block q lives in buffer q % nbuf.  Blocks 0..nbuf-1 are issued up front;
    // block q + nbuf is issued by the last warp to finish block q (shared counter), so warps
    // are never barrier-synchronised per block and can drift up to nbuf - 1 blocks apart.
    const int nbuf = a.nbuf;
    if (threadIdx.x == 0) {
        for (int q = 0; q < min(nbuf, nb); ++q)
            issue_block(smem + q * stage_f + kPadL * kColF, xsrc + (long)(blk0 + q) * n * kColF, n,
                        &full[q]);
    }

    // ---- 3. tasks: (angle k, 32-bin chunk) pairs dealt round-robin to the warps, so every
    // warp holds a mix of angles (near-0 and near-45 degree angles have different footprints)
    const int ntask = kcnt * a.chunks;
    const float fn1 = (float)(n - 1);
    float acc[kMaxT][BB];
#pragma unroll
    for (int t = 0; t < kMaxT; ++t)
#pragma unroll
        for (int b = 0; b < BB; ++b) acc[t][b] = 0.f;

    for (int i = 0; i < nb; ++i) {
        const int lb = (blk0 + i) * R;
        const int cb = i % nbuf;
        const float *cur = smem + cb * stage_f;
        mbar_wait(&full[cb], (unsigned)((i / nbuf) & 1));
#pragma unroll
        for (int t = 0; t < kMaxT; ++t) {
            const int tau = warp + kWarps * t;
            if (tau >= ntask) break;  // warp-uniform
            const int k = tau / a.chunks;
            const int chunk = tau - k * a.chunks;
            const int j = chunk * 32 + lane;
            const double Pl = sPl[k];
            const double ad = sP0[k] + (double)lb * Pl + (double)j * sPj[k];
            const double fl = floor(ad);
            const int base = (int)fl;
            const float frac = (float)(ad - fl);
            const float ab = sAbsB[k], sec = sSec[k], plf = sPlf[k];
            // does any bin of this chunk see a line of this block?
            const float span = (float)(R - 1) * plf;
            const float lo = (float)base + frac + fminf(0.f, span);
            const float hi = (float)base + frac + fmaxf(0.f, span);
            const bool act = j < n_det && hi + sec > 0.f && lo - sec < fn1;
            if (!__any_sync(0xffffffffu, act)) continue;
            const float c1 = 2.f * ab - 1.f, c2 = 2.f - 3.f * ab;
            const float fs = frac - sec;
            float blk[BB];
#pragma unroll
            for (int b = 0; b < BB; ++b) blk[b] = 0.f;
#pragma unroll
            for (int s = 0; s < R; ++s) {
                const int l = (lane + s) & (R - 1);
                // e = a* - 1/|beta| relative to base; candidate_0 = floor(e) + 1 and with
                // phi = e - floor(e) the hat weights of the 3 candidates are
                //   w0 = |b| (1 - phi), w1 = 1 - |2|b| - 1 - |b| phi|, w2 = 2 - 3|b| + |b| phi
                const float e = fmaf((float)l, plf, fs);
                const float fl2 = floorf(e);
                const float phi = e - fl2;
                int ci = base + (int)fl2 + 1;
                ci = min(max(ci, -3), n);
                const float w0 = fmaf(-ab, phi, ab);
                const float w1 = 1.f - fabsf(fmaf(-ab, phi, c1));
                const float w2 = fmaf(ab, phi, c2);
                const float *px = cur + (ci + kPadL) * kColF + l * BB;
                float v0[BB], v1[BB], v2[BB];
                ld_px<BB>(px, v0);
                ld_px<BB>(px + kColF, v1);
#pragma unroll
                for (int b = 0; b < BB; ++b) blk[b] = fmaf(w1, v1[b], fmaf(w0, v0[b], blk[b]));
                if (w2 > 0.f) {
                    ld_px<BB>(px + 2 * kColF, v2);
#pragma unroll
                    for (int b = 0; b < BB; ++b) blk[b] = fmaf(w2, v2[b], blk[b]);
                }
            }
#pragma unroll
            for (int b = 0; b < BB; ++b) acc[t][b] += blk[b];
        }
        // release the buffer; the last warp out refills it with block i + nbuf
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();  // this warp's reads of the buffer are complete
            const int old = atomicAdd(&done[cb], 1);
            if (old == kWarps * (i / nbuf + 1) - 1 && i + nbuf < nb) {
                fence_proxy_async();  // generic-proxy reads -> async-proxy writes
                issue_block(smem + cb * stage_f + kPadL * kColF,
                            xsrc + (long)(blk0 + i + nbuf) * n * kColF, n, &full[cb]);
            }
        }
    }
    __syncthreads();  // all blocks consumed: the buffers become the partials array

    // ---- 4. partials -> shared memory [kcnt][n_det][BB], then fixed-order cluster sum
    float *part = smem;
#pragma unroll
    for (int t = 0; t < kMaxT; ++t) {
        const int tau = warp + kWarps * t;
        if (tau >= ntask) break;
        const int k = tau / a.chunks;
        const int j = (tau - k * a.chunks) * 32 + lane;
        if (j < n_det) {
#pragma unroll
            for (int b = 0; b < BB; ++b) part[((long)k * n_det + j) * BB + b] = acc[t][b];
        }
    }
    cluster.sync();
    const int T = kcnt * n_det * BB;
    const int per = (T + S - 1) / S;
    const int o0 = rank * per, o1 = min(T, o0 + per);
    const long img_stride = (long)a.m * n_det;
    for (int o = o0 + threadIdx.x; o < o1; o += kThreads) {
        float s = 0.f;
        for (int q = 0; q < S; ++q) s += cluster.map_shared_rank(part, q)[o];
        const int b = o % BB;
        const int kj = o / BB;
        const int k = kj / n_det, j = kj - k * n_det;
        job.p[(long)(b0 + b) * img_stride + (long)sSlot[k] * n_det + j] = s;
    }
    cluster.sync();
}

// Cluster size S (line split): the number of busy units is about jobs * groups * (m/K + 1);
// pick S in [2, 8] so that busy CTAs fill whole waves of 2 CTAs per SM.
int pick_cluster(long units, int num_sms, int ctas_per_sm) {
    const long slots = (long)num_sms * ctas_per_sm;
    int best = 4;
    double best_cost = 1e30;
    for (int S = 2; S <= 8; ++S) {
        const long ctas = units * S;
        const double waves = (double)((ctas + slots - 1) / slots);
        const double cost = waves / S * (1.0 + 0.02 * S);  // per-CTA reduction overhead
        if (cost < best_cost) {
            best_cost = cost;
            best = S;
        }
    }
    return best;
}

template <int BB>
cudaError_t launch_bb(FwdArgs a, int njobs, int num_sms, cudaStream_t s) {
    constexpr int R = kColF / BB;
    a.nblk = (a.g.n + R - 1) / R;
    const size_t stage_b = sizeof(float) * (size_t)(a.g.n + kPadL + kPadR) * kColF;
    const size_t part_b = sizeof(float) * (size_t)a.K * a.g.n_det * BB;
    const size_t limit = 225 * 1024;  // dynamic shared memory budget per CTA (1 CTA / SM)
    a.nbuf = 3 * stage_b <= limit ? 3 : (2 * stage_b <= limit ? 2 : 1);
    size_t smem = a.nbuf * stage_b;
    if (part_b > smem) smem = part_b;
    if (smem > limit) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(k_radon_fwd<BB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ngroups = (a.m + a.K - 1) / a.K;  // per class, worst case
    const long busy = (long)njobs * (a.B / BB) * ((a.m + a.K - 1) / a.K + 1);
    const int S = pick_cluster(busy, num_sms, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(S * 2 * ngroups), (unsigned)(a.B / BB), (unsigned)njobs);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_radon_fwd<BB>, a);
    if (e != cudaSuccess) return e;
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
    if (a.K > kKMax) a.K = kKMax;
    if (a.K < 1) return cudaErrorInvalidValue;  // n_det > kWarps * kMaxT * 32
    const int bb = pick_bb(B, idx_stride);
    switch (bb) {
        case 4: return launch_bb<4>(a, njobs, plan->num_sms, s);
        case 2: return launch_bb<2>(a, njobs, plan->num_sms, s);
        default: return launch_bb<1>(a, njobs, plan->num_sms, s);
    }
}

}  // namespace skei
