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
//     per pixel — so a whole block is ONE TMA bulk copy (cp.async.bulk + mbarrier, up to
//     triple-buffered, issued by one thread: no staging instructions, no registers) and one
//     LDS.BB fetches a candidate pixel of BB images.
//   * Work unit = (job, group of BB images sharing the sketch, class, group of K angles);
//     staged pixels are reused by all K angles of the unit.  The kernel is persistent (one
//     CTA per SM) and stream-K scheduled: the U x nblk (unit, line block) work is cut into
//     equal contiguous ranges, one per CTA, so every SM streams the same number of blocks;
//     a unit cut by a range boundary is finished by the last of its pieces (see step 4).
//     With 0.9-1 units per CTA (cfg3: 144 units on 148 SMs) every CTA takes one whole unit.
//     The block stream continues across units, so the next unit's first blocks are in
//     flight while the current unit's epilogue runs.
//   * Bank-conflict-free gathers: lane L visits the lines of a block in the order
//     l = L' ^ gray(s) (L' = L mod R).  The lanes of one shared-memory phase (8 lanes for
//     LDS.128, 16 for LDS.64, 32 for LDS.32) then read R distinct line slots, i.e. distinct
//     banks, whatever pixel each lane's bin needs (a lane-per-bin layout gives 2-way
//     conflicts at every angle with |beta| < 1 because 8 bins span more than 8 pixels), and
//     consecutive lines differ in one bit, so the position moves by one add per line.
//   * 512 threads (<= 128 registers each), one CTA per SM.  Task = (angle, 64 consecutive
//     bins); lane L owns the bin pair (c0 + 2L, c0 + 2L + 1), whose line positions differ by
//     1/|beta|, so per line the pair needs the 3-5 consecutive candidate pixels c0..c4: c0
//     feeds the lower bin, c1 and c2 both, c3 (and c4) the upper one.  A thread owns up to
//     kMaxT tasks (4 for groups of 4 images) and keeps 2 x BB accumulators per task in
//     registers: K = 16 kMaxT / chunks angles per unit.  A class's angles are dealt to its
//     units round-robin (every unit mixes angles from the whole class range, so units cost
//     about the same).  Per unit the block table counts, for every chunk, the blocks it
//     touches; chunks touching none are dropped (their bins written as 0) and the rest dealt
//     to the 16 warps by that cost in snake order.  A warp's next task descriptor is loaded
//     one task ahead.  The line loop is compiled with and without the fifth candidate and
//     picked per task (warp-uniform: |beta| of the task's angle).
//   * Decoupled pipeline: no per-block barrier.  The last warp to finish a staged block
//     (shared-memory counter) refills its buffer with the block nbuf ahead, so warps drift
//     up to nbuf - 1 blocks apart and per-block load imbalance averages out.
//   * Per (bin pair, line): the lower bin's line position from an fp64 per-block base plus
//     an fp32 offset (split precision), floor / fraction, one unsigned-min clamp
//     into the zero pad columns, 7 hat weights, 3-5 LDS.BB (c3 / c4 only where their weight
//     is > 0) issued kAhead = 1 line ahead of use, 6-7 x BB/2 packed fp32x2 FFMA2.  The R lines
//     of a block are summed into a partial before it is added to the running total
//     (two-level summation).  A chunk skips a block none of its bins sees.
//   * Unit end: a whole unit's sums are complete in registers -> p; for the MC job also
//     r = p - y_S and per-unit partial sums of r^2, summed in a fixed order by the last CTA
//     to finish (completion counter).  A split unit's pieces go to L2 slots and the last
//     piece to arrive adds them in CTA order (deterministic, no float atomics).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "internal.h"
#include "tma.h"

namespace skei {
namespace {

#ifndef SKEI_FWD_THREADS
#define SKEI_FWD_THREADS 512
#endif
constexpr int kThreads = SKEI_FWD_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxQ = 1024; // image groups per launch (shared-memory unit table)
constexpr int kChunk = 64;  // bins per task: lane L owns the pair c0 + 2L, c0 + 2L + 1
// task slots per warp (each lane: kMaxT * 2 * BB accumulator registers)
#ifndef SKEI_FWD_KT4
#define SKEI_FWD_KT4 4
#endif
template <int BB>
constexpr int max_tasks() { return BB == 4 ? SKEI_FWD_KT4 : BB == 2 ? 8 : 8; }
// max over BB of kMaxT * BB (a split unit's piece: K * n_det * BB <= kWarps * kMaxT * kChunk * BB
// floats) and min over BB of kMaxT (the most units an image group can have)
constexpr int cmax_(int a, int b) { return a > b ? a : b; }
constexpr int kMaxTaskBB = cmax_(cmax_(4 * max_tasks<4>(), 2 * max_tasks<2>()), max_tasks<1>());
constexpr int kMinTasks = max_tasks<4>() < max_tasks<2>() ? max_tasks<4>() : max_tasks<2>();
static_assert(kMinTasks <= max_tasks<1>(), "");
constexpr int kKMax = 16;   // angles per CTA
constexpr int kSmallK = 3, kSmallBlocks = 8;  // small problems: see launch_bb
#ifndef SKEI_FWD_AHEAD
#define SKEI_FWD_AHEAD 1
#endif
constexpr int kAhead = SKEI_FWD_AHEAD;  // pixel loads issued this many lines ahead of use
#ifndef SKEI_FWD_C3_ALWAYS
#define SKEI_FWD_C3_ALWAYS 0  // load the fourth candidate unconditionally (A/B knob)
#endif
#ifndef SKEI_FWD_STATS_EVERY
#define SKEI_FWD_STATS_EVERY 37  // -DSKEI_FWD_STATS: print the counters of every n-th CTA
#endif
#ifndef SKEI_FWD_STRIDED
#define SKEI_FWD_STRIDED 1  // a unit takes every ng-th angle of its class (A/B knob)
#endif
#ifndef SKEI_FWD_WHOLE
#define SKEI_FWD_WHOLE 1  // whole units per CTA when there are 0.9 - 1 units per CTA (A/B knob)
#endif
#ifndef SKEI_FWD_WCOST
#define SKEI_FWD_WCOST 1  // task costs weighted by the angle's expected per-line work (A/B knob)
#endif
#ifndef SKEI_FWD_WT_CAND
#define SKEI_FWD_WT_CAND 10.0
#endif
#ifndef SKEI_FWD_WT_WIDE
#define SKEI_FWD_WT_WIDE 6.0
#endif
constexpr double kWtBase = 31.0, kWtCand = SKEI_FWD_WT_CAND, kWtWide = SKEI_FWD_WT_WIDE;
#ifndef SKEI_FWD_WIDE_SPLIT
#define SKEI_FWD_WIDE_SPLIT 1  // compile the line loop with / without the fifth candidate
#endif
constexpr int kMaxPieces = 256;  // pieces of one split unit (<= CTAs <= 256)
constexpr int kMaxDevices = 64;  // devices with cached launch attributes
constexpr int kMaxBand = 64;     // band angles of the source class considered for a move
#ifndef SKEI_FWD_BAND
#define SKEI_FWD_BAND 1  // flexible class band near the diagonals (A/B knob)
#endif
// Floating tasks (A/B knob, off): the unit's SKEI_FWD_FLOAT costliest tasks are not dealt to a
// warp; a warp done with its own tasks of a staged block takes them from the block's queue
// and adds their block sums, in block order, to sums kept in shared memory (bitwise the
// same results; parity suite green with 10).  Measured at cfg3 (round 2, session 5): the
// warps' mbarrier wait fell from 13% to 3% of their time, but every (task, block) pair got
// 16-20% slower and the kernel went from 264.8 to 269.5 us (6 floating tasks: 278.6): with
// all 16 warps busy the SM's shared-memory pipe / issue slots are the limit, i.e. the "wait"
// of the static deal is time in which the other warps run faster, not idle capacity.
#ifndef SKEI_FWD_FLOAT
#define SKEI_FWD_FLOAT 0
#endif
#ifndef SKEI_FWD_LANE_SKIP
#define SKEI_FWD_LANE_SKIP 0  // A/B knob: lanes outside the block's bin range skip the line loop
#endif
constexpr int kMaxFloat = SKEI_FWD_FLOAT < kWarps ? SKEI_FWD_FLOAT : kWarps;
constexpr int kFloatBytes = 32 * 2 * 4 * (int)sizeof(float);  // a floating task's sums (BB = 4)
constexpr int kCand = 5;    // candidate pixels of a bin pair per line
constexpr int kPadL = 5;    // zero pixel columns left of the line data (candidates from -5)
constexpr int kPadR = 8;    // ... and right of it (candidates reach n + 4; a column block
                            // staged from the row-packed copy spans R ceil(n / R) <= n + 7)
constexpr int kColF = 32;   // floats per staged pixel column (R * BB)

struct FwdArgs {
    FwdJob job[2];
    int njobs;
    const int32_t *idx;
    int m, idx_stride, B, nq;  // nq = image groups = B / BB (fused: B)
    // job-fused groups (BB = 2): group q is image q, its slots 0 / 1 are job 0 / job 1 (x1 and
    // x2 of one image share its sketch, so they share the projector's geometry); job[0].xr /
    // xc hold the fused packed layout, slot b's projections go to job[b].p, MC on slot 0
    int fused;
    int nfloat;  // floating tasks per unit (<= kMaxFloat; 0: every task is pinned to a warp)
    int K;       // angles per unit: K * chunks <= kWarps * kMaxT tasks
    int chunks;  // ceil(n_det / 32)
    int nblk;    // packed blocks per image group (ceil(n / R))
    int nbuf;    // staging buffers
    Geom g;
    // fused MC residual of job 0 (job.y != NULL): partials [B][mc_slots], counter, mc [B]
    float *mc_part;
    int mc_slots;
    unsigned *mc_ctr;
    float *mc_out;
    // flexible class band (shared sketches; 0 = off): angles within `band` index units of a
    // diagonal (|4 i - n_full| or |4 i - 3 n_full| <= band, i.e. min(|cos|, |sin|) >= 0.68)
    // are exact in either class (the line loop holds for |beta| >= 2/3), so a few of them may
    // change class to make the class sizes multiples of K (fewer, whole units)
    int band;
    unsigned *queue;  // piece counters of the stream-K split units, indexed by the unit's
                      // first CTA (< gridDim.x; zero before the launch, self-resetting)
    float *scratch;   // split-unit pieces [gridDim.x][2][K * n_det * BB]
    // tm_col (groups of 4, job.xc == NULL): the column class is staged from the ROW-packed
    // copy through job j's 4-D tensor map tm[j] — dims (image 4, column n, line 8, row block
    // nq nblk), byte strides (128, 16, 128 n) — whose box (4, 8, 8, nblk) lands in shared
    // memory as [row][column][image], the column-packed block (a transposing copy: 16-byte
    // runs), so rotate + pack writes one packed copy per image instead of two
    int tm_col;
    CUtensorMap tm[2];
};

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

// ld.shared of one staged pixel of BB images at a 32-bit shared-window address
template <int BB>
__device__ __forceinline__ void lds_px(unsigned addr, float (&v)[BB]) {
    if constexpr (BB == 4) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                     : "r"(addr));
    } else if constexpr (BB == 2) {
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v[0]), "=f"(v[1]) : "r"(addr));
    } else {
        asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v[0]) : "r"(addr));
    }
}

// L2 (ld.global.cg) load of BB consecutive floats (16-byte aligned for BB = 4)
template <int BB>
__device__ __forceinline__ void ldcg_vec(const float *p, float (&v)[BB]) {
    if constexpr (BB == 4) {
        const float4 t = __ldcg(reinterpret_cast<const float4 *>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if constexpr (BB == 2) {
        const float2 t = __ldcg(reinterpret_cast<const float2 *>(p));
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = __ldcg(p);
    }
}

// blk += w v over BB images, as packed fp32x2 FMAs (bitwise the same as scalar fmaf)
template <int BB>
__device__ __forceinline__ void fma_px(float (&blk)[BB], float w, const float (&v)[BB]) {
    if constexpr (BB == 1) {
        blk[0] = fmaf(w, v[0], blk[0]);
    } else {
        const float2 w2 = make_float2(w, w);
#pragma unroll
        for (int b = 0; b < BB; b += 2) {
            const float2 r = __ffma2_rn(w2, make_float2(v[b], v[b + 1]), make_float2(blk[b], blk[b + 1]));
            blk[b] = r.x;
            blk[b + 1] = r.y;
        }
    }
}

// L2 (st.global.cg) store of BB consecutive floats
template <int BB>
__device__ __forceinline__ void stg_vec(float *p, const float (&v)[BB]) {
    if constexpr (BB == 4) {
        __stcg(reinterpret_cast<float4 *>(p), make_float4(v[0], v[1], v[2], v[3]));
    } else if constexpr (BB == 2) {
        __stcg(reinterpret_cast<float2 *>(p), make_float2(v[0], v[1]));
    } else {
        __stcg(p, v[0]);
    }
}

// Work decomposition shared by every CTA: for each image group q, nrow[q] = angles of its
// sketch in the row class; units of q = ceil(nrow/K) + ceil((m - nrow)/K); uoff = prefix.
struct Units {
    const int *uoff;  // [nq + 1]
    const int *nrow;  // [nq]
    int per_job;      // uoff[nq]
};
struct UnitId {
    int job, q, cls, grp;
};
__device__ __forceinline__ UnitId decode_unit(const Units &U, int nq, int K, int u) {
    UnitId d;
    d.job = u / U.per_job;
    const int rem = u - d.job * U.per_job;
    int lo = 0, hi = nq - 1;  // last q with uoff[q] <= rem
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (U.uoff[mid] <= rem) lo = mid; else hi = mid - 1;
    }
    d.q = lo;
    const int gi = rem - U.uoff[lo];
    const int gr = (U.nrow[lo] + K - 1) / K;
    d.cls = gi < gr ? 0 : 1;
    d.grp = d.cls ? gi - gr : gi;
    return d;
}

template <int BB, bool FUSED>
__global__ void __launch_bounds__(kThreads, 1) k_radon_fwd(const __grid_constant__ FwdArgs a) {
    constexpr int R = kColF / BB;
    constexpr int kMaxT = max_tasks<BB>();
    extern __shared__ __align__(128) float smem_raw[];
    // nbuf stage buffers from a 128-byte aligned base (the line-offset XOR below needs it)
    float *smem = smem_raw + (((128u - (smem_u32(smem_raw) & 127u)) & 127u) >> 2);
    __shared__ __align__(8) uint64_t full[3];
    __shared__ int done[3];  // warps that finished each buffer (monotonic)
    __shared__ double sP0[kKMax], sPj[kKMax], sPl[kKMax];
    __shared__ float sAbsB[kKMax];
    // per unit angle k, one 48-byte record (one base address per task in the block loop):
    // [0] |beta|, 1/|beta|, Pl, min(Pj, 0); [1] hat offsets 2|b| - 1, 3|b| - 2, 4|b| - 2,
    // 5|b| - 2; [2].x Pj (all fp32)
    __shared__ float4 sAngT[kKMax][3];
    __shared__ int sSlot[kKMax];
    __shared__ int sWt[kKMax];  // per unit angle: cost weight of one (task, block) pair
    __shared__ int sCount;
    __shared__ int s_uoff[kMaxQ + 1], s_nrow[kMaxQ];
    __shared__ int s_mv[3];           // class band moves: shift (+: col -> row), key bound (D, I)
    __shared__ int s_bkey[kMaxBand];  // the source side's band angles, key = (dist << 16) | index
    __shared__ float s_red[kWarps][BB];
    __shared__ bool s_last;
    __shared__ int4 s_task[kWarps * kMaxT];  // per task: angle slot, chunk bin, chunk Pj split
    __shared__ int s_cost[kWarps * kMaxT];   // per task: blocks its chunk touches
    // floating tasks (the unit's costliest): any warp that has finished its own tasks of a
    // staged block takes them from the block's queue; their running sums live in shared memory
    __shared__ int4 s_float[kMaxFloat > 0 ? kMaxFloat : 1];
    __shared__ int s_fseq[kMaxFloat > 0 ? kMaxFloat : 1];  // next block whose sum may be added
    __shared__ int s_fq[3];                                // per buffer: grabs so far (unit)
    __shared__ int s_nfl;
    __shared__ int s_defer[2], s_dnpc[2];  // split units this CTA finishes after its stream
    __shared__ int s_dpiece[2][kMaxPieces];  // ... their piece slots in CTA order

    const int cid = blockIdx.x, ncl = gridDim.x;
    const int n = a.g.n, n_det = a.g.n_det, n_full = a.g.n_full;
    const int K = a.K, nq = a.nq;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int stage_f = (n + kPadL + kPadR) * kColF;
    int4 *btab = reinterpret_cast<int4 *>(smem + a.nbuf * stage_f);  // [K][nb] block table
    // [nfloat][32 lanes][2 BB] sums of the floating tasks, behind the block table
    float *facc = reinterpret_cast<float *>(btab + (size_t)a.K * a.nblk);
    constexpr bool kFloat = kMaxFloat > 0 && BB == 4 && !FUSED;
    const int nfloat = kFloat ? a.nfloat : 0;
    const long part_f = (long)K * n_det * BB;
    SKEI_DCHECK(part_f <= (long)kWarps * kMaxTaskBB * kChunk && ncl <= kMaxPieces && K <= kKMax &&
                    nq <= kMaxQ,
                "forward scratch / piece / table sizes");

    // ---- 1. the class rule and the class sizes per image group -> unit table (identical in
    // every CTA).  Strict rule: row class iff |cos| >= |sin| (4 i <= n_full or 4 i >= 3 n_full).
    // With a flexible band (shared sketch): the shift s in [-a, b] (a / b: band angles strictly
    // in the row / column class) that minimises ceil(n_row / K) + ceil(n_col / K), smallest |s|
    // first; the |s| band angles nearest a diagonal (key (distance, index)) change class.
    auto strict_row = [&](int i) { return (4 * i <= n_full) || (4 * i >= 3 * n_full); };
    auto diag_dist = [&](int i) { return min(abs(4 * i - n_full), abs(4 * i - 3 * n_full)); };
    if (warp == 0) {
        int nr0 = 0, na = 0, nb = 0;
        if (a.band > 0) {
            for (int base = 0; base < a.m; base += 32) {
                const int k = base + lane;
                bool r = false, ba = false, bb = false;
                if (k < a.m) {
                    const int i = a.idx[k];
                    r = strict_row(i);
                    const bool bd = diag_dist(i) <= a.band;
                    ba = bd && r;
                    bb = bd && !r;
                }
                nr0 += __popc(__ballot_sync(0xffffffffu, r));
                na += __popc(__ballot_sync(0xffffffffu, ba));
                nb += __popc(__ballot_sync(0xffffffffu, bb));
            }
        }
        int sh = 0;
        if (a.band > 0) {
            auto units_of = [&](int nr) { return (nr + K - 1) / K + (a.m - nr + K - 1) / K; };
            int best = units_of(nr0);
            for (int t = 1; t <= max(na, nb); ++t) {
                if (t <= na && units_of(nr0 - t) < best) { best = units_of(nr0 - t); sh = -t; }
                if (t <= nb && units_of(nr0 + t) < best) { best = units_of(nr0 + t); sh = t; }
            }
            sh = max(-kMaxBand, min(kMaxBand, sh));
        }
        int nsrc = 0;  // the source side's band angles -> s_bkey
        if (sh != 0) {
            for (int base = 0; base < a.m; base += 32) {
                const int k = base + lane;
                bool src = false;
                int key = 0;
                if (k < a.m) {
                    const int i = a.idx[k];
                    src = diag_dist(i) <= a.band && (sh < 0) == strict_row(i);
                    key = (diag_dist(i) << 16) | i;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, src);
                const int pre = nsrc + __popc(bal & ((1u << lane) - 1u));
                if (src && pre < kMaxBand) s_bkey[pre] = key;
                nsrc += __popc(bal);
            }
            nsrc = min(nsrc, kMaxBand);
            __syncwarp();
            for (int e = lane; e < nsrc; e += 32) {  // the |s|-th smallest key bounds the moves
                const int key = s_bkey[e];
                int rk = 0;
                for (int o = 0; o < nsrc; ++o) rk += s_bkey[o] < key;
                if (rk == abs(sh) - 1) s_mv[1] = key;
            }
        }
        if (lane == 0) {
            s_mv[0] = sh;
            if (sh == 0) s_mv[1] = -1;
        }
    }
    __syncthreads();
    const int mv_sh = s_mv[0], mv_key = s_mv[1];
    auto is_row = [&](int i) -> bool {
        const bool st = strict_row(i);
        if (mv_sh == 0 || diag_dist(i) > a.band || (mv_sh < 0) != st) return st;
        return ((diag_dist(i) << 16) | i) <= mv_key ? !st : st;
    };
    for (int q = warp; q < nq; q += kWarps) {
        const int32_t *iq = a.idx + (a.idx_stride ? (long)q * (FUSED ? 1 : BB) * a.idx_stride : 0);
        int cnt = 0;
        for (int base = 0; base < a.m; base += 32) {
            const int k = base + lane;
            bool row = false;
            if (k < a.m) row = is_row(iq[k]);
            cnt += __popc(__ballot_sync(0xffffffffu, row));
        }
        if (lane == 0) s_nrow[q] = cnt;
    }
    // zero pad columns of every stage buffer (never written by the bulk copies)
    for (int e = threadIdx.x; e < a.nbuf * (kPadL + kPadR) * kColF; e += kThreads) {
        const int bi = e / ((kPadL + kPadR) * kColF);
        const int e2 = e - bi * (kPadL + kPadR) * kColF;
        const int qq = e2 / kColF, w = e2 - qq * kColF;
        const int col = qq < kPadL ? qq : kPadL + n + (qq - kPadL);
        smem[bi * stage_f + col * kColF + w] = 0.f;
    }
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&full[2], 1);
        done[0] = done[1] = done[2] = 0;
        s_defer[0] = s_defer[1] = -1;
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc_u = 0;
        for (int q = 0; q < nq; ++q) {
            s_uoff[q] = acc_u;
            acc_u += (s_nrow[q] + K - 1) / K + (a.m - s_nrow[q] + K - 1) / K;
        }
        s_uoff[nq] = acc_u;
    }
    __syncthreads();
    const Units U{s_uoff, s_nrow, s_uoff[nq]};
    const int total_units = a.njobs * U.per_job;
    // ---- stream-K work split: the work is W = U x nblk line blocks; CTA c takes the
    // contiguous range [w(c), w(c+1)), w(c) = c W / ncl, so every CTA streams the same number
    // of blocks whatever U is.  A unit cut by a range boundary is computed in pieces by
    // consecutive CTAs: each piece's partial projection goes to an L2 slot, and the last
    // piece to finish (per-unit counter) adds the pieces in CTA order and finishes the unit.
    const int nbc = a.nblk;
    const long W = (long)total_units * nbc;
    // nearly one unit per CTA (0.9 ncl <= U <= ncl, e.g. cfg3's 144 units on 148 SMs): whole
    // units, one per CTA — no split units, so no piece stores, fix-ups or second prologue /
    // epilogue, for at most 1/0.9 of the per-CTA blocks
    const bool whole = SKEI_FWD_WHOLE && total_units <= ncl && 10L * total_units >= 9L * ncl;
    auto wstart = [&](int c) -> long {
        return whole ? (long)min(c, total_units) * nbc : (long)c * W / ncl;
    };
    const long w0 = wstart(cid), w1 = wstart(cid + 1);
    const int u_first = (int)(w0 / nbc), u_last = w1 > w0 ? (int)((w1 - 1) / nbc) : u_first - 1;
    auto cta_of = [&](long w) -> int {  // the CTA whose range holds block w
        int c = (int)(w * ncl / W);
        while (c + 1 < ncl && wstart(c + 1) <= w) ++c;
        while (c > 0 && wstart(c) > w) --c;
        return c;
    };
    float *pieces = a.scratch;  // [ncl][2][part_f]: the pieces of a CTA's first / last unit

    // this CTA's blocks of unit u: [lo, hi)
    auto unit_blocks = [&](int u, int &lo, int &hi) {
        lo = (int)max(w0 - (long)u * nbc, 0L);
        hi = (int)min(w1 - (long)u * nbc, (long)nbc);
    };
    int G = 0;  // this CTA's block stream: its blocks of u_first .. u_last in order
    for (int u = u_first; u <= u_last; ++u) {
        int lo, hi;
        unit_blocks(u, lo, hi);
        G += hi - lo;
    }
    // stage block g of this CTA's stream into buffer b: one bulk copy of the packed block, or
    // (tm_col, column class) one transposing tensor-map box from the row-packed copy
    auto issue = [&](int g, int b) {
        for (int u = u_first;; ++u) {
            int lo, hi;
            unit_blocks(u, lo, hi);
            if (g < hi - lo) {
                const UnitId d = decode_unit(U, nq, K, u);
                const FwdJob &jb = d.job ? a.job[1] : a.job[0];
                SKEI_DCHECK(d.q < nq && lo + g < a.nblk && d.job < a.njobs, "forward block source");
                float *dst = smem + b * stage_f + kPadL * kColF;
                if (d.cls == 1 && a.tm_col) {
                    mbar_expect_tx(&full[b], (unsigned)(a.nblk * R * kColF * sizeof(float)));
                    tma_load_4d(dst, &a.tm[d.job], 0, (lo + g) * R, 0, d.q * a.nblk, &full[b]);
                } else {
                    issue_block(dst, (d.cls ? jb.xc : jb.xr) + ((long)d.q * a.nblk + lo + g) * n * kColF, n,
                                &full[b]);
                }
                return;
            }
            g -= hi - lo;
        }
    };
    // TMA pipeline: block g lives in buffer g % nbuf; blocks 0..nbuf-1 are issued up front,
    // block g + nbuf by the last warp to finish block g (shared counter), so warps are not
    // barrier-synchronised per block and the stream runs on across unit boundaries.
    const int nbuf = max(1, min(a.nbuf, G));
    if (threadIdx.x == 0) {
        fence_proxy_async();  // the zeroed pads (a tensor-map box may rewrite some, as zeros)
        for (int g = 0; g < nbuf && g < G; ++g) issue(g, g);
    }

    // this lane's line order: the s-th line visited is l = lane' ^ gray(s) (lane' = lane mod R,
    // gray(s) = s ^ (s >> 1)), so the 32 / BB lanes of one shared-memory phase read R distinct
    // lines (distinct bank groups) whatever pixels they hit, and consecutive lines differ in
    // one bit i: the position e moves by +-2^i Pl (one add, signs fixed per lane and step).
    constexpr int LB = R == 32 ? 5 : R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const int lane_r = lane & (R - 1);
    const float lf0 = (float)lane_r;
    const float lane2f = (float)(2 * lane - 31);  // the lane's pair relative to the chunk's middle
    float sgn[LB];  // +-2^i: + if bit i of lane' is 0 (flipping it on moves the line up)
#pragma unroll
    for (int i = 0; i < LB; ++i) sgn[i] = ((lane_r >> i) & 1) ? -(float)(1 << i) : (float)(1 << i);
    // byte offset of line lane' in a staged pixel column (the clamp below addresses pixel
    // columns from the first pad column, kPadL = kCand); bits 0..6, the buffer bases are
    // 128-byte aligned
    static_assert(kPadL == kCand && kPadR >= kCand, "pads must hold a whole candidate window");
    const unsigned lofs0 = (unsigned)(lane_r * BB * sizeof(float));
    const unsigned smem_b = smem_u32(smem);
    const unsigned cmax = (unsigned)(n + kCand);

#ifdef SKEI_FWD_STATS
    long long st_wait = 0, st_epi = 0, st_pro = 0, st_active = 0, st_lanes = 0;
    long long st_tc[kMaxT] = {}, st_tn[kMaxT] = {};  // per task slot: cycles, active blocks
    long long st_fl = 0;  // floating (task, block) pairs this warp ran
    const long long st_t0 = clock64();
#endif
    int gbase = 0;  // stream index of the current unit's first block
    for (int u = u_first; u <= u_last; ++u) {
        int ulo, uhi;
        unit_blocks(u, ulo, uhi);
        const int nbu = uhi - ulo;  // this CTA's blocks of the unit
        const bool full_unit = w0 <= (long)u * nbc && (long)(u + 1) * nbc <= w1;
#ifdef SKEI_FWD_STATS
        const long long tp0 = clock64();
#endif
        const UnitId d = decode_unit(U, nq, K, u);
        const FwdJob job = d.job ? a.job[1] : a.job[0];
        const int b0 = FUSED ? d.q : d.q * BB;  // the group's first image (fused: its image)
        const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);

        // ---- 2. the unit's angles + geometry: the class's angles (in sketch order) are dealt to
        // its ngc = ceil(n_class / K) units round-robin, unit grp taking ranks grp, grp + ngc, ...
        // (strided: every unit mixes angles from the whole class range, so units cost about
        // the same — a unit of consecutive angles near 0 degrees projects onto ~1.4x the bins
        // of one near 45 — and sizes differ by at most one angle)
        const int ncls = d.cls == 0 ? s_nrow[d.q] : a.m - s_nrow[d.q];
        const int ngc = (ncls + K - 1) / K;
        (void)ngc;
        if (warp == 0) {
            int seen = 0;
            for (int base = 0; base < a.m; base += 32) {
                const int k = base + lane;
                bool in = false;
                if (k < a.m) {
                    const int i = idx[k];
                    const bool row_class = is_row(i);
                    in = (d.cls == 0) ? row_class : !row_class;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pre = seen + __popc(bal & ((1u << lane) - 1u));
#if SKEI_FWD_STRIDED
                if (in && pre % ngc == d.grp) sSlot[pre / ngc] = k;
#else
                if (in && pre >= d.grp * K && pre < d.grp * K + K) sSlot[pre - d.grp * K] = k;
#endif
                seen += __popc(bal);
            }
#if SKEI_FWD_STRIDED
            const int cnt = max(0, (seen - d.grp + ngc - 1) / ngc);
#else
            const int cnt = max(0, min(K, seen - d.grp * K));
#endif
            if (lane == 0) sCount = cnt;
            __syncwarp();
            if (lane < cnt) {
                const double2 cs = a.g.trig[idx[sSlot[lane]]];
                const double c = cs.x, sn = cs.y, h = a.g.h, hd = a.g.hd;
                double P0, Pj, Pl, ab;
                if (d.cls == 0) {  // lines = rows r, along = columns
                    P0 = h - (hd + h * sn) / c;
                    Pj = 1.0 / c;
                    Pl = sn / c;
                    ab = fabs(c);
                } else {  // lines = columns c, along = rows
                    P0 = h + (hd - h * c) / sn;
                    Pj = -1.0 / sn;
                    Pl = c / sn;
                    ab = fabs(sn);
                }
                sP0[lane] = P0;
                sPj[lane] = Pj;
                sPl[lane] = Pl;
                sAbsB[lane] = (float)ab;
                sAngT[lane][2] = make_float4((float)Pj, 0.f, 0.f, 0.f);
                sAngT[lane][0] = make_float4((float)ab, (float)(1.0 / ab), (float)Pl,
                                         (float)fmin(Pj, 0.0));
                sAngT[lane][1] = make_float4((float)(2.0 * ab - 1.0), (float)(3.0 * ab - 2.0),
                                          (float)(4.0 * ab - 2.0), (float)(5.0 * ab - 2.0));
                // the task's cost per block: a line issues ~kWtBase instructions plus ~kWtCand
                // per expected extra candidate (c3 is loaded where phi > 4 - 3/|b|, c4 where
                // phi > 5 - 3/|b|, phi uniform), plus the wide loop's fixed extra
                const double p3 = 1.0 - fmin(fmax(4.0 - 3.0 / ab, 0.0), 1.0);
                const double p4 = 1.0 - fmin(fmax(5.0 - 3.0 / ab, 0.0), 1.0);
                sWt[lane] = SKEI_FWD_WCOST
                                ? (int)(16.0 * (kWtBase + kWtCand * (p3 + p4) + (4.0 * ab - 1.0 < 2.0 ? kWtWide : 0.0)) /
                                        kWtBase + 0.5)
                                : 1;
            }
        }
        for (int tau = threadIdx.x; tau < kWarps * kMaxT; tau += kThreads) s_cost[tau] = 0;
        __syncthreads();
        const int kcnt = sCount;
        const int ntask = kcnt * a.chunks;
        // per (angle, block): the block's first-line position of bin 0, A = P0 + lb Pl, split
        // into (int base, fp32 frac) in fp64, and the exact range [jlo, jhi] of bins whose
        // candidates can fall inside the image for some line of the block
        SKEI_DCHECK(kcnt * nbu <= K * a.nblk && kcnt * a.chunks <= kWarps * kMaxT, "forward unit tables");
        for (int e = threadIdx.x; e < kcnt * nbu; e += kThreads) {
            const int k = e / nbu, i = e - k * nbu;
            const double Pl = sPl[k], Pj = sPj[k];
            const double A = sP0[k] + (double)((ulo + i) * R) * Pl;
            const double fA = floor(A);
            const double sec = 1.0 / (double)sAbsB[k];
            const double lmin = fmin(0.0, (R - 1) * Pl), lmax = fmax(0.0, (R - 1) * Pl);
            // bin j touches the block iff A + j Pj + [lmin, lmax] meets (-sec - 1, n - 1 + sec + 1)
            const double u0 = (-sec - 1.0 - A - lmax) / Pj, u1 = (n - 1 + sec + 1.0 - A - lmin) / Pj;
            const double jl = fmax(-1.0, floor(fmin(u0, u1))), jh = fmin((double)n_det, ceil(fmax(u0, u1)));
            int4 ent;
            ent.x = (int)fA;
            ent.y = __float_as_int((float)(A - fA));
            ent.z = (int)jl;
            ent.w = (int)jh;
            btab[e] = ent;
            // the chunks c with 64 c <= jh and 64 c + 63 >= jl touch this block
            const int clo = ent.z <= 0 ? 0 : ent.z / kChunk;
            const int chi = ent.w < 0 ? -1 : min(a.chunks - 1, ent.w / kChunk);
            const int wt = sWt[k];
            for (int c = clo; c <= chi; ++c) atomicAdd(&s_cost[k * a.chunks + c], wt);
        }

        // ---- 3. tasks: (angle k, 64-bin chunk) pairs.  A warp runs a task's whole line loop
        // on every block its chunk touches, so a task costs the number of such blocks
        // (counted while the block table is built); chunks that touch no block are dropped.
        // The others are ranked by cost (descending, ties by index) and dealt to the warps
        // in snake order (rank r -> round r / kWarps, warp r mod kWarps, reversed on odd
        // rounds), which balances the warps to within about one task.  Per task: angle slot
        // k (< 0: none), first bin of the chunk c0, and (c0 + 31) Pj + min(Pj, 0) split into
        // (int, fp32 fraction) in fp64; a lane adds its (2 lane - 31) Pj in fp32 (|.| < 44),
        // giving the position of the lower of its two bins (the one nearer pixel 0).
        __syncthreads();  // block table and task costs complete
        for (int tau = threadIdx.x; tau < kWarps * kMaxT; tau += kThreads)
            s_task[tau] = make_int4(-1, 0, 0, 0);
        if (threadIdx.x < 3) s_fq[threadIdx.x] = 0;
        if (threadIdx.x == 3) s_nfl = 0;
        if (threadIdx.x >= 32 && threadIdx.x < 32 + kMaxFloat) s_fseq[threadIdx.x - 32] = -1;
        __syncthreads();
        for (int tau = threadIdx.x; tau < ntask; tau += kThreads) {
            const int cst = s_cost[tau];
            if (cst == 0) continue;
            int r = 0;
            for (int o = 0; o < ntask; ++o) {
                const int co = s_cost[o];
                r += (co > cst) || (co == cst && o < tau);
            }
            int4 td;
            td.x = tau / a.chunks;
            td.y = (tau - td.x * a.chunks) * kChunk;
            const double J = (double)(td.y + 31) * sPj[td.x] + fmin(sPj[td.x], 0.0);
            const double fJ = floor(J);
            td.z = (int)fJ;
            td.w = __float_as_int((float)(J - fJ));
            if (r < nfloat) {  // the costliest tasks float (they touch the most blocks)
                s_float[r] = td;
                atomicMax(&s_nfl, r + 1);
                continue;
            }
            r -= nfloat;
            const int round = r / kWarps, wi = r - round * kWarps;
            const int w = (round & 1) ? kWarps - 1 - wi : wi;
            s_task[w + kWarps * round] = td;
        }
        __syncthreads();  // block table and task table complete
        const int nfl = kFloat ? s_nfl : 0;
#ifdef SKEI_FWD_STATS
        st_pro += clock64() - tp0;
#endif
        // acc[t][0..BB): the lower bin of the lane's pair (the one nearer pixel 0 of the
        // line), acc[t][BB..2BB): the upper one
        float acc[kMaxT][2 * BB];
#pragma unroll
        for (int t = 0; t < kMaxT; ++t)
#pragma unroll
            for (int b = 0; b < 2 * BB; ++b) acc[t][b] = 0.f;

        for (int i = 0; i < nbu; ++i) {
            const int g = gbase + i;
            const int cb = g % nbuf;
            const unsigned cur_b = smem_b + (unsigned)(cb * stage_f * sizeof(float));
#ifdef SKEI_FWD_STATS
            const long long tw0 = clock64();
#endif
            mbar_wait(&full[cb], (unsigned)((g / nbuf) & 1));
#ifdef SKEI_FWD_STATS
            st_wait += clock64() - tw0;
#endif
            // one task's line loop over the staged block: lo / hi = the block's sums of the
            // lane's lower / upper bin (shared by the warps' own tasks and the floating ones)
            auto task_block = [&](const int4 td, const int4 ent, const int k, float (&lo)[BB],
                                  float (&hi)[BB]) {
                int base = ent.x + td.z;
                float frac = __int_as_float(ent.y) + __int_as_float(td.w);
                if (frac >= 1.f) {
                    frac -= 1.f;
                    base += 1;
                }
                const float4 ang = sAngT[k][0];  // |beta|, 1/|beta|, Pl, min(Pj, 0)
                const float4 off = sAngT[k][1];  // hat offsets 2|b| - 1, 3|b| - 2, 4|b| - 2, 5|b| - 2
                const float ab = ang.x, plf = ang.z;
                // 1 - (d3 - 1) = |b| phi + (3 - 4|b|) and likewise for d4: the upper bin's
                // weights of c3 / c4 in one FFMA (their loads are predicated on the same value)
                const float k3 = 1.f - off.z, k4 = 1.f - off.w;
                // a candidate window of 5 pixels can be needed only if 4|beta| - 1 < 2
                const bool wide = off.z < 1.f;
                // + (2 lane - 31) Pj (|.| < 44, fp32): the lane's lower bin within the chunk
                const float fs = fmaf(lane2f, sAngT[k][2].x, frac - ang.y);
                // candidate_0 + kCand = base + 6 + floor(e); floor(e) is taken as an exact
                // fp32 integer and moved to the integer unit by the 1.5 * 2^23 bias (|e| < 2^22)
                const int base6 = base + 1 + kCand - 0x4B400000;
                float d[LB];
#pragma unroll
                for (int b = 0; b < LB; ++b) d[b] = sgn[b] * plf;
                const unsigned pbase = cur_b + lofs0;  // bits 0..6 = line lane'
                float e = fmaf(lf0, plf, fs);
#pragma unroll
                for (int b = 0; b < BB; ++b) lo[b] = hi[b] = 0.f;
                // the line loop, compiled twice: with and without the fifth candidate (wide is
                // warp-uniform — a property of the task's angle — so the branch between the two
                // never diverges, and the ~92% of angles with 4|b| - 1 >= 2 issue no c4 code)
                auto run_lines = [&](auto wide_tag) {
                constexpr bool kWide = decltype(wide_tag)::value;
                // one line: e = a*_lo - 1/|beta| relative to base (a*_lo: the line position
                // that projects onto the lower bin's centre, the upper one's is a*_lo + 1/|b|).
                // Candidates c_k = floor(e) + 1 + k, k = 0..4, lie at detector offsets
                // delta_k = |b| (k + 1 - phi) - 1 from the lower bin (phi = e - floor(e)), so
                // their hat weights are, for the lower bin,
                //   w0 = |b| (1 - phi), w1 = 1 - |d1|, w2 = max(0, -(d2 - 1))
                // and for the upper bin (hat(delta - 1))
                //   w1' = max(0, d1), w2' = 1 - |d2 - 1|, w3' = max(0, 1 - (d3 - 1)),
                //   w4' = max(0, 1 - (d4 - 1)),
                // every other (candidate, bin) weight being 0 for |beta| in [1/sqrt 2, 1].
                // The 5 candidate pixels are loaded kAhead lines ahead of their use; c3 only
                // where w3' > 0, c4 only where w4' > 0 (possible only if 4|b| - 1 < 2).
                constexpr int D = kAhead < R ? kAhead : R - 1;  // lines in flight ahead of use
                float v[D + 1][kCand][BB], ph[D + 1];
                auto load_line = [&](int st, float (&vv)[kCand][BB], float &phs) {
                    const int gc = st ^ (st >> 1);
                    const float fl2 = floorf(e);
                    const float phi = e - fl2;
                    phs = phi;
                    // candidate_0 + 5 clamped to [0, n + 5] in one unsigned min (lanes whose
                    // pair misses the line land in the zero pad columns)
                    const unsigned cu =
                        min((unsigned)(base6 + __float_as_int(fl2 + 12582912.f)), cmax);
                    const unsigned pa = (pbase ^ (unsigned)(gc * BB * sizeof(float))) +
                                        cu * (unsigned)(kColF * sizeof(float));
                    SKEI_DCHECK(pa >= cur_b && pa + (kCand - 1) * kColF * sizeof(float) + BB * sizeof(float) <=
                                    cur_b + (unsigned)(stage_f * sizeof(float)),
                                "forward candidate address");
                    lds_px<BB>(pa, vv[0]);
                    lds_px<BB>(pa + kColF * sizeof(float), vv[1]);
                    lds_px<BB>(pa + 2 * kColF * sizeof(float), vv[2]);
#if SKEI_FWD_C3_ALWAYS
                    lds_px<BB>(pa + 3 * kColF * sizeof(float), vv[3]);
#else
                    if (fmaf(ab, phi, k3) > 0.f) lds_px<BB>(pa + 3 * kColF * sizeof(float), vv[3]);
#endif
                    if constexpr (kWide) {
                        if (fmaf(ab, phi, k4) > 0.f)
                            lds_px<BB>(pa + 4 * kColF * sizeof(float), vv[4]);
                    }
                };
                auto use_line = [&](const float (&vv)[kCand][BB], float phi) {
                    const float w0 = fmaf(-ab, phi, ab);
                    const float d1 = fmaf(-ab, phi, off.x);
                    const float e2 = fmaf(-ab, phi, off.y);
                    const float w1 = 1.f - fabsf(d1), u1 = fmaxf(d1, 0.f);
                    const float w2 = fmaxf(-e2, 0.f), u2 = 1.f - fabsf(e2);
                    const float u3 = fmaxf(fmaf(ab, phi, k3), 0.f);
                    fma_px<BB>(lo, w0, vv[0]);
                    fma_px<BB>(lo, w1, vv[1]);
                    fma_px<BB>(hi, u1, vv[1]);
                    fma_px<BB>(lo, w2, vv[2]);
                    fma_px<BB>(hi, u2, vv[2]);
                    fma_px<BB>(hi, u3, vv[3]);
                    if constexpr (kWide) {
                        const float u4 = fmaxf(fmaf(ab, phi, k4), 0.f);
                        fma_px<BB>(hi, u4, vv[4]);
                    }
                };
                // e of line gray(sn) from that of line gray(sn - 1)
                auto advance = [&](int sn) {
                    const int gc = sn ^ (sn >> 1);
                    // the bit gray(sn) flips (lowest set bit of sn; folds when unrolled)
                    const int ib = (sn & 1) ? 0 : (sn & 2) ? 1 : (sn & 4) ? 2 : (sn & 8) ? 3 : 4;
                    if (ib >= 3) {  // re-anchor every 8 lines: e exact to one rounding
                        e = fmaf((float)(lane_r ^ gc), plf, fs);
                    } else {
                        e = ((gc >> ib) & 1) ? e + d[ib] : e - d[ib];
                    }
                };
                // c3 / c4 are not loaded where their weight is 0: keep their registers finite
#pragma unroll
                for (int q2 = 0; q2 <= D; ++q2)
#pragma unroll
                    for (int b = 0; b < BB; ++b) {
                        v[q2][3][b] = 0.f;
                        if constexpr (kWide) v[q2][4][b] = 0.f;
                    }
#pragma unroll
                for (int st = 0; st < D; ++st) {
                    if (st > 0) advance(st);
                    load_line(st, v[st], ph[st]);
                }
#pragma unroll
                for (int st = 0; st < R; ++st) {
                    const int cur = st % (D + 1);
                    if (st + D < R) {
                        advance(st + D);
                        load_line(st + D, v[(st + D) % (D + 1)], ph[(st + D) % (D + 1)]);
                    }
                    use_line(v[cur], ph[cur]);
                }
                };
#if SKEI_FWD_LANE_SKIP
                // lanes whose bin pair no line of the block can see skip the line loop (their
                // sums stay 0): a quarter-warp of such lanes issues no shared-memory wavefronts
                const int jlane = td.y + 2 * lane;
                if (jlane + 1 < ent.z || jlane > ent.w) return;
#endif
#if SKEI_FWD_WIDE_SPLIT
                if (wide)
                    run_lines(std::true_type{});
                else
                    run_lines(std::false_type{});
#else
                run_lines(std::true_type{});
#endif
            };
            int4 tdn = s_task[warp];  // the next task's descriptor, loaded one task ahead
            // the task loop is unrolled (acc[t] register-indexed) only while the code stays
            // small; otherwise each task's block sum is added to acc[t] by predicated adds
            constexpr bool kUnrollT = R * kMaxT <= 64;
#pragma unroll(kUnrollT ? kMaxT : 1)
            for (int t = 0; t < kMaxT; ++t) {
                const int4 td = tdn;  // warp-uniform (broadcast)
                const int k = td.x;
                if (k < 0) break;
                const int4 ent = btab[k * nbu + i];
                if (t + 1 < kMaxT) tdn = s_task[warp + kWarps * (t + 1)];
                if (td.y > ent.w || td.y + kChunk - 1 < ent.z) continue;  // chunk misses the block
#ifdef SKEI_FWD_STATS
                const long long tt0 = clock64();
                ++st_active;
                st_lanes += max(0, min(td.y + kChunk - 1, min(ent.w, n_det - 1)) - max(td.y, ent.z) + 1);
#endif
                float lo[BB], hi[BB];
                task_block(td, ent, k, lo, hi);
#ifdef SKEI_FWD_STATS
#pragma unroll
                for (int tt = 0; tt < kMaxT; ++tt)
                    if (tt == t) {
                        st_tc[tt] += clock64() - tt0;
                        ++st_tn[tt];
                    }
#endif
                if constexpr (kUnrollT) {
#pragma unroll
                    for (int b = 0; b < BB; ++b) {
                        acc[t][b] += lo[b];
                        acc[t][BB + b] += hi[b];
                    }
                } else {
#pragma unroll
                    for (int tt = 0; tt < kMaxT; ++tt)
                        if (tt == t) {
#pragma unroll
                            for (int b = 0; b < BB; ++b) {
                                acc[tt][b] += lo[b];
                                acc[tt][BB + b] += hi[b];
                            }
                        }
                }
            }
            // floating tasks: a warp done with its own tasks of this block takes the block's
            // floating tasks from a shared queue until none is left (each warp's last grab
            // fails, so a block adds nfl + kWarps to its buffer's counter).  The block sums are
            // added to the task's shared-memory sums in block order (s_fseq; a chunk's blocks
            // are consecutive, and block i's queue opens only after block i - 1's is empty, so
            // the sum a warp waits for is already being computed): the result is bitwise the
            // one a warp-owned task gives.
            if constexpr (kFloat) {
                if (nfl > 0) {
                    const int fbase = (nfl + kWarps) * (i / nbuf);
                    for (;;) {
                        int f = 0;
                        if (lane == 0) f = atomicAdd(&s_fq[cb], 1) - fbase;
                        f = __shfl_sync(0xffffffffu, f, 0);
                        if (f >= nfl) break;
                        const int4 td = s_float[f];
                        const int k = td.x;
                        const int4 ent = btab[k * nbu + i];
                        if (td.y > ent.w || td.y + kChunk - 1 < ent.z) continue;
#ifdef SKEI_FWD_STATS
                        ++st_active;
                        ++st_fl;
#endif
                        float lo[BB], hi[BB];
                        task_block(td, ent, k, lo, hi);
                        bool first = i == 0;
                        if (!first) {
                            const int4 pe = btab[k * nbu + i - 1];
                            first = td.y > pe.w || td.y + kChunk - 1 < pe.z;
                        }
                        float4 *fa = reinterpret_cast<float4 *>(facc) + (size_t)f * 64 + lane;
                        float4 alo = make_float4(0.f, 0.f, 0.f, 0.f), ahi = alo;
                        if (!first) {
                            if (lane == 0) {
                                while (*reinterpret_cast<volatile int *>(&s_fseq[f]) != i) {
                                }
                                __threadfence_block();
                            }
                            __syncwarp();
                            alo = fa[0];
                            ahi = fa[32];
                        }
                        alo.x += lo[0], alo.y += lo[1], alo.z += lo[2], alo.w += lo[3];
                        ahi.x += hi[0], ahi.y += hi[1], ahi.z += hi[2], ahi.w += hi[3];
                        fa[0] = alo;
                        fa[32] = ahi;
                        __syncwarp();
                        if (lane == 0) {
                            __threadfence_block();
                            *reinterpret_cast<volatile int *>(&s_fseq[f]) = i + 1;
                        }
                    }
                }
            }
            // release the buffer; the last warp out refills it with block g + nbuf
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();  // this warp's reads of the buffer are complete
                const int old = atomicAdd(&done[cb], 1);
                if (old == kWarps * (g / nbuf + 1) - 1 && g + nbuf < G) {
                    fence_proxy_async();  // generic-proxy reads -> async-proxy writes
                    issue(g + nbuf, cb);
                }
            }
        }

#if defined(SKEI_FWD_STATS) && defined(SKEI_FWD_STATS_TASKS)
        if (lane == 0 && (blockIdx.x % SKEI_FWD_STATS_EVERY) == 0) {
#pragma unroll
            for (int t = 0; t < kMaxT; ++t) {
                const int4 td = s_task[warp + kWarps * t];
                if (td.x < 0) continue;
                printf("FWDTASK cta %d warp %d slot %d ab1e4 %d c0 %d cost %d blocks %lld cycles %lld cls %d\n",
                       blockIdx.x, warp, t, (int)(sAngT[td.x][0].x * 10000.f), td.y,
                       s_cost[td.x * a.chunks + td.y / kChunk], st_tn[t], st_tc[t], d.cls);
                st_tn[t] = st_tc[t] = 0;
            }
        }
#endif
#ifdef SKEI_FWD_STATS
        const long long te0 = clock64();
#endif
        // ---- 4. unit epilogue.  A whole unit is complete in this CTA's registers: each lane
        // writes its (angle, bin) sums to p and, for the MC job, r = p - y_S and sum r^2.  A
        // split unit's piece goes to this CTA's L2 slot; the last piece to arrive (counter)
        // adds the pieces in CTA order and finishes the unit.
        gbase += nbu;
        const long img_stride = (long)a.m * n_det;
        const bool mc = job.y != nullptr;
        float racc[BB];
#pragma unroll
        for (int b = 0; b < BB; ++b) racc[b] = 0.f;
        // slot b's projection image (fused: job b's output for image b0)
        auto slot_p = [&](int b) -> float * {
            return FUSED ? a.job[b].p + (long)b0 * img_stride : job.p + (long)(b0 + b) * img_stride;
        };
        auto finish_bin = [&](int slot, int j, const float (&sv)[BB]) {
            const long pj = (long)slot * n_det + j;
#pragma unroll
            for (int b = 0; b < BB; ++b) slot_p(b)[pj] = sv[b];
            if (mc) {
                const long yj = (long)(job.y_sketched ? slot : idx[slot]) * n_det + j;
                const long ys = (long)(job.y_sketched ? a.m : n_full) * n_det;
#pragma unroll
                for (int b = 0; b < (FUSED ? 1 : BB); ++b) {
                    const float dr = sv[b] - __ldg(job.y + (long)(b0 + b) * ys + yj);
                    if (job.r) job.r[(long)(b0 + b) * img_stride + pj] = dr;
                    racc[b] = fmaf(dr, dr, racc[b]);
                }
            }
        };
        bool finish = full_unit;
        // chunks that touch no block of the unit (dropped tasks) sum to zero
        float zero[BB];
#pragma unroll
        for (int b = 0; b < BB; ++b) zero[b] = 0.f;
        // the lane's pair (j0, j0 + 1) of task t: acc holds (lower, upper); the lower bin is
        // j0 unless Pj < 0
        auto pair_sums = [&](int t, float (&s0)[BB], float (&s1)[BB]) {
            const bool neg = sAngT[s_task[warp + kWarps * t].x][0].w < 0.f;
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                s0[b] = neg ? acc[t][BB + b] : acc[t][b];
                s1[b] = neg ? acc[t][b] : acc[t][BB + b];
            }
        };
        // the same for floating task f (angle slot k): its sums are in shared memory
        auto float_sums = [&](int f, int k, float (&s0)[BB], float (&s1)[BB]) {
            const bool neg = sAngT[k][0].w < 0.f;
            const float *fa = facc + ((size_t)f * 64 + lane) * 4;
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                const float l = fa[b < 4 ? b : 0], h = fa[128 + (b < 4 ? b : 0)];
                s0[b] = neg ? h : l;
                s1[b] = neg ? l : h;
            }
        };
        if (full_unit) {
#pragma unroll
            for (int t = 0; t < kMaxT; ++t) {
                const int4 td = s_task[warp + kWarps * t];
                if (td.x < 0) break;
                const int j = td.y + 2 * lane;
                float s0[BB], s1[BB];
                pair_sums(t, s0, s1);
                if (j < n_det) finish_bin(sSlot[td.x], j, s0);
                if (j + 1 < n_det) finish_bin(sSlot[td.x], j + 1, s1);
            }
            for (int tau = warp; tau < ntask; tau += kWarps) {
                if (s_cost[tau] != 0) continue;
                const int k = tau / a.chunks, j = (tau - k * a.chunks) * kChunk + 2 * lane;
                if (j < n_det) finish_bin(sSlot[k], j, zero);
                if (j + 1 < n_det) finish_bin(sSlot[k], j + 1, zero);
            }
            if constexpr (kFloat) {
                if (nfl > 0) {
                    __syncthreads();  // every floating task's sums complete
                    if (warp < nfl) {
                        const int4 td = s_float[warp];
                        const int j = td.y + 2 * lane;
                        float s0[BB], s1[BB];
                        float_sums(warp, td.x, s0, s1);
                        if (j < n_det) finish_bin(sSlot[td.x], j, s0);
                        if (j + 1 < n_det) finish_bin(sSlot[td.x], j + 1, s1);
                    }
                }
            }
        } else {
            float *mine = pieces + ((long)cid * 2 + (u == u_first ? 0 : 1)) * part_f;
#pragma unroll
            for (int t = 0; t < kMaxT; ++t) {
                const int4 td = s_task[warp + kWarps * t];
                if (td.x < 0) break;
                const int j = td.y + 2 * lane;
                float s0[BB], s1[BB];
                pair_sums(t, s0, s1);
                if (j < n_det) stg_vec<BB>(mine + ((long)td.x * n_det + j) * BB, s0);
                if (j + 1 < n_det) stg_vec<BB>(mine + ((long)td.x * n_det + j + 1) * BB, s1);
            }
            for (int tau = warp; tau < ntask; tau += kWarps) {
                if (s_cost[tau] != 0) continue;
                const int k = tau / a.chunks, j = (tau - k * a.chunks) * kChunk + 2 * lane;
                if (j < n_det) stg_vec<BB>(mine + ((long)k * n_det + j) * BB, zero);
                if (j + 1 < n_det) stg_vec<BB>(mine + ((long)k * n_det + j + 1) * BB, zero);
            }
            if constexpr (kFloat) {
                if (nfl > 0) {
                    __syncthreads();  // every floating task's sums complete
                    if (warp < nfl) {
                        const int4 td = s_float[warp];
                        const int j = td.y + 2 * lane;
                        float s0[BB], s1[BB];
                        float_sums(warp, td.x, s0, s1);
                        if (j < n_det) stg_vec<BB>(mine + ((long)td.x * n_det + j) * BB, s0);
                        if (j + 1 < n_det) stg_vec<BB>(mine + ((long)td.x * n_det + j + 1) * BB, s1);
                    }
                }
            }
            __threadfence();
            __syncthreads();  // the whole piece written (and fenced)
            if (threadIdx.x == 0) {
                // the pieces: non-empty CTA ranges c0 .. c1, slot 0 if u is the CTA's first unit
                // (the last piece to arrive finishes the unit after this CTA's block stream,
                // step 4b, where the projector's registers are free for batched loads)
                const int c0 = cta_of((long)u * nbc), c1 = cta_of((long)u * nbc + nbc - 1);
                const int di = u == u_first ? 0 : 1;
                int npc = 0;
                for (int c = c0; c <= c1; ++c) {
                    const long ws = wstart(c);
                    if (wstart(c + 1) == ws) continue;
                    SKEI_DCHECK(npc < kMaxPieces, "forward pieces per split unit");
                    s_dpiece[di][npc++] = c * 2 + (u == (int)(ws / nbc) ? 0 : 1);
                }
                const bool last = atomicAdd(a.queue + c0, 1u) == (unsigned)(npc - 1);
                if (last) {
                    a.queue[c0] = 0u;  // ready for the next launch
                    s_defer[di] = u;
                    s_dnpc[di] = npc;
                }
            }
        }
        if (mc && finish) {  // per-unit partial of each image of the group
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                float v = racc[b];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) s_red[warp][b] = v;
            }
        }
        __syncthreads();  // s_red complete; s_task / sSlot free for the next unit
        if (mc && finish && threadIdx.x < (FUSED ? 1 : BB)) {
            float v = 0.f;
            for (int w = 0; w < kWarps; ++w) v += s_red[w][threadIdx.x];
            SKEI_DCHECK(u - U.uoff[d.q] < a.mc_slots, "forward MC partial slot");
            a.mc_part[(long)(b0 + threadIdx.x) * a.mc_slots + (u - U.uoff[d.q])] = v;
        }
#ifdef SKEI_FWD_STATS
        st_epi += clock64() - te0;
#endif
    }

    // ---- 4b. split units whose last piece this CTA produced: out = the pieces summed in CTA
    // order (p; for the MC job r = p - y_S and the unit's partial of sum r^2).  kFin outputs
    // per thread and round, their piece and y_S loads in flight together.
#ifdef SKEI_FWD_STATS
    const long long tf0 = clock64();
#endif
    for (int di = 0; di < 2; ++di) {
        const int u = s_defer[di];
        if (u < 0) continue;
        const UnitId d = decode_unit(U, nq, K, u);
        const FwdJob job = d.job ? a.job[1] : a.job[0];
        const int b0 = FUSED ? d.q : d.q * BB;
        const int32_t *idx = a.idx + (a.idx_stride ? (long)b0 * a.idx_stride : 0);
        const int ncls = d.cls == 0 ? s_nrow[d.q] : a.m - s_nrow[d.q];
        const int ngc = (ncls + K - 1) / K;
        (void)ngc;
        __syncthreads();  // sSlot free
        if (warp == 0) {  // the unit's angle slots, as in step 2
            int seen = 0;
            for (int base = 0; base < a.m; base += 32) {
                const int k = base + lane;
                bool in = false;
                if (k < a.m) {
                    const int i = idx[k];
                    const bool row_class = is_row(i);
                    in = (d.cls == 0) ? row_class : !row_class;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pre = seen + __popc(bal & ((1u << lane) - 1u));
#if SKEI_FWD_STRIDED
                if (in && pre % ngc == d.grp) sSlot[pre / ngc] = k;
#else
                if (in && pre >= d.grp * K && pre < d.grp * K + K) sSlot[pre - d.grp * K] = k;
#endif
                seen += __popc(bal);
            }
#if SKEI_FWD_STRIDED
            if (lane == 0) sCount = max(0, (seen - d.grp + ngc - 1) / ngc);
#else
            if (lane == 0) sCount = max(0, min(K, seen - d.grp * K));
#endif
        }
        __syncthreads();
        const int total = sCount * n_det, npc = s_dnpc[di];
        const long img_stride = (long)a.m * n_det;
        const long ys = (long)(job.y_sketched ? a.m : n_full) * n_det;
        const bool mc = job.y != nullptr;
        const int *pc = s_dpiece[di];
        float racc[BB];
#pragma unroll
        for (int b = 0; b < BB; ++b) racc[b] = 0.f;
        constexpr int kFin = 4;
        for (int o0 = threadIdx.x; o0 < total; o0 += kThreads * kFin) {
            float sv[kFin][BB], yv[kFin][BB];
#pragma unroll
            for (int q = 0; q < kFin; ++q) {
                const int o2 = o0 + q * kThreads;
                if (o2 < total) {
                    const int k = o2 / n_det, j = o2 - k * n_det;
                    ldcg_vec<BB>(pieces + (long)pc[0] * part_f + (long)o2 * BB, sv[q]);
                    if (mc) {
                        const int slot = sSlot[k];
                        const long yj = (long)(job.y_sketched ? slot : idx[slot]) * n_det + j;
#pragma unroll
                        for (int b = 0; b < BB; ++b) yv[q][b] = __ldg(job.y + (long)(b0 + b) * ys + yj);
                    }
                }
            }
            for (int c = 1; c < npc; ++c) {  // the pieces in CTA order
                float v[kFin][BB];
#pragma unroll
                for (int q = 0; q < kFin; ++q)
                    if (o0 + q * kThreads < total)
                        ldcg_vec<BB>(pieces + (long)pc[c] * part_f + (long)(o0 + q * kThreads) * BB, v[q]);
#pragma unroll
                for (int q = 0; q < kFin; ++q)
#pragma unroll
                    for (int b = 0; b < BB; ++b) sv[q][b] += v[q][b];
            }
#pragma unroll
            for (int q = 0; q < kFin; ++q) {
                const int o2 = o0 + q * kThreads;
                if (o2 >= total) continue;
                const int k = o2 / n_det, j = o2 - k * n_det;
                const long pj = (long)sSlot[k] * n_det + j;
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    (FUSED ? a.job[b].p + (long)b0 * img_stride : job.p + (long)(b0 + b) * img_stride)[pj] = sv[q][b];
                if (mc) {
#pragma unroll
                    for (int b = 0; b < (FUSED ? 1 : BB); ++b) {
                        const float dr = sv[q][b] - yv[q][b];
                        if (job.r) job.r[(long)(b0 + b) * img_stride + pj] = dr;
                        racc[b] = fmaf(dr, dr, racc[b]);
                    }
                }
            }
        }
        if (mc) {  // the unit's partial of each image of the group
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                float v = racc[b];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) s_red[warp][b] = v;
            }
            __syncthreads();
            if (threadIdx.x < (FUSED ? 1 : BB)) {
                float v = 0.f;
                for (int w = 0; w < kWarps; ++w) v += s_red[w][threadIdx.x];
                SKEI_DCHECK(u - U.uoff[d.q] < a.mc_slots, "forward MC partial slot");
            a.mc_part[(long)(b0 + threadIdx.x) * a.mc_slots + (u - U.uoff[d.q])] = v;
            }
        }
    }
#ifdef SKEI_FWD_STATS
    const long long st_fin = clock64() - tf0;
#endif

#ifdef SKEI_FWD_STATS
    if (lane == 0 && (blockIdx.x % SKEI_FWD_STATS_EVERY) == 0)
        printf("FWDSTAT cta %d warp %d units %d G %d wait %lld pro %lld epi %lld total %lld active %lld "
               "lanes %lld esync %lld fin %lld\n", blockIdx.x, warp, u_last - u_first + 1, G, st_wait,
               st_pro, st_epi, clock64() - st_t0, st_active, st_lanes, st_fl, st_fin);
#endif
    // ---- 5. MC residual final: the last CTA sums each image's (unit, rank) partials in order
    if (!a.job[0].y) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.mc_ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int b = warp; b < a.B; b += kWarps) {
        const int q = FUSED ? b : b / BB;
        const int ns = U.uoff[q + 1] - U.uoff[q];
        double sum = 0.0;
        for (int i = lane; i < ns; i += 32) sum += (double)__ldcg(a.mc_part + (long)b * a.mc_slots + i);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        if (lane == 0) a.mc_out[b] = (float)sum;
    }
    if (threadIdx.x == 0) *a.mc_ctr = 0u;  // ready for the next launch
}

template <int BB, bool FUSED = false>
cudaError_t launch_bb(FwdArgs a, int num_sms, cudaStream_t s) {
    constexpr int R = kColF / BB;
    a.K = (kWarps * max_tasks<BB>()) / a.chunks;
    if (a.K > kKMax) a.K = kKMax;
    if (a.K < 1) return cudaErrorInvalidValue;  // n_det > kWarps * kMaxT * kChunk
#ifdef SKEI_FWD_KCAP_ENV
    if (const char *kc = std::getenv("SKEI_FWD_KCAP")) {
        const int cap = std::atoi(kc);
        if (cap >= 1 && cap < a.K) a.K = cap;
    }
#endif
    a.nblk = (a.g.n + R - 1) / R;
    a.nq = a.fused ? a.B : a.B / BB;
    if (a.nq > kMaxQ) return cudaErrorInvalidValue;
    // Small problems (fewer than kSmallBlocks line blocks per CTA at the largest K): units of
    // at most kSmallK angles, so the work spreads over angles as well as line blocks — a
    // CTA's per-unit prologue and its split-unit piece shrink with K, and a unit is cut into
    // fewer pieces.  Measured (round 2, fifth session): cfg2 forward 60.6 -> 50.0 us (K 10 ->
    // 3; K = 2: 51.3, K = 1: 63.8), cfg1 41.1 -> 36.1 us; cfg5 (22 blocks per CTA) gets slower
    // with any smaller K (249.6 us at K = 5, 265.8 at 3) and keeps the largest.
    {
        const long units = ((long)a.njobs * a.nq * a.m + a.K - 1) / a.K;
        if (units * a.nblk < (long)kSmallBlocks * num_sms && a.K > kSmallK) a.K = kSmallK;
    }
    const size_t stage_b = sizeof(float) * (size_t)(a.g.n + kPadL + kPadR) * kColF;
    const size_t tab_b = sizeof(int4) * (size_t)a.K * a.nblk;  // block table (any S)
    // dynamic shared memory budget: 227 KB per CTA less the static tables.  The function
    // attributes are set once per device (the launch path stays free of driver queries: it
    // runs every pass, also on the e2e host path)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    static int limit_of[kMaxDevices];  // 0: not yet set up on that device
    static std::mutex mu;
    int limit_i;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (limit_of[dev] == 0) {
            cudaFuncAttributes fa;
            e = cudaFuncGetAttributes(&fa, k_radon_fwd<BB, FUSED>);
            if (e != cudaSuccess) return e;
            const int lim = 227 * 1024 - (int)fa.sharedSizeBytes;
            e = cudaFuncSetAttribute(k_radon_fwd<BB, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
            if (e != cudaSuccess) return e;
            // persistent grid: one CTA per SM (the kernel needs one SM's registers and shared
            // memory; the split-unit scratch, the piece counters and kMaxPieces assume grid <=
            // num_sms <= 256)
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_radon_fwd<BB, FUSED>, kThreads, lim);
            if (e != cudaSuccess) return e;
            if (per_sm < 1) return cudaErrorInvalidConfiguration;
            limit_of[dev] = lim;
        }
        limit_i = limit_of[dev];
    }
    const size_t limit = (size_t)limit_i;
    a.nbuf = 3 * stage_b + tab_b <= limit ? 3 : (2 * stage_b + tab_b <= limit ? 2 : 1);
    size_t smem = a.nbuf * stage_b + tab_b + 128;  // + alignment slack
    if (smem > limit) return cudaErrorInvalidValue;
    // floating tasks (groups of 4): as many as the shared memory left over holds
    a.nfloat = 0;
    if (BB == 4 && !FUSED && kMaxFloat > 0) {
        const size_t room = (limit - smem) / kFloatBytes;
        a.nfloat = room < (size_t)kMaxFloat ? (int)room : kMaxFloat;
        smem += (size_t)a.nfloat * kFloatBytes;
    }
    if (num_sms > kMaxPieces || num_sms > kPassCounters - 2) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)num_sms, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    e = cudaLaunchKernelEx(&cfg, k_radon_fwd<BB, FUSED>, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// The driver's tensor-map encoder, through the runtime's entry-point query (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// the column-class tensor map of a row-packed copy (groups of 4; see FwdArgs::tm_col),
// from a small cache keyed by (copy, n, groups): the pass reuses its workspace every step
cudaError_t col_tensor_map(CUtensorMap *tm, const float *xr, int n, int nq) {
    struct Entry {
        const float *xr;
        int n, nq;
        CUtensorMap tm;
    };
    constexpr int kCache = 16;
    static Entry cache[kCache];
    static int next = 0;
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (int i = 0; i < kCache; ++i)
            if (cache[i].xr == xr && cache[i].n == n && cache[i].nq == nq) {
                *tm = cache[i].tm;
                return cudaSuccess;
            }
    }
    const auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    const int nblk = (n + 7) / 8;
    if (nblk > 256) return cudaErrorInvalidValue;  // box dimensions are <= 256
    cuuint64_t dims[4] = {4, (cuuint64_t)n, 8, (cuuint64_t)nq * nblk};
    cuuint64_t strides[3] = {128, 16, (cuuint64_t)n * 128};
    cuuint32_t box[4] = {4, 8, 8, (cuuint32_t)nblk};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(xr), dims, strides, box,
                           es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> lk(mu);
    cache[next] = Entry{xr, n, nq, *tm};
    next = (next + 1) % kCache;
    return cudaSuccess;
}

}  // namespace

size_t fwd_scratch_floats(const skei_plan *plan) {
    // two split-unit piece slots per CTA (grid = num_sms), each K * n_det * BB <=
    // kWarps * kMaxT * kChunk * BB floats
    return (size_t)2 * plan->num_sms * kWarps * kMaxTaskBB * kChunk;
}

size_t fwd_mc_slots(const skei_plan *plan, int B, int m, int idx_stride) {
    (void)B;
    (void)idx_stride;
    const int chunks = (plan->n_det + kChunk - 1) / kChunk;
    int K = (kWarps * kMinTasks) / chunks;  // the smallest K over the group sizes BB
    if (K > kKMax) K = kKMax;
    if (K < 1) K = 1;
    if (K > kSmallK) K = kSmallK;  // small problems run with K <= kSmallK (launch_bb)
#ifdef SKEI_FWD_KCAP_ENV
    K = 1;
#endif
    return (size_t)((m + K - 1) / K + 2);  // units per image group
}

cudaError_t launch_radon_fwd(const skei_plan *plan, const FwdJob *jobs, int njobs, int B,
                             const int32_t *idx, int m, int idx_stride, const FwdScratch &scr,
                             cudaStream_t s, const FwdMc *mc, bool fused) {
    if (fused && njobs != 2) return cudaErrorInvalidValue;
    FwdArgs a = {};
    a.fused = fused ? 1 : 0;
    a.queue = scr.queue;
    a.scratch = scr.part;
    a.mc_part = mc ? mc->part : nullptr;
    a.mc_slots = (int)fwd_mc_slots(plan, B, m, idx_stride);
    a.mc_ctr = mc ? mc->ctr : nullptr;
    a.mc_out = mc ? mc->out : nullptr;
    a.job[0] = jobs[0];
    a.job[1] = njobs > 1 ? jobs[1] : jobs[0];
    a.njobs = fused ? 1 : njobs;  // fused: one unit stream, the jobs are the groups' slots
    a.idx = idx;
    a.m = m;
    a.idx_stride = idx_stride;
    a.B = B;
    a.g = geom_of(plan);
    a.chunks = (plan->n_det + kChunk - 1) / kChunk;
    // band: |4 i - n_full| pi / (4 n_full) <= acos(0.68) - pi / 4 keeps min(|cos|, |sin|) >= 0.68
    a.band = (SKEI_FWD_BAND && idx_stride == 0)
                 ? (int)floor((acos(0.68) - M_PI / 4) * 4.0 * plan->n_full / M_PI)
                 : 0;
    if (!mc) a.job[0].y = nullptr;
    // column class from the row-packed copy (jobs without a column-packed copy): groups of 4
    a.tm_col = 0;
    const int njob = fused ? 1 : njobs;
    const bool no_xc = !jobs[0].xc || (njob > 1 && !jobs[1].xc);
    if (no_xc) {
        if (fused || fwd_bb(B, idx_stride) != 4 || !jobs[0].xr) return cudaErrorInvalidValue;
        if (njob > 1 && (jobs[1].xc || !jobs[1].xr)) return cudaErrorInvalidValue;
        if (jobs[0].xc) return cudaErrorInvalidValue;
        for (int j = 0; j < njob; ++j) {
            const cudaError_t e = col_tensor_map(&a.tm[j], jobs[j].xr, plan->n, B / 4);
            if (e != cudaSuccess) return e;
        }
        if (njob == 1) a.tm[1] = a.tm[0];
        a.tm_col = 1;
    }
    if (fused) return launch_bb<2, true>(a, plan->num_sms, s);
    const int bb = fwd_bb(B, idx_stride);
    switch (bb) {
        case 4: return launch_bb<4>(a, plan->num_sms, s);
        case 2: return launch_bb<2>(a, plan->num_sms, s);
        default: return launch_bb<1>(a, plan->num_sms, s);
    }
}

}  // namespace skei
