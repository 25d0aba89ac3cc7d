// internal.h — private declarations of the skei CUDA library (sm_100a).
// Nothing here is part of the ABI (include/skei.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

// Device-side invariant checks of the checked build (nvcc -DSKEI_CHECKS, e.g.
// `python tools/build_variant.py ab/libskei_checked.so -DSKEI_CHECKS`, then SKEI_LIB=... for the
// tests): the sanitizer substitute on this pool, where compute-sanitizer is closed.  A failed
// check prints its site and traps (the launch then fails with an illegal-instruction error).
// Compiled out of the product build.
#ifdef SKEI_CHECKS
#define SKEI_DCHECK(cond, what)                                                              \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("SKEI_DCHECK failed: %s at %s:%d (block %d,%d thread %d)\n", what, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);            \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define SKEI_DCHECK(cond, what) \
    do {                        \
    } while (0)
#endif

#include "../../include/skei.h"

constexpr int kMaxFftPass = 8;

struct skei_plan {
    int device;
    int n, n_det, n_full, fft_len, log2_fft;
    int num_sms;
    double2 *d_trig;  // [n_full] (cos, sin) of theta_i = i*pi/n_full, fp64
    float *d_ramp;    // [fft_len] R[k] / P, fp32 (from an fp64 DFT)
    // FFT pass plan (ramp.cu): radix, sub-transform length Ns and twiddle-table offset per
    // pass; d_twp[off + r Ns + k] = exp(-2 pi i r k / (R Ns)), fp32 rounded from fp64
    int fft_npass, fft_radix[kMaxFftPass], fft_ns[kMaxFftPass], fft_twoff[kMaxFftPass];
    float2 *d_twp;
    double2 *d_rot;   // [360] (cos g, sin g) of g degrees, fp64, exact at multiples of 90
};

namespace skei {

// Kernel-facing geometry constants, passed by value.
struct Geom {
    int n, n_det, n_full;
    double h;   // (n-1)/2
    double hd;  // (n_det-1)/2
    const double2 *trig;
};

inline Geom geom_of(const skei_plan *p) {
    Geom g;
    g.n = p->n;
    g.n_det = p->n_det;
    g.n_full = p->n_full;
    g.h = (p->n - 1) * 0.5;
    g.hd = (p->n_det - 1) * 0.5;
    g.trig = p->d_trig;
    return g;
}

// ---- launchers (return cudaGetLastError()) ----
// Packed forward-projector input (rotate.cu): for image group g (BB images), class
// (rows / cols) and block of R = 32/BB lines, [n pixels][R lines][BB images] floats.
size_t pack_floats(const skei_plan *plan, int B, int bb);  // one packed copy (one class)
struct RotPackJob {
    const float *x;      // [B][n][n]
    float *out;          // plain output [B][n][n] or NULL
    const int32_t *g;    // rotation (device) or NULL = identity
    int g_stride;        // 0 shared, 1 per image
    float *xr, *xc;      // row- / col-packed outputs or NULL
    unsigned *zero;      // if set, block (0,0,0) zeroes zero[0..kPassCounters) (pass counters)
    const float *xm = nullptr;  // identity job only: pack (and write) ascale * (x - xm)
    float ascale = 1.f;
};
// Pass counters: [0] MC completion, [1] EI completion, [2..] the forward's stream-K split-unit
// piece counters (one per cluster, <= 256 SMs).
constexpr int kPassCounters = 2 + 256;
struct RotPackArgs {
    RotPackJob job[2];
    const double2 *rot;  // plan->d_rot
    int n, B, nblk, tiles_c;
    int pdl;             // launched programmatically behind k_draw: the rotation job waits
    int fuse;            // job-fused layout (bb = 1, 2 jobs): image b's x1 and x2 are the two
                         // slots of group b, blocks of 16 lines: [b][blk][pixel][line][job]
};
// fuse: the job-fused packed layout (see RotPackArgs), for a forward launch with fused jobs
cudaError_t launch_rotate_pack(const skei_plan *plan, const RotPackJob *jobs, int njobs, int B,
                               int bb, cudaStream_t s, bool pdl = false, bool fuse = false);
cudaError_t launch_rotate(const skei_plan *plan, const float *x, float *out, int B,
                          const int32_t *g, int g_stride, cudaStream_t s);
// out = T_g^T y (gather form of the rotation's transpose)
cudaError_t launch_rotate_adj(const skei_plan *plan, const float *y, float *out, int B,
                              const int32_t *g, int g_stride, cudaStream_t s);

// Forward projector on packed input; up to two jobs (e.g. A_S x1 and A_S x2) per launch.
// fused: the two jobs of each image share its sketch and are processed as the two slots of
// one group (the job-fused packed layout of launch_rotate_pack; jobs[0].xr / xc point to it).
// Job 0 may fuse the MC residual: y != NULL -> r = p - y_S (if r != NULL) and mc = sum r^2.
struct FwdJob {
    // row- / column-packed copies; xc == NULL (groups of 4 only): the column class is staged
    // from xr through a transposing tensor map (radon_fwd.cu, FwdArgs::tm_col)
    const float *xr, *xc;
    float *p;
    const float *y;  // full sinogram [B][n_full][n_det] or NULL (job 0 only)
    float *r;        // residual [B][m][n_det] or NULL
    int y_sketched = 0;  // y holds only the sketched rows, [B][m][n_det] (row k = angle idx[k])
};
struct FwdMc {
    float *part;    // [B][fwd_mc_slots] partial sums
    unsigned *ctr;  // completion counter, zero before the launch (self-resetting)
    float *out;     // mc [B]
};
// Forward scratch: work-queue counter (zero before the launch) and per-CTA partials.
struct FwdScratch {
    unsigned *queue;
    float *part;  // fwd_scratch_floats
};
size_t fwd_mc_slots(const skei_plan *plan, int B, int m, int idx_stride);
size_t fwd_scratch_floats(const skei_plan *plan);
cudaError_t launch_radon_fwd(const skei_plan *plan, const FwdJob *jobs, int njobs, int B,
                             const int32_t *idx, int m, int idx_stride, const FwdScratch &scr,
                             cudaStream_t s, const FwdMc *mc = nullptr, bool fused = false);

// Backprojection; up to two jobs sharing one angle list (FBP of q and gradient of r).
// Job 0 may fuse ei = sum (x2 - x_job0)^2 (identity network): partial sums per tile.
// Interleaved padded sinogram for the backprojector's bulk window copies: row (b, k) ->
// [b / 4][k][kAdjPad + j][b % 4], rows of n_det + 2 kAdjPad bins, the pads zero, so one
// angle's detector window of a tile is one contiguous, in-bounds 16-byte-aligned copy.
constexpr int kAdjPad = 48;
inline size_t adj_il_floats(const skei_plan *plan, int B, int m) {
    return (size_t)((B + 3) / 4) * m * (plan->n_det + 2 * kAdjPad) * 4;
}
// The job-fused pass (one image per group): q and r of image b interleaved as the two slots
// of one row, [b][k][kAdjPad + j][2], rows of even width (16-byte-aligned even windows)
inline int adj_fused_wp(const skei_plan *plan) { return (plan->n_det + 2 * kAdjPad + 1) & ~1; }
inline size_t adj_fused_floats(const skei_plan *plan, int B, int m) {
    return (size_t)B * m * adj_fused_wp(plan) * 2;
}
// pi: the same sinogram as p in the interleaved layout (or NULL: staged from p)
// base: if set, x = base + scale A^T p (same layout as x)
struct AdjJob {
    const float *p;
    float *x;
    float scale;
    const float *pi = nullptr;
    const float *base = nullptr;
};
struct AdjEi {
    const float *x2;  // [B][n][n]
    float *part;      // [B][adj_ei_part_floats / B]
    unsigned *ctr;    // completion counter, zero before the launch (self-resetting)
    float *out;       // ei [B]
};
size_t adj_ei_part_floats(const skei_plan *plan, int B);
// reduce-scatter epilogue: output row r of job j, image b is stored
// (P2P over NVLink / symmetric memory) into the receive buffer of the rank o that owns row r
// (bands as dist.batch_range(n, o, world): start(o) = o q + min(o, n mod world), q = n /
// world), at peer[o] + ((j B + b) bmax + r - start(o)) n + c; peer[o] already points at this
// rank's slot of rank o's buffer [world][2][B][bmax][n].  world 0: off.
constexpr int kMaxRsPeers = 8;
struct AdjRs {
    float *peer[kMaxRsPeers];
    int world = 0, bmax = 0;
};
// row0, rows: backproject only output rows [row0, row0 + rows) into [B][rows][n] outputs
// (rows < 0: whole images)
// fused: the two jobs are the slots of each image's group (job-fused pass): both jobs' pi
// point to the fused interleaved q / r rows (adj_fused_floats)
cudaError_t launch_radon_adj(const skei_plan *plan, const AdjJob *jobs, int njobs, int B,
                             const int32_t *idx, int m, int idx_stride, cudaStream_t s,
                             const AdjEi *ei = nullptr, int row0 = 0, int rows = -1,
                             bool fused = false, const AdjRs *rs = nullptr);
// the receive side of the reduce-scatter: this rank's band [B][rows][n] of both jobs, the
// world slots of recv [world][2][B][bmax][n] summed in slot (rank) order, and the band's ei
// partial sum (x2 - x_fbp)^2 (x2 whole images [B][n][n], rows from row0) into ei [B];
// part: >= B * band_reduce_part_floats(n, rows) floats of scratch
size_t band_reduce_part_floats(int n, int rows);
cudaError_t launch_band_reduce(const float *recv, int world, int B, int bmax, int n, int row0,
                               int rows, const float *x2, float *xfbp, float *grad, float *ei,
                               float *part, cudaStream_t s);

void fft_plan(int P, int *npass, int *radix, int *ns, int *twoff, int *twtotal);
// Theorem-1 deviation helpers (deviation.cu): part = [B][kNormChunks] fp64 chunk partials
constexpr int kNormChunks = 128;
cudaError_t launch_sumsq(const float *w, int B, long per, double *part, cudaStream_t s);
cudaError_t launch_normalise(const float *w, float *v, int B, long per, const double *part,
                             float *lambda, int num_sms, cudaStream_t s);
cudaError_t launch_iota(int32_t *a, int n, cudaStream_t s);
// REI: pn = p + sigma eps (rei.cu; R23)
cudaError_t launch_rei_noise(const float *p, float *pn, int B, int m, int n_det, float sigma,
                             uint64_t seed, uint64_t iter, uint64_t image0, int num_sms,
                             cudaStream_t s);
// peers of the fused all-gather (ramp.cu): local rows (b, k) of q and r also go to rows
// (b, row0 + k) of every peer's [B][m_total][n_det] q and r buffers
constexpr int kMaxPeers = 8;
struct RampPeers {
    int n;
    float *q[kMaxPeers];
    float *r[kMaxPeers];
    int m_local, row0, m_total;
};
cudaError_t launch_ramp(const skei_plan *plan, const float *p, float *q, int rows,
                        cudaStream_t s, float *qi = nullptr, int m = 0, int bb = 0,
                        const float *rs = nullptr, float *ri = nullptr, float rscale = 1.f,
                        const RampPeers *peers = nullptr, bool fused = false);

// Residual: partials in ws (float2 per (image, chunk)), then final reduce.
size_t residual_ws_bytes(const skei_plan *plan, int B, int m);
cudaError_t launch_residual(const skei_plan *plan, const float *p1, const float *y,
                            const int32_t *idx, int m, int idx_stride, const float *x2,
                            const float *x3, int B, float *mc, float *ei, float *r,
                            void *ws, cudaStream_t s);

cudaError_t launch_draw(uint64_t seed, uint64_t iter, uint64_t image0, int count, int shared,
                        int n_full, int m, int mode, int32_t *g, int32_t *idx, cudaStream_t s);

cudaError_t launch_smem_probe(float *sink, int blocks, int iters, cudaStream_t s);
cudaError_t launch_l2_probe(const float *buf, long n_floats, float *sink, int blocks, int iters,
                            cudaStream_t s);

// Host draw (library implementation of DESIGN.md R5).
int host_draw(uint64_t seed, uint64_t iter, uint64_t image, int n_full, int m, int mode,
              int32_t *g, int32_t *idx);

// Batch grouping: images sharing one angle list are processed together in groups of bb.
// Image group of the forward projector (same rule as pick_bb; kept separate because the
// packed input layout depends on it).
inline int fwd_bb(int B, int idx_stride) {
    if (idx_stride != 0) return 1;
    if (B % 4 == 0) return 4;
    if (B % 2 == 0) return 2;
    return 1;
}

inline int pick_bb(int B, int idx_stride) {
    if (idx_stride != 0) return 1;
    if (B % 4 == 0) return 4;
    if (B % 2 == 0) return 2;
    return 1;
}

}  // namespace skei
