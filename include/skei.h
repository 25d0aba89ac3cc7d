/*
 * skei.h — C ABI of the B200-native sketched Equivariant Imaging operator pass
 * (arXiv 2411.05771, "Sketched Equivariant Imaging").  PAPER.md references are
 * lines of the paper's source; "R<n>" are the readings listed in DESIGN.md §2.
 *
 * The problem statement is y = A x + eps (Eq. 1) with A the
 * parallel-beam Radon transform of sparse-view CT (L283) and A^+ its filtered
 * backprojection (L40-L43, Eq. 2).  Sketched EI replaces A, A^+ by A_S := S A and
 * A_S^+ with S an angle-subsampling operator (L92, §2.1; Eq. 6).  One
 * iteration of Algorithm 1 (L117-L122) needs, besides the network:
 *   draw (g, S) -> x2 = T_g x1 -> A_S x2, A_S x1 -> ramp -> A_S^+ A_S x2 ->
 *   ||y_S - A_S x1||^2, ||x2 - x3||^2 -> 2 A_S^T (A_S x1 - y_S).
 * Each step is one entry point below; skei_pass chains them.
 *
 * Conventions (all entry points):
 *   - Tensors are fp32, C-contiguous, DEVICE pointers owned by the caller (e.g.
 *     torch tensors) unless a parameter says "host".  The library never frees them.
 *   - Image x      : [B][n][n], row r = 0 at the top, column c = 0 at the left;
 *                    pixel centre (u, v) = (c - (n-1)/2, (n-1)/2 - r)        (R2)
 *   - Sinogram p,y : [B][rows][n_det], angle-major; bin j at s_j = j - (n_det-1)/2,
 *                    spacing 1 pixel                                          (R3)
 *   - Angles       : int32 indices i into theta_i = i*pi/n_full, measured
 *                    counter-clockwise from +u (R2, R4).  A sketch is m strictly
 *                    increasing indices in [0, n_full); idx_stride = 0 shares one
 *                    list across the batch, idx_stride = m gives image b the list
 *                    at idx + b*m.  Index lists are trusted (not re-validated on
 *                    the device).
 *   - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream), performs no device allocation and no hidden sync, and is
 *     deterministic: no floating-point atomics, fixed reduction order, bitwise-
 *     repeatable.  The only atomics are integer completion counters (atomicAdd on
 *     unsigned words in the workspace) that elect which CTA performs a fixed-order
 *     final sum; the counters reset themselves before the kernel exits.
 *   - Arguments are validated on the host before any launch; a failing check
 *     returns SKEI_ERR_SHAPE / SKEI_ERR_CONFIG / SKEI_ERR_ARG and launches nothing.
 *     A launch failure returns SKEI_ERR_CUDA; asynchronous faults surface at the
 *     caller's next synchronisation.
 *   - A plan is immutable after creation and may be used from several streams and
 *     threads concurrently (it owns only read-only device tables).  A workspace `ws`
 *     may NOT be shared by calls that can run concurrently (two streams, or two
 *     threads' calls on one stream that may interleave): it holds the packed images,
 *     the filtered sinogram and the self-resetting completion counters of the call in
 *     flight.  Calls on one stream may reuse one workspace back to back.
 */
#ifndef SKEI_H
#define SKEI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SKEI_OK = 0,
    SKEI_ERR_SHAPE = 1,     /* inconsistent sizes (SPEC-style "shape error")          */
    SKEI_ERR_CONFIG = 2,    /* invalid configuration (m > n_full, bad fft_len, ...)   */
    SKEI_ERR_ARG = 3,       /* NULL pointer / out-of-range scalar argument            */
    SKEI_ERR_CUDA = 4,      /* a CUDA runtime call or kernel launch failed            */
    SKEI_ERR_NO_DEVICE = 5  /* no usable sm_100 device                                */
} skei_status;

typedef void *skei_stream; /* cudaStream_t */

/* Geometry of one CT system: n x n images, n_det detector bins, n_full angles on
 * [0, pi).  fft_len = ramp FFT length P: a power of two >= 2*n_det - 1 (the length
 * at which the zero-padded circular convolution equals the linear one, DESIGN.md
 * §7 "k_ramp"); 0 selects the smallest such power of two.  Limits: 2 <= n <= 1536
 * (a line block of the forward projector, (n + 8) x 128 bytes, must fit in one SM's
 * shared memory), 1 <= n_det <= 3072, 1 <= n_full <= 16384, 16 <= P <= 8192 (fft_len 0
 * selects max(16, pow2 >= 2 n_det - 1)). */
typedef struct {
    int32_t n;
    int32_t n_det;
    int32_t n_full;
    int32_t fft_len;
} skei_geometry;

typedef struct skei_plan skei_plan; /* opaque */

/* Builds the plan on `device`: fp64 trig table of the n_full angles, the ramp
 * spectrum R[k] = DFT_P of the wrapped doubled Ram-Lak kernel (computed in fp64,
 * stored fp32, pre-divided by P) and the FFT twiddles (fp64 -> fp32).  *out
 * receives the plan (owned by the caller; release with skei_plan_destroy).
 * Errors: SKEI_ERR_ARG (NULL), SKEI_ERR_CONFIG (limits above), SKEI_ERR_NO_DEVICE,
 * SKEI_ERR_CUDA. */
skei_status skei_plan_create(const skei_geometry *geom, int device, skei_plan **out);
void skei_plan_destroy(skei_plan *plan);                 /* NULL is a no-op */
skei_status skei_plan_geometry(const skei_plan *plan, skei_geometry *out); /* resolved fft_len */
const char *skei_status_string(skei_status status);     /* static string, never NULL */
const char *skei_last_cuda_error(void);                  /* thread-local, after SKEI_ERR_CUDA */

/* Device scratch needed by skei_radon_fwd / skei_fbp / skei_ei_residual / skei_pass
 * for `batch` images and sketch size m (bytes; 256-byte aligned pieces): the filtered
 * sinogram, the residual partial sums and slots for four packed copies of the images (the
 * forward projector's TMA-friendly input layout, ~4 * batch * n^2 floats; groups of 4
 * images sharing a sketch use two of them, one row-lines copy per image). */
size_t skei_workspace_bytes(const skei_plan *plan, int32_t batch, int32_t m);

/* ---------------------------------------------------------------- a1: draws --
 * Algorithm 1 step 2: sample g ~ G (|G| = 360 integer-degree
 * rotations 1..360, L284) and a sketch S (L102: sample one of N predefined
 * sketches; L299: interleaved minibatches).  Counter-based SplitMix64 keyed by
 * (seed, stream, iter, image) — DESIGN.md §2 R5 gives the exact algorithm; the
 * oracle implements it independently and the integers are bit-identical.
 *   mode 0 = interleaved: requires n_full % m == 0; S = {b + k*n_full/m}.
 *   mode 1 = uniform:     a uniformly random m-subset of [0, n_full), ascending.
 *   image = UINT64_MAX    -> the per-pass shared draw, else a per-image draw.
 * skei_draw is HOST code: g_deg (1 int) and angle_idx (m ints) are host pointers.
 * Errors: SKEI_ERR_ARG (NULL), SKEI_ERR_CONFIG (m < 1, m > n_full, mode, divisibility). */
skei_status skei_draw(uint64_t seed, uint64_t iter, uint64_t image, int32_t n_full,
                      int32_t m, int32_t mode, int32_t *g_deg, int32_t *angle_idx);

/* Same draws generated on the device for `count` images image0 .. image0+count-1
 * (or, if shared != 0, the single shared draw: count must be 1): g_dev[count],
 * idx_dev[count][m] are device pointers.  Bit-identical to skei_draw.
 * Errors: as skei_draw; SKEI_ERR_CONFIG if n_full > 16384. */
skei_status skei_draw_device(uint64_t seed, uint64_t iter, uint64_t image0, int32_t count,
                             int32_t shared, int32_t n_full, int32_t m, int32_t mode,
                             int32_t *g_dev, int32_t *idx_dev, skei_stream stream);

/* ------------------------------------------------------------- a2: rotation --
 * out = T_g x (x2 = T_g(x1); EI group action L65): bilinear
 * interpolation about the image centre, zero outside the grid, content rotated
 * counter-clockwise by g degrees; g in {90,180,270,360} are exact permutations
 * (R11).  g_deg: device int32, one value (g_stride = 0) or one per image
 * (g_stride = 1).  x, out: [B][n][n]; out must not alias x. */
skei_status skei_rotate(const skei_plan *plan, const float *x, float *out, int32_t B,
                        const int32_t *g_deg, int32_t g_stride, skei_stream stream);

/* --------------------------------- next row: rotation transpose --
 * out = T_g^T y, the exact transpose of skei_rotate (the bilinear weights handed back
 * from every output pixel to the in-grid neighbours of its source position), needed to
 * carry the EI term's gradient through x2 = T_g x1 (Eq. 6, Alg. 1
 * steps 4-6 L120-L122).  Computed as a per-pixel gather over the <= 16 output pixels
 * whose source can touch it (no atomics, deterministic).  Source positions in fp64.
 * g_deg, g_stride, y, out as skei_rotate; out must not alias y.
 * Errors: SKEI_ERR_ARG (NULL, g_stride, aliasing), SKEI_ERR_SHAPE (B < 1). */
skei_status skei_rotate_adjoint(const skei_plan *plan, const float *y, float *out, int32_t B,
                                const int32_t *g_deg, int32_t g_stride, skei_stream stream);

/* ---------------- next row: communication-reduced single-image split --
 * The backprojections of the pass restricted to output rows [row0, row0 + rows): with q
 * (the filtered sinogram) and r (the residual) of ALL m sketched angles at hand — after
 * an all-gather of the ranks' angle shards, 2 B m n_det floats — every rank computes its
 * own row band of x_fbp = (pi / 2 m_total) A_S^T q and grad = 2 A_S^T r, and the band's
 * ei partial sum (x2 - x_fbp)^2 (fused, fixed-order reduction), instead of whole-image
 * partials that need an all-reduce of 2 B n^2 floats.  q, r: [B][m][n_det]; x2: [B][n][n]
 * (whole images); xfbp_band, grad_band: [B][rows][n]; ei_band: [B]; all device.
 * Errors: SKEI_ERR_SHAPE (B, m, or the band outside [0, n)), SKEI_ERR_ARG (NULL, strides,
 * m_total < m, ws too small). */
/* The fused exchange of that split (no NCCL on the data path): q = ramp(p) for this
 * rank's m_local sketched rows (written to q_local [B][m_local][n_det]) with every output
 * row ALSO stored, from the ramp kernel's last pass, into row (b, row0 + k) of each of the
 * n_peers buffers peer_q[g] [B][m_total][n_det] — device pointers valid on this GPU
 * (NVLink P2P / symmetric memory, this rank's own buffer among them) — and the residual
 * rows r [B][m_local][n_det] likewise into peer_r[g].  The transfer overlaps the FFT tile
 * by tile; after a cross-rank barrier every rank holds the whole q and r for
 * skei_backproject_band.  peer_q, peer_r: HOST arrays of n_peers (<= 8) device pointers.
 * Errors: SKEI_ERR_SHAPE (B, m_local < 1, rows outside [0, m_total)), SKEI_ERR_ARG. */
skei_status skei_ramp_allgather(const skei_plan *plan, int32_t B, const float *p,
                                const float *r, int32_t m_local, int32_t row0, int32_t m_total,
                                float *q_local, float *const *peer_q, float *const *peer_r,
                                int32_t n_peers, skei_stream stream);

skei_status skei_backproject_band(const skei_plan *plan, int32_t B, const float *q,
                                  const float *r, const int32_t *idx, int32_t m,
                                  int32_t idx_stride, int32_t m_total, const float *x2,
                                  int32_t row0, int32_t rows, float *xfbp_band,
                                  float *grad_band, float *ei_band, void *ws, size_t ws_bytes,
                                  skei_stream stream);

/* ---------- next row: the backprojector with its reduce-scatter fused --
 * The other communication-reduced form of the single-image angle split: each rank
 * backprojects only its own angle shard — x_fbp partial (pi / 2 m_total) A_{S_r}^T q and
 * grad partial 2 A_{S_r}^T r (the pass's sums over angles split over ranks, PAPER.md L70,
 * L92) — and the kernel's epilogue stores every output row straight into the receive
 * buffer of the rank that owns the row's band (P2P stores over NVLink into symmetric
 * memory), so the reduce-scatter of 2 B n^2 floats overlaps the backprojection tile by
 * tile; no NCCL on the data path.  Row bands as dist.batch_range(n, o, world): rank o owns
 * rows [o q + min(o, n mod world), ... + q + (o < n mod world)), q = n / world; bmax =
 * ceil(n / world).  Receive buffer of every rank: [world slots][2 jobs][B][bmax][n] fp32
 * (skei_rs_recv_floats), slot s written only by rank s, job 0 = x_fbp, job 1 = grad.
 * q, r: this rank's m sketched rows [B][m][n_det] (device); idx, idx_stride as skei_fbp;
 * peer_recv: HOST array of `world` (<= 8) device pointers to the ranks' receive buffers,
 * valid on this GPU (this rank's own among them).  Errors: SKEI_ERR_SHAPE (B, m),
 * SKEI_ERR_ARG (NULL, strides, m_total < m, world / rank out of range). */
size_t skei_rs_recv_floats(const skei_plan *plan, int32_t B, int32_t world);
skei_status skei_backproject_scatter(const skei_plan *plan, int32_t B, const float *q,
                                     const float *r, const int32_t *idx, int32_t m,
                                     int32_t idx_stride, int32_t m_total,
                                     float *const *peer_recv, int32_t world, int32_t rank,
                                     skei_stream stream);
/* The receive side, after a cross-rank barrier (every rank's scatter has landed): this
 * rank's band of x_fbp and grad, xfbp_band / grad_band [B][rows][n], as the world slots of
 * recv (this rank's receive buffer) summed in slot (rank) order — fixed order, bitwise
 * reproducible — and the band's ei partial sum_(band) (x2 - x_fbp)^2 into ei_band [B] (x2:
 * whole images [B][n][n]; per-CTA partials summed in CTA order in fp64).  An all-reduce of
 * the B ei partials (and the mc partials) completes the losses.  ws >=
 * skei_workspace_bytes(plan, B, 1).  Errors: SKEI_ERR_SHAPE (B < 1), SKEI_ERR_ARG. */
skei_status skei_band_reduce(const skei_plan *plan, int32_t B, const float *recv, int32_t world,
                             int32_t rank, const float *x2, float *xfbp_band, float *grad_band,
                             float *ei_band, void *ws, size_t ws_bytes, skei_stream stream);

/* ------------------- next row: the Theorem-1 sketching deviation --
 * delta = ||A^T (S^T S - I) A||_2 (Theorem 1, proof L575-L583) for the
 * sqrt(n_full/m)-scaled row subsampling onto the sketched angles idx, by `iters` power
 * iterations on D v = (n_full/m) A_S^T A_S v - A^T A v (A: all n_full angles), batched
 * over B independent start images.  v: [B][n][n] device, in: start vectors (normalised
 * first), out: the last normalised iterate; lambda: [B] device, out: ||D v|| of the last
 * iteration (-> delta).  The operators are the pass's kernels (packing, forward projector,
 * backprojector accumulating into a base); the norms are fixed-order fp64 reductions.
 * ws >= skei_workspace_bytes(plan, B, n_full) (NOTE: n_full, not m).
 * Errors: SKEI_ERR_SHAPE (B, m), SKEI_ERR_ARG (NULL, iters < 1, strides, ws too small). */
skei_status skei_sketch_deviation(const skei_plan *plan, int32_t B, const int32_t *idx,
                                  int32_t m, int32_t idx_stride, int32_t iters, float *v,
                                  float *lambda, void *ws, size_t ws_bytes, skei_stream stream);

/* The transpose of skei_fbp (next row): p = (pi / 2 m_total) ramp(A_S x)
 * (the ramp kernel is even, so ramp is symmetric), i.e. the vector-Jacobian product of
 * the sketched FBP.  x: [B][n][n], p: [B][m][n_det] device; other arguments and errors as
 * skei_fbp. */
skei_status skei_fbp_adjoint(const skei_plan *plan, const float *x, float *p, int32_t B,
                             const int32_t *idx, int32_t m, int32_t idx_stride, int32_t m_total,
                             void *ws, size_t ws_bytes, skei_stream stream);

/* ------------------------- next row: the EI branch's gradient --
 * grad = d ||x2 - x3||^2 / d x1 for x2 = T_g x1 and the identity network
 * x3 = M x2, M = (pi/2m) A_S^T ramp A_S (the sketched FBP, R16; Eq. 6
 * L97-L101, Alg. 1 steps 4-6 L120-L122).  M is symmetric, so
 *   grad = T_g^T (I - M) d,   d = 2 (x2 - x3),
 * computed as: d (packed for the projector), A_S d, ramp, u = d - (pi/2m) A_S^T q,
 * T_g^T u — five launches on `stream`.  x2, x3: [B][n][n] device (skei_pass's x2 and
 * xfbp); g_deg, g_stride as skei_rotate; idx, m, idx_stride as skei_radon_fwd;
 * grad: [B][n][n] device, must not alias x2 or x3; ws >= skei_workspace_bytes(plan, B, m).
 * Errors: SKEI_ERR_SHAPE (B < 1, m < 1 or m > n_full), SKEI_ERR_ARG (NULL, strides,
 * aliasing, ws too small). */
skei_status skei_ei_grad(const skei_plan *plan, int32_t B, const float *x2, const float *x3,
                         const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                         int32_t idx_stride, float *grad, void *ws, size_t ws_bytes,
                         skei_stream stream);

/* ------------------------------------------------------ a3: forward A_S --------
 * p[b][k][j] = sum_{r,c} x[b][r][c] * max(0, 1 - |u_c cos th + v_r sin th - s_j|),
 * th = theta_{idx_b[k]} (BASELINE.json north_star projector; PAPER.md L283
 * "discrete radon transform"; sketched rows L92 A_S := S A).  Computed as a
 * gather per (angle, detector bin) — no atomics.  x: [B][n][n]; p: [B][m][n_det].
 * The images are first packed into ws (line blocks), so ws must hold
 * >= skei_workspace_bytes(plan, B, m) bytes.  Errors: SKEI_ERR_SHAPE (B < 1, m < 1
 * or m > n_full), SKEI_ERR_ARG (NULL, idx_stride not 0 or m, ws too small). */
skei_status skei_radon_fwd(const skei_plan *plan, const float *x, float *p, int32_t B,
                           const int32_t *idx, int32_t m, int32_t idx_stride, void *ws,
                           size_t ws_bytes, skei_stream stream);

/* ---------------------------------------------------- a5/a8: adjoint A_S^T ------
 * x[b] = scale * A_S^T p[b]: the exact transpose of skei_radon_fwd (linear
 * interpolation of each sinogram row at t = u cos th + v sin th, out-of-range
 * taps dropped), a per-pixel gather over the m angles.  p: [B][m][n_det];
 * x: [B][n][n] (overwritten).  scale = 2 gives the MC-loss gradient
 * 2 A_S^T r.  Errors as skei_radon_fwd. */
skei_status skei_radon_adj(const skei_plan *plan, const float *p, float *x, int32_t B,
                           const int32_t *idx, int32_t m, int32_t idx_stride, float scale,
                           skei_stream stream);

/* ------------------------------------------------------------- a4: ramp --------
 * q[r] = h2 (*) p[r] for each of `rows` sinogram rows of length n_det: linear
 * convolution with the doubled Ram-Lak kernel h2(0) = 1/2, h2(odd n) =
 * -2/(pi^2 n^2), h2(even n != 0) = 0 (R8), computed as a zero-padded length-P
 * complex FFT (two real rows per transform) x R[k] -> inverse FFT, truncated to
 * n_det.  p, q: [rows][n_det]; q may alias p.  Errors: SKEI_ERR_SHAPE (rows < 1). */
skei_status skei_ramp_filter(const skei_plan *plan, const float *p, float *q, int32_t rows,
                             skei_stream stream);

/* ------------------------------------------------------------ a4+a5: FBP -------
 * x[b] = (pi / (2 m_total)) * A_S^T ramp(p[b])  — the sketched pseudo-inverse
 * A_S^+ (BASELINE.json north_star; PAPER.md L92 A_S^+, L102 "FBP").  m_total is
 * the sketch size the density compensation refers to (= m, or the full sketch
 * size when the m angles are one rank's shard of an angle-split pass).  No
 * circular mask (R10).  ws: >= skei_workspace_bytes(plan, B, m) bytes of device
 * scratch.  Errors: as skei_radon_adj; SKEI_ERR_ARG if m_total < m. */
skei_status skei_fbp(const skei_plan *plan, const float *p, float *x, int32_t B,
                     const int32_t *idx, int32_t m, int32_t idx_stride, int32_t m_total,
                     void *ws, size_t ws_bytes, skei_stream stream);

/* --------------------------------------------------------- a7: residuals -------
 * r[b][k][j] = p1[b][k][j] - y[b][idx_b[k]][j];  mc[b] = sum r^2;
 * ei[b] = sum (x2[b] - x3[b])^2  (PAPER.md L122 loss terms; Eq. 6;
 * unnormalised squared l2 norms, R15).  p1: [B][m][n_det] (= A_S x1);
 * y: [B][n_full][n_det] full measured sinogram; x2, x3: [B][n][n]; mc, ei: [B];
 * r: [B][m][n_det] or NULL (not written).  Two-stage deterministic reduction.
 * Either part may be skipped: p1 = y = mc = NULL computes only ei (idx then only sizes
 * the workspace), x2 = x3 = ei = NULL only r and mc.  ws as skei_fbp. */
skei_status skei_ei_residual(const skei_plan *plan, const float *p1, const float *y,
                             const int32_t *idx, int32_t m, int32_t idx_stride,
                             const float *x2, const float *x3, int32_t B,
                             float *mc, float *ei, float *r,
                             void *ws, size_t ws_bytes, skei_stream stream);

/* ------------------------------------------------------ the whole pass (§8(a)) --
 * One sketched-EI operator pass for B images given their draws (g, S):
 *   x2 = T_g x1;  p2 = A_S x2;  p1 = A_S x1;  q = ramp(p2);
 *   xfbp = (pi/2m) A_S^T q;  x3 = x3_in if non-NULL else xfbp (identity network,
 *   R16);  r = p1 - y_S;  mc = ||r||^2;  ei = ||x2 - x3||^2;  grad = 2 A_S^T r.
 * All outputs are required device buffers of the shapes above.  ws as skei_fbp
 * (skei_workspace_bytes(plan, B, m)). */
typedef struct {
    float *x2, *p1, *p2, *q, *xfbp, *r, *grad, *mc, *ei;
} skei_pass_outputs;

skei_status skei_pass(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                      const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                      int32_t idx_stride, const float *x3_in, const skei_pass_outputs *out,
                      void *ws, size_t ws_bytes, skei_stream stream);

/* End-to-end variant from HOST buffers: copies host x1 [B][n][n], host y
 * [B][n_full][n_det], host g [B or 1] and host idx into the caller's device
 * buffers (d_x1, d_y, d_g, d_idx, same shapes), runs skei_pass, and copies
 * mc/ei back into host h_mc[B], h_ei[B].  Only the m sketched rows of each image's y
 * need to cross the link (the pass only reads y_S, Alg. 1 step 6).  Equispaced
 * sketches (uniform mode: idx_b[k] = idx_b[0] + k d; for a shared sketch also d | n_full)
 * are copied in place as a pitched sub-array of y — one 3-D copy for a shared sketch,
 * one 2-D copy per image otherwise — into the head of d_y as y_S [B][m][n_det], with no
 * host gather and h_ystage untouched (transfers under 2 MB with an h_ystage keep the
 * gather: it is cheaper than the pitched copy's per-row cost).  Otherwise, if h_ystage (host, >= B*m*n_det floats,
 * pinned) is given: image b's rows idx_b[0..m) (its own sketch when
 * idx_stride = m) are gathered into it on the calling thread (up to 8 host threads for
 * batches over 4 MB of rows) and sent as one copy into the head of d_y as y_S
 * [B][m][n_det].  h_ystage is rewritten at call time, so a previous call's copy from it
 * must have completed.  Without h_ystage (may be NULL) a shared sketch (idx_stride 0)
 * uses one strided copy per run of consecutive angle indices and per-image sketches
 * copy all of y.
 * Results are identical to skei_pass on device copies.  Host buffers should be
 * pinned for the copies to be asynchronous.  The caller synchronises `stream`
 * before reading h_mc / h_ei.  Errors: as skei_pass; SKEI_ERR_ARG if a host
 * angle index is outside [0, n_full). */
skei_status skei_pass_host(const skei_plan *plan, int32_t B, const float *h_x1,
                           const float *h_y, const int32_t *h_g, int32_t g_stride,
                           const int32_t *h_idx, int32_t m, int32_t idx_stride,
                           float *d_x1, float *d_y, int32_t *d_g, int32_t *d_idx,
                           const skei_pass_outputs *out, float *h_mc, float *h_ei,
                           float *h_ystage, void *ws, size_t ws_bytes, skei_stream stream);

/* ---------------------------- next row: the REI variant of the pass --
 * Robust EI: the EI branch reconstructs from simulated noisy measurements,
 * x3 = F(A_S^+ (A_S x2 + sigma eps)).  Identical to skei_pass with x3 = NULL except
 * q = ramp(p2 + sigma eps) (p2 is still reported noise-free; x_fbp, ei follow from q).
 * eps[b][k][j] ~ N(0, 1): Box-Muller (cos branch) on words 2s, 2s+1 (s = k n_det + j) of
 * the counter-based SplitMix64 stream keyed by (noise_seed, stream 5, noise_iter,
 * image0 + b) — DESIGN.md R23; reproducible, independent of the launch configuration.
 * sigma = 0 gives skei_pass's results.  Errors: as skei_pass; SKEI_ERR_ARG if sigma < 0. */
skei_status skei_pass_rei(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                          const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                          int32_t idx_stride, float sigma, uint64_t noise_seed,
                          uint64_t noise_iter, uint64_t image0, const skei_pass_outputs *out,
                          void *ws, size_t ws_bytes, skei_stream stream);

/* skei_pass with stage timing: `events` holds n_events (>= 6) cudaEvent_t handles
 * created by the caller, NULL entries skipped; event 0 is recorded before the first stage
 * and event i after stage i of: 1 rotate + packing, 2 forward (A_S x1 with the fused MC
 * residual, and A_S x2: one launch), 3 ramp, 4 the two backprojections (FBP and gradient,
 * one launch, with the fused EI residual), 5 end.  Under stream capture the events
 * become external event-record nodes.  Otherwise identical to skei_pass with x3 = NULL
 * (same launches, same results). */
skei_status skei_pass_profiled(const skei_plan *plan, int32_t B, const float *x1,
                               const float *y, const int32_t *g_deg, int32_t g_stride,
                               const int32_t *idx, int32_t m, int32_t idx_stride,
                               const skei_pass_outputs *out, void *ws, size_t ws_bytes,
                               void *const *events, int32_t n_events, skei_stream stream);

/* The whole of Algorithm 1 steps 2-6 in one call: the device draw
 * a1 (skei_draw_device's draws, bit-identical to skei_draw) followed by skei_pass with
 * x3 = NULL on those draws.  The rotation-and-packing launch is programmatically
 * serialised behind the draw kernel, so packing x1 overlaps the draw (only the rotation of
 * x1 waits for g).  draw->shared = 1: one draw for the batch (g_dev[1], idx_dev[1][m]);
 * 0: a draw per image image0 + b (g_dev[B], idx_dev[B][m]); both device buffers are
 * written by the call and read by the rest of the pass.  events: NULL, or n_events >= 6
 * stage events as in skei_pass_profiled (event 0 before the draw).  Results are identical
 * to skei_draw_device + skei_pass.  Errors: SKEI_ERR_ARG (NULL plan, draw, g_dev,
 * idx_dev; shared not 0/1; events with n_events < 6), SKEI_ERR_SHAPE (B < 1, m < 1,
 * m > n_full), SKEI_ERR_CONFIG (mode, divisibility), else as skei_pass. */
typedef struct {
    uint64_t seed, iter, image0;  /* the draw's key (R5); image0 unused when shared */
    int32_t shared;               /* 1: shared per pass, 0: per image */
    int32_t mode;                 /* 0 interleaved, 1 uniform */
} skei_draw_spec;
skei_status skei_pass_draw(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                           const skei_draw_spec *draw, int32_t m, int32_t *g_dev,
                           int32_t *idx_dev, const skei_pass_outputs *out, void *ws,
                           size_t ws_bytes, void *const *events, int32_t n_events,
                           skei_stream stream);

/* Diagnostic: shared-memory read bandwidth probe (the roofline denominator of the
 * gather kernels).  Launches `blocks` CTAs of 1024 threads that each
 * stream LDS.128 over a 32 KB shared buffer `iters` times; `sink` (device, >= blocks
 * floats) receives per-block checksums so the loads cannot be elided.  Bytes read =
 * blocks * 1024 * 16 * 32 * iters. */
skei_status skei_smem_probe(float *sink, int32_t blocks, int32_t iters, skei_stream stream);

/* Diagnostic: L2 read bandwidth probe (the bound of the forward
 * projector's re-staging of packed line blocks, which after the first unit come from L2).
 * `blocks` CTAs of 1024 threads each read the whole device buffer buf[n_floats] `iters`
 * times with L1-bypassing 16-byte loads (each CTA from its own starting offset); size buf
 * well under the L2 (cudaDevAttrL2CacheSize) so the sweeps after the first hit L2.
 * sink: device, >= blocks floats (checksums).  Bytes read = blocks * n_floats * 4 * iters.
 * Errors: SKEI_ERR_ARG (NULL, blocks / iters < 1, n_floats < 4096 or not a multiple of 4,
 * buf not 16-byte aligned). */
skei_status skei_l2_probe(const float *buf, int64_t n_floats, float *sink, int32_t blocks,
                          int32_t iters, skei_stream stream);

/* Library build info: "skei <version> sm_100a". */
const char *skei_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SKEI_H */
