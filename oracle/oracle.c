/*
 * oracle/oracle.c — ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the sketched-EI CT
 * operator pass of arXiv 2411.05771 (PAPER.md = /root/reference/PAPER.md):
 *   Algorithm 1: step 2 "obtain randomly sketched operators
 *   A_S, A_S^+, sample g" (L118), step 4 x2 = T_g x1 (L120), the operator part of
 *   step 5 A_S^+ A_S x2 (L121), and the residuals of step 6
 *   ||y_S - A_S x1||^2 + lambda ||x2 - x3||^2 (L122), plus the data-term gradient
 *   2 A_S^T (A_S x1 - y_S).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
 * may load this library.  It shares no code, header, table or helper with the CUDA
 * path in paper_2411_05771_b200/; neither includes nor links the other.
 *
 * Every routine is the plain definition written out with naive loops, in fp64:
 *   - forward projection as a SCATTER over pixels (the CUDA path gathers over bins),
 *   - the ramp filter as a DIRECT O(n_det^2) linear convolution (the CUDA path uses
 *     a zero-padded FFT),
 *   - the backprojection as a per-pixel gather,
 *   - direct bilinear rotation, direct sums of squares,
 *   - its own SplitMix64 draw generator.
 * The readings of the paper behind every constant are listed in DESIGN.md §2
 * (R1..R22); each function names the one it follows.  Parity status of each function
 * (the pins in tests/test_oracle_pins.py) is listed in DESIGN.md §4; none is unpinned.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_PI 3.14159265358979323846

/* ------------------------------------------------------------------ draws (R5) --
 * SURVEY §8(c) O-1.  PAPER.md L102 ("predefine a set of N sketching operators ...
 * randomly sample a S_i"), L299 ("N minibatches ... from interleaved angles"),
 * L284 (|G| = 360 rotations of 1..360 degrees); BASELINE.json north_star
 * ("a seeded uniform subset of m of the full angles"; draws "bit-identical").
 * mix() is the SplitMix64 finaliser applied after the golden-ratio increment, so
 * oracle_word(key, i) is the i-th output of a SplitMix64 stream seeded with key. */
static uint64_t oracle_mix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_word(uint64_t key, uint64_t i)
{
    return oracle_mix(key + i * 0x9E3779B97F4A7C15ULL);
}

uint64_t oracle_key(uint64_t seed, uint64_t stream, uint64_t iter, uint64_t image)
{
    return oracle_mix(oracle_mix(oracle_mix(oracle_mix(seed) ^ stream) ^ iter) ^ image);
}

/* U(n) = floor(w * n / 2^64) */
static uint64_t oracle_below(uint64_t w, uint64_t n)
{
    return (uint64_t)(((unsigned __int128)w * (unsigned __int128)n) >> 64);
}

/* mode 0 = interleaved partition, 1 = uniform m-subset (north_star).
 * Returns 0 on success, 2 on a config error. */
int oracle_draw(uint64_t seed, uint64_t iter, uint64_t image, int n_full, int m, int mode,
                int *g_deg, int *idx)
{
    if (n_full < 1 || m < 1 || m > n_full) return 2;
    uint64_t krot = oracle_key(seed, 1, iter, image);
    *g_deg = 1 + (int)oracle_below(oracle_word(krot, 0), 360);
    uint64_t ksk = oracle_key(seed, 2, iter, image);
    if (mode == 0) {
        if (n_full % m != 0) return 2;
        int nb = n_full / m;
        int b = (int)oracle_below(oracle_word(ksk, 0), (uint64_t)nb);
        for (int k = 0; k < m; ++k) idx[k] = b + k * nb;
        return 0;
    }
    if (mode != 1) return 2;
    int *a = (int *)malloc(sizeof(int) * (size_t)n_full);
    if (!a) return 2;
    for (int i = 0; i < n_full; ++i) a[i] = i;
    for (int i = 0; i < m; ++i) {
        int j = i + (int)oracle_below(oracle_word(ksk, (uint64_t)i), (uint64_t)(n_full - i));
        int t = a[i]; a[i] = a[j]; a[j] = t;
    }
    /* sort the chosen m ascending (insertion sort: plain and obviously correct) */
    for (int i = 1; i < m; ++i) {
        int v = a[i], j = i - 1;
        while (j >= 0 && a[j] > v) { a[j + 1] = a[j]; --j; }
        a[j + 1] = v;
    }
    for (int k = 0; k < m; ++k) idx[k] = a[k];
    free(a);
    return 0;
}

/* ------------------------------------------------------------- rotation (R11) --
 * x2 = T_g x1 (|G| = 360 integer degrees, L284).  Bilinear, zero
 * outside, about the image centre, content rotated counter-clockwise for g > 0:
 * out(u, v) = x(u cos g + v sin g, -u sin g + v cos g).  cos/sin are exact at
 * multiples of 90 degrees so g = 90/180/270/360 are exact permutations. */
static void oracle_cossin_deg(int g, double *c, double *s)
{
    int gm = ((g % 360) + 360) % 360;
    if (gm == 0) { *c = 1; *s = 0; return; }
    if (gm == 90) { *c = 0; *s = 1; return; }
    if (gm == 180) { *c = -1; *s = 0; return; }
    if (gm == 270) { *c = 0; *s = -1; return; }
    *c = cos(ORACLE_PI * gm / 180.0);
    *s = sin(ORACLE_PI * gm / 180.0);
}

void oracle_rotate(const double *x, double *out, int N, int g)
{
    double cg, sg;
    oracle_cossin_deg(g, &cg, &sg);
    double h = (N - 1) / 2.0;
    for (int r = 0; r < N; ++r) {
        for (int c = 0; c < N; ++c) {
            double u = c - h, v = h - r;
            double us = u * cg + v * sg;
            double vs = -u * sg + v * cg;
            double cs = us + h, rs = h - vs;
            double r0 = floor(rs), c0 = floor(cs);
            double a = rs - r0, b = cs - c0;
            double acc = 0.0;
            for (int dr = 0; dr < 2; ++dr) {
                for (int dc = 0; dc < 2; ++dc) {
                    long rr = (long)r0 + dr, cc = (long)c0 + dc;
                    if (rr < 0 || rr >= N || cc < 0 || cc >= N) continue;
                    double w = (dr ? a : 1.0 - a) * (dc ? b : 1.0 - b);
                    acc += w * x[rr * N + cc];
                }
            }
            out[(long)r * N + c] = acc;
        }
    }
}

/* ------------------------------------------ rotation transpose (R11, §8(f) #1) --
 * out = T_g^T y: the transpose of oracle_rotate, written as a SCATTER: every output
 * pixel (r, c) of the rotation hands y[r][c] back to the (in-grid) bilinear neighbours
 * of its source position with the same weights.  It is what the EI term's gradient
 * needs to pass d||x2 - x3||^2 / dx2 back through x2 = T_g x1 (Eq. 6,
 * Alg. 1 steps 4-6 L120-L122). */
void oracle_rotate_adj(const double *y, double *out, int N, int g)
{
    double cg, sg;
    oracle_cossin_deg(g, &cg, &sg);
    double h = (N - 1) / 2.0;
    for (long i = 0; i < (long)N * N; ++i) out[i] = 0.0;
    for (int r = 0; r < N; ++r) {
        for (int c = 0; c < N; ++c) {
            double u = c - h, v = h - r;
            double us = u * cg + v * sg;
            double vs = -u * sg + v * cg;
            double cs = us + h, rs = h - vs;
            double r0 = floor(rs), c0 = floor(cs);
            double a = rs - r0, b = cs - c0;
            double val = y[(long)r * N + c];
            for (int dr = 0; dr < 2; ++dr) {
                for (int dc = 0; dc < 2; ++dc) {
                    long rr = (long)r0 + dr, cc = (long)c0 + dc;
                    if (rr < 0 || rr >= N || cc < 0 || cc >= N) continue;
                    double w = (dr ? a : 1.0 - a) * (dc ? b : 1.0 - b);
                    out[rr * N + cc] += w * val;
                }
            }
        }
    }
}

/* ------------------------------------------------------- forward A_S (R1-R4) --
 * p[k][j] = sum_{r,c} x[r][c] * max(0, 1 - |u_c cos th + v_r sin th - s_j|),
 * th = idx[k] * pi / n_full, u_c = c-(N-1)/2, v_r = (N-1)/2-r, s_j = j-(n_det-1)/2
 * (BASELINE.json north_star formula; "discrete radon transform").
 * Written as a SCATTER: each pixel deposits (1-f) x at j0 and f x at j0+1 where
 * t - s_0 = j0 + f; taps outside [0, n_det) are dropped (R18). */
void oracle_fwd(const double *x, double *p, int N, int n_det, int n_full,
                const int *idx, int m)
{
    double h = (N - 1) / 2.0, hd = (n_det - 1) / 2.0;
    memset(p, 0, sizeof(double) * (size_t)m * (size_t)n_det);
    for (int k = 0; k < m; ++k) {
        double th = ORACLE_PI * idx[k] / n_full;
        double ct = cos(th), st = sin(th);
        double *row = p + (long)k * n_det;
        for (int r = 0; r < N; ++r) {
            for (int c = 0; c < N; ++c) {
                double val = x[(long)r * N + c];
                double t = (c - h) * ct + (h - r) * st;
                double pos = t + hd;
                double j0 = floor(pos);
                double f = pos - j0;
                long j = (long)j0;
                if (j >= 0 && j < n_det) row[j] += (1.0 - f) * val;
                if (j + 1 >= 0 && j + 1 < n_det) row[j + 1] += f * val;
            }
        }
    }
}

/* -------------------------------------------------------- adjoint A_S^T (R1) --
 * a[r][c] = scale * sum_k sum_j p[k][j] max(0, 1 - |t_rc(th_k) - s_j|): the exact
 * transpose of oracle_fwd, written as a per-pixel gather (linear interpolation of
 * row k at t with out-of-range taps dropped). */
void oracle_adj(const double *p, double *x, int N, int n_det, int n_full,
                const int *idx, int m, double scale)
{
    double h = (N - 1) / 2.0, hd = (n_det - 1) / 2.0;
    for (long i = 0; i < (long)N * N; ++i) x[i] = 0.0;
    for (int k = 0; k < m; ++k) {
        double th = ORACLE_PI * idx[k] / n_full;
        double ct = cos(th), st = sin(th);
        const double *row = p + (long)k * n_det;
        for (int r = 0; r < N; ++r) {
            for (int c = 0; c < N; ++c) {
                double t = (c - h) * ct + (h - r) * st;
                double pos = t + hd;
                double j0 = floor(pos);
                double f = pos - j0;
                long j = (long)j0;
                double acc = 0.0;
                if (j >= 0 && j < n_det) acc += (1.0 - f) * row[j];
                if (j + 1 >= 0 && j + 1 < n_det) acc += f * row[j + 1];
                x[(long)r * N + c] += acc;
            }
        }
    }
    for (long i = 0; i < (long)N * N; ++i) x[i] *= scale;
}

/* ------------------------------------------------------------ ramp (R8, R9) --
 * q[k][i] = sum_{j=0}^{n_det-1} h2(i-j) p[k][j] with the doubled Ram-Lak (Kak-Slaney)
 * kernel h2(0) = 1/2, h2(even != 0) = 0, h2(odd n) = -2/(pi^2 n^2); its
 * infinite-length response is 2|f| on |f| <= 1/2.  Direct linear convolution, output
 * truncated to n_det (BASELINE.json north_star "Ram-Lak ramp"; PAPER.md L283
 * `iradon`). */
static double oracle_h2(long n)
{
    if (n == 0) return 0.5;
    if (n % 2 == 0) return 0.0;
    return -2.0 / (ORACLE_PI * ORACLE_PI * (double)n * (double)n);
}

void oracle_ramp(const double *p, double *q, int rows, int n_det)
{
    for (int k = 0; k < rows; ++k) {
        const double *pr = p + (long)k * n_det;
        double *qr = q + (long)k * n_det;
        for (int i = 0; i < n_det; ++i) {
            double acc = 0.0;
            for (int j = 0; j < n_det; ++j) acc += oracle_h2((long)i - j) * pr[j];
            qr[i] = acc;
        }
    }
}

/* ------------------------------------------------------- sketched FBP (R7,R9) --
 * A_S^+ p = (pi / (2 m_total)) A_S^T ramp(p)  (BASELINE.json north_star
 * "A_S^+ = (pi/2m) A_S^T ramp"; "A_S^+ ... stable approximations
 * ... FBP").  No circular mask (R10).  m_total = the sketch size the density
 * compensation refers to (= m unless the angles are sharded across ranks). */
void oracle_fbp(const double *p, double *x, int N, int n_det, int n_full,
                const int *idx, int m, int m_total)
{
    double *q = (double *)malloc(sizeof(double) * (size_t)m * (size_t)n_det);
    oracle_ramp(p, q, m, n_det);
    oracle_adj(q, x, N, n_det, n_full, idx, m, ORACLE_PI / (2.0 * m_total));
    free(q);
}

/* -------------------------------------------------------- residuals (R14-R16) --
 * r = p1 - y[S]; mc = sum r^2; ei = sum (x2 - x3)^2  (PAPER.md L122 loss of Alg. 1
 * step 6 and Eq. 6, unnormalised squared norms). */
void oracle_residual(const double *p1, const double *y, const int *idx, int m, int n_det,
                     const double *x2, const double *x3, int N,
                     double *mc, double *ei, double *r)
{
    double s = 0.0;
    for (int k = 0; k < m; ++k) {
        for (int j = 0; j < n_det; ++j) {
            double d = p1[(long)k * n_det + j] - y[(long)idx[k] * n_det + j];
            if (r) r[(long)k * n_det + j] = d;
            s += d * d;
        }
    }
    *mc = s;
    double e = 0.0;
    for (long i = 0; i < (long)N * N; ++i) {
        double d = x2[i] - x3[i];
        e += d * d;
    }
    *ei = e;
}

/* ---------------------------------------------------- the whole pass (§8(a)) --
 * One image of the pass, given its draw (g, idx):
 *   x2 = T_g x1; p2 = A_S x2; p1 = A_S x1; q = ramp(p2); xfbp = (pi/2m) A_S^T q;
 *   x3 = xfbp if x3_in == NULL (identity network, R16) else x3_in;
 *   r = p1 - y_S; mc = ||r||^2; ei = ||x2 - x3||^2; grad = 2 A_S^T r.
 * y is the full measured sinogram [n_full][n_det].  Any output pointer may be NULL
 * except those the later steps need internally (allocated here). */
static void oracle_pass_impl(const double *x1, const double *y, int N, int n_det, int n_full,
                             int g, const int *idx, int m, const double *x3_in,
                             const double *p2_noise,
                             double *x2, double *p1, double *p2, double *q, double *xfbp,
                             double *r, double *grad, double *mc, double *ei);

void oracle_pass(const double *x1, const double *y, int N, int n_det, int n_full,
                 int g, const int *idx, int m, const double *x3_in,
                 double *x2, double *p1, double *p2, double *q, double *xfbp,
                 double *r, double *grad, double *mc, double *ei)
{
    oracle_pass_impl(x1, y, N, n_det, n_full, g, idx, m, x3_in, NULL, x2, p1, p2, q, xfbp, r,
                     grad, mc, ei);
}

/* ------------------------------------- REI simulated noise (R23, §8(f) #3) --
 * eps[k][j] ~ N(0, 1) i.i.d. for sketch row k, bin j of one image: sample s = k n_det + j
 * is Box-Muller (cos branch) on words 2s and 2s+1 of the counter-based stream keyed by
 * (seed, stream 5 = REI noise, iter, image), u = ((w >> 11) + 1/2) 2^-53 in (0, 1)
 * (SURVEY §8(c) O-8's uniform; PAPER.md L104 REI "simulated noise"). */
void oracle_rei_noise(uint64_t seed, uint64_t iter, uint64_t image, int m, int n_det, double *eps)
{
    uint64_t key = oracle_key(seed, 5, iter, image);
    for (long s = 0; s < (long)m * n_det; ++s) {
        double u1 = ((double)(oracle_word(key, 2 * (uint64_t)s) >> 11) + 0.5) * 0x1p-53;
        double u2 = ((double)(oracle_word(key, 2 * (uint64_t)s + 1) >> 11) + 0.5) * 0x1p-53;
        eps[s] = sqrt(-2.0 * log(u1)) * cos(2.0 * ORACLE_PI * u2);
    }
}

/* ------------------------------------------- the REI pass (R23, §8(f) #3) --
 * The robust-EI variant: the EI branch's reconstruction
 * sees simulated measurement noise, x3 = F(A_S^+ (A_S x2 + sigma eps)): identical to
 * oracle_pass except q = ramp(p2 + sigma eps) (p2 itself is reported noise-free). */
void oracle_pass_rei(const double *x1, const double *y, int N, int n_det, int n_full,
                     int g, const int *idx, int m, double sigma, uint64_t seed,
                     uint64_t iter, uint64_t image,
                     double *x2, double *p1, double *p2, double *q, double *xfbp,
                     double *r, double *grad, double *mc, double *ei)
{
    double *noise = (double *)malloc(sizeof(double) * (size_t)m * (size_t)n_det);
    oracle_rei_noise(seed, iter, image, m, n_det, noise);
    for (long s = 0; s < (long)m * n_det; ++s) noise[s] *= sigma;
    oracle_pass_impl(x1, y, N, n_det, n_full, g, idx, m, NULL, noise, x2, p1, p2, q, xfbp, r,
                     grad, mc, ei);
    free(noise);
}

static void oracle_pass_impl(const double *x1, const double *y, int N, int n_det, int n_full,
                             int g, const int *idx, int m, const double *x3_in,
                             const double *p2_noise,
                             double *x2, double *p1, double *p2, double *q, double *xfbp,
                             double *r, double *grad, double *mc, double *ei)
{
    size_t nn = (size_t)N * N, mn = (size_t)m * n_det;
    double *bx2 = x2 ? x2 : (double *)malloc(sizeof(double) * nn);
    double *bp1 = p1 ? p1 : (double *)malloc(sizeof(double) * mn);
    double *bp2 = p2 ? p2 : (double *)malloc(sizeof(double) * mn);
    double *bq = q ? q : (double *)malloc(sizeof(double) * mn);
    double *bxf = xfbp ? xfbp : (double *)malloc(sizeof(double) * nn);
    double *br = r ? r : (double *)malloc(sizeof(double) * mn);
    double lmc, lei;

    oracle_rotate(x1, bx2, N, g);
    oracle_fwd(bx2, bp2, N, n_det, n_full, idx, m);
    oracle_fwd(x1, bp1, N, n_det, n_full, idx, m);
    if (p2_noise) {  /* REI: the FBP input is p2 + sigma eps */
        double *pn = (double *)malloc(sizeof(double) * mn);
        for (size_t s = 0; s < mn; ++s) pn[s] = bp2[s] + p2_noise[s];
        oracle_ramp(pn, bq, m, n_det);
        free(pn);
    } else {
        oracle_ramp(bp2, bq, m, n_det);
    }
    oracle_adj(bq, bxf, N, n_det, n_full, idx, m, ORACLE_PI / (2.0 * m));
    oracle_residual(bp1, y, idx, m, n_det, bx2, x3_in ? x3_in : bxf, N, &lmc, &lei, br);
    if (grad) oracle_adj(br, grad, N, n_det, n_full, idx, m, 2.0);
    if (mc) *mc = lmc;
    if (ei) *ei = lei;

    if (!x2) free(bx2);
    if (!p1) free(bp1);
    if (!p2) free(bp2);
    if (!q) free(bq);
    if (!xfbp) free(bxf);
    if (!r) free(br);
}

/* --------------------------------------- EI-branch gradient (R16, §8(f) #1) --
 * grad = d ||x2 - x3||^2 / d x1 for x2 = T_g x1 and the identity network
 * x3 = M x2, M = (pi/2m) A_S^T H2 A_S (the sketched FBP of the sketched projection,
 * Alg. 1 step 5 L121; R16).  ei = ||(I - M) T_g x1||^2 and M is symmetric (H2 is an
 * even kernel, A_S^T is the transpose of A_S), so
 *   grad = T_g^T (I - M) d,  d = 2 (x2 - x3),
 * evaluated step by step with the routines above (Eq. 6). */
void oracle_ei_grad(const double *x1, int N, int n_det, int n_full, int g, const int *idx,
                    int m, double *grad)
{
    size_t nn = (size_t)N * N, mn = (size_t)m * n_det;
    double *x2 = (double *)malloc(sizeof(double) * nn);
    double *x3 = (double *)malloc(sizeof(double) * nn);
    double *d = (double *)malloc(sizeof(double) * nn);
    double *md = (double *)malloc(sizeof(double) * nn);
    double *p = (double *)malloc(sizeof(double) * mn);
    oracle_rotate(x1, x2, N, g);
    oracle_fwd(x2, p, N, n_det, n_full, idx, m);
    oracle_fbp(p, x3, N, n_det, n_full, idx, m, m);        /* x3 = M x2 */
    for (size_t i = 0; i < nn; ++i) d[i] = 2.0 * (x2[i] - x3[i]);
    oracle_fwd(d, p, N, n_det, n_full, idx, m);
    oracle_fbp(p, md, N, n_det, n_full, idx, m, m);        /* M d */
    for (size_t i = 0; i < nn; ++i) d[i] -= md[i];        /* (I - M) d */
    oracle_rotate_adj(d, grad, N, g);
    free(x2);
    free(x3);
    free(d);
    free(md);
    free(p);
}

/* ----------------------- Theorem-1 deviation (§8(f) #4) --
 * delta = ||A^T (S^T S - I) A||_2 for the sqrt(n_full/m)-scaled row-subsampling sketch S of
 * the sketched angles idx, i.e. the spectral norm of the symmetric operator
 *   D v = (n_full / m) A_S^T A_S v - A^T A v
 * (A: all n_full angles; the quantity bounding the sketched-vs-full EI regulariser in the
 * proof of Theorem 1), estimated by plain power iteration from v0 (normalised
 * to ||v|| = 1 first): v <- D v / ||D v||, lambda = ||D v|| (of the last iterate). */
void oracle_sketch_deviation(int N, int n_det, int n_full, const int *idx, int m, int iters,
                             const double *v0, double *v_out, double *lambda)
{
    size_t nn = (size_t)N * N;
    int *all = (int *)malloc(sizeof(int) * (size_t)n_full);
    double *v = (double *)malloc(sizeof(double) * nn);
    double *u = (double *)malloc(sizeof(double) * nn);
    double *w = (double *)malloc(sizeof(double) * nn);
    double *pf = (double *)malloc(sizeof(double) * (size_t)n_full * n_det);
    double *ps = (double *)malloc(sizeof(double) * (size_t)m * n_det);
    for (int i = 0; i < n_full; ++i) all[i] = i;
    double s = 0.0;
    for (size_t i = 0; i < nn; ++i) s += v0[i] * v0[i];
    s = sqrt(s);
    for (size_t i = 0; i < nn; ++i) v[i] = v0[i] / s;
    double lam = 0.0;
    for (int it = 0; it < iters; ++it) {
        oracle_fwd(v, pf, N, n_det, n_full, all, n_full);
        oracle_adj(pf, u, N, n_det, n_full, all, n_full, 1.0);          /* A^T A v */
        oracle_fwd(v, ps, N, n_det, n_full, idx, m);
        oracle_adj(ps, w, N, n_det, n_full, idx, m, (double)n_full / m); /* (n_full/m) A_S^T A_S v */
        double nrm = 0.0;
        for (size_t i = 0; i < nn; ++i) {
            w[i] -= u[i];
            nrm += w[i] * w[i];
        }
        lam = sqrt(nrm);
        if (lam == 0.0) break;
        for (size_t i = 0; i < nn; ++i) v[i] = w[i] / lam;
    }
    if (v_out) memcpy(v_out, v, sizeof(double) * nn);
    *lambda = lam;
    free(all);
    free(v);
    free(u);
    free(w);
    free(pf);
    free(ps);
}
