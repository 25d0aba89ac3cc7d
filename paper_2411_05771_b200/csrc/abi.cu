// abi.cu — the extern "C" entry points of include/skei.h: host-side validation,
// plan tables, workspace sizing and the pass orchestration.  Every numeric step runs
// in the kernels of the sibling .cu files.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "internal.h"

#ifndef SKEI_PACK_ONE
#define SKEI_PACK_ONE 1  // groups of 4: one (row-) packed copy per image, columns via a tensor map
#endif

using namespace skei;

namespace {

thread_local char g_cuda_err[256] = "";

skei_status cuda_fail(cudaError_t e) {
    std::snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e),
                  cudaGetErrorString(e));
    return SKEI_ERR_CUDA;
}

#define SKEI_CUDA(call)                        \
    do {                                       \
        cudaError_t e_ = (call);               \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

// Scoped device switch: the library must not change the caller's current device.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

double ramlak2(long n) {  // doubled Ram-Lak kernel h2 (R8)
    if (n == 0) return 0.5;
    if (n % 2 == 0) return 0.0;
    return -2.0 / (M_PI * M_PI * (double)n * (double)n);
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Workspace: [q: B*m*n_det floats][residual partials][4 packed images: x1 rows/cols, x2
// rows/cols, each pack_floats() for the largest image group]
struct WsLayout {
    size_t q, res, pack[4], ctr, mcpart, eipart, fscr, qi, ri, aux, total;
};
WsLayout ws_layout(const skei_plan *plan, int B, int m) {
    WsLayout w;
    size_t off = 0;
    w.q = off;
    off += align256(sizeof(float) * (size_t)B * m * plan->n_det);
    w.res = off;
    off += align256(residual_ws_bytes(plan, B, m));
    size_t pk = 0;
    for (int bb = 1; bb <= 4; bb *= 2) {
        const size_t f = pack_floats(plan, B, bb);
        if (f > pk) pk = f;
    }
    // the job-fused copies (blocks of 16 lines x 2 jobs, one class) span two consecutive slots
    const size_t fused = (size_t)B * ((plan->n + 15) / 16) * plan->n * 32;
    if ((fused + 1) / 2 > pk) pk = (fused + 1) / 2;
    for (int i = 0; i < 4; ++i) {
        w.pack[i] = off;
        off += align256(sizeof(float) * pk);
    }
    w.ctr = off;  // completion counters of the fused reductions + forward split units
    off += align256(sizeof(unsigned) * kPassCounters);
    w.mcpart = off;
    off += align256(sizeof(float) * (size_t)B * fwd_mc_slots(plan, B, m, 0));
    w.eipart = off;
    off += align256(sizeof(float) * adj_ei_part_floats(plan, B));
    w.fscr = off;  // forward split-unit pieces
    off += align256(sizeof(float) * fwd_scratch_floats(plan));
    // interleaved padded q and r for the backprojector's bulk copies (job-fused pass: one
    // buffer of both, spanning qi and ri)
    size_t il = adj_il_floats(plan, B, m);
    if ((adj_fused_floats(plan, B, m) + 1) / 2 > il) il = (adj_fused_floats(plan, B, m) + 1) / 2;
    w.qi = off;
    off += align256(sizeof(float) * il);
    w.ri = off;
    off += align256(sizeof(float) * il);
    w.aux = off;  // skei_sketch_deviation: the full angle list and the fp64 norm partials
    off += align256(sizeof(int32_t) * (size_t)plan->n_full) +
           align256(sizeof(double) * (size_t)B * kNormChunks);
    w.total = off;
    return w;
}
inline float *ws_f(void *ws, size_t off) { return reinterpret_cast<float *>((char *)ws + off); }
// the column-packed copy's workspace slot, or NULL where the forward stages the column class
// from the row-packed copy (groups of 4; radon_fwd.cu, tm_col)
inline float *xc_slot(void *ws, size_t off, int B, int idx_stride) {
    return (SKEI_PACK_ONE && fwd_bb(B, idx_stride) == 4) ? nullptr : ws_f(ws, off);
}

skei_status check_idx_args(const skei_plan *plan, int B, const int32_t *idx, int m,
                           int idx_stride) {
    if (!plan || !idx) return SKEI_ERR_ARG;
    if (B < 1 || m < 1 || m > plan->n_full) return SKEI_ERR_SHAPE;
    if (idx_stride != 0 && idx_stride != m) return SKEI_ERR_ARG;
    return SKEI_OK;
}

}  // namespace

extern "C" {

const char *skei_version(void) { return "skei 0.1 sm_100a"; }

const char *skei_status_string(skei_status s) {
    switch (s) {
        case SKEI_OK: return "ok";
        case SKEI_ERR_SHAPE: return "shape error";
        case SKEI_ERR_CONFIG: return "config error";
        case SKEI_ERR_ARG: return "invalid argument";
        case SKEI_ERR_CUDA: return "CUDA error";
        case SKEI_ERR_NO_DEVICE: return "no usable sm_100 device";
    }
    return "unknown status";
}

const char *skei_last_cuda_error(void) { return g_cuda_err; }

skei_status skei_plan_create(const skei_geometry *geom, int device, skei_plan **out) {
    if (!geom || !out) return SKEI_ERR_ARG;
    *out = nullptr;
    const int n = geom->n, n_det = geom->n_det, n_full = geom->n_full;
    if (n < 2 || n > 1536 || n_det < 1 || n_det > 3072 || n_full < 1 || n_full > 16384)
        return SKEI_ERR_CONFIG;
    int P = geom->fft_len;
    if (P == 0) {
        P = 2;
        while (P < 2 * n_det - 1) P *= 2;
    }
    if (P < 16 && geom->fft_len == 0) P = 16;  // the FFT kernel needs P >= 16
    if (!is_pow2(P) || P < 2 * n_det - 1 || P > 8192 || P < 16) return SKEI_ERR_CONFIG;

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return SKEI_ERR_NO_DEVICE;
    DeviceGuard guard(device);
    if (!guard.ok) return SKEI_ERR_NO_DEVICE;
    cudaDeviceProp prop;
    SKEI_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return SKEI_ERR_NO_DEVICE;  // built for sm_100a only

    // fp64 tables on the host
    std::vector<double2> trig(n_full);
    for (int i = 0; i < n_full; ++i) {
        // theta_i = i*pi/n_full; exact values at 0 and pi/2
        if (2 * i == n_full) {
            trig[i] = make_double2(0.0, 1.0);
        } else {
            double th = M_PI * (double)i / (double)n_full;
            trig[i] = make_double2(std::cos(th), std::sin(th));
        }
    }
    std::vector<float> ramp(P);
    {
        // R[k] = sum_n h_P[n] cos(2 pi k n / P), h_P = h2 wrapped onto P points (even),
        // = 1/2 + 2 sum_{odd l < P/2} h2(l) cos(2 pi k l / P); stored / P (inverse-FFT scale).
        std::vector<double> R(P / 2 + 1);
        for (int k = 0; k <= P / 2; ++k) {
            double acc = 0.5;
            for (int l = 1; l < P / 2; l += 2) {
                long t = ((long)k * l) % P;
                acc += 2.0 * ramlak2(l) * std::cos(2.0 * M_PI * (double)t / (double)P);
            }
            R[k] = acc;
        }
        for (int k = 0; k < P; ++k) ramp[k] = (float)(R[k <= P / 2 ? k : P - k] / (double)P);
    }
    std::vector<double2> rot(360);  // (cos g, sin g), g in degrees; exact at multiples of 90
    for (int g = 0; g < 360; ++g) {
        if (g == 0) rot[g] = make_double2(1.0, 0.0);
        else if (g == 90) rot[g] = make_double2(0.0, 1.0);
        else if (g == 180) rot[g] = make_double2(-1.0, 0.0);
        else if (g == 270) rot[g] = make_double2(0.0, -1.0);
        else rot[g] = make_double2(std::cos(M_PI * g / 180.0), std::sin(M_PI * g / 180.0));
    }
    int npass = 0, radix[kMaxFftPass], ns[kMaxFftPass], twoff[kMaxFftPass], twtotal = 0;
    fft_plan(P, &npass, radix, ns, twoff, &twtotal);
    std::vector<float2> tw(twtotal);
    for (int ip = 0; ip < npass; ++ip)
        for (int k = 0; k < ns[ip]; ++k)
            for (int r = 0; r < radix[ip]; ++r) {
                // exp(-2 pi i r k / (R Ns)), reduced exactly before the fp64 trig; r-major,
                // so the threads of a warp (consecutive k) load consecutive entries
                const long num = ((long)r * k) % ((long)radix[ip] * ns[ip]);
                const double a = 2.0 * M_PI * (double)num / ((double)radix[ip] * ns[ip]);
                tw[twoff[ip] + r * ns[ip] + k] = make_float2((float)std::cos(a), (float)(-std::sin(a)));
            }

    skei_plan *p = new skei_plan();
    p->device = device;
    p->n = n;
    p->n_det = n_det;
    p->n_full = n_full;
    p->fft_len = P;
    p->log2_fft = 0;
    while ((1 << p->log2_fft) < P) ++p->log2_fft;
    p->num_sms = prop.multiProcessorCount < 256 ? prop.multiProcessorCount : 256;  // kPassCounters
    cudaError_t e = cudaMalloc(&p->d_trig, sizeof(double2) * n_full);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_ramp, sizeof(float) * P);
    p->fft_npass = npass;
    for (int i = 0; i < npass; ++i) {
        p->fft_radix[i] = radix[i];
        p->fft_ns[i] = ns[i];
        p->fft_twoff[i] = twoff[i];
    }
    if (e == cudaSuccess) e = cudaMalloc(&p->d_twp, sizeof(float2) * twtotal);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_rot, sizeof(double2) * 360);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_rot, rot.data(), sizeof(double2) * 360, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_trig, trig.data(), sizeof(double2) * n_full, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_ramp, ramp.data(), sizeof(float) * P, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_twp, tw.data(), sizeof(float2) * twtotal, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        skei_plan_destroy(p);
        return cuda_fail(e);
    }
    *out = p;
    return SKEI_OK;
}

void skei_plan_destroy(skei_plan *plan) {
    if (!plan) return;
    DeviceGuard guard(plan->device);
    if (plan->d_trig) cudaFree(plan->d_trig);
    if (plan->d_ramp) cudaFree(plan->d_ramp);
    if (plan->d_twp) cudaFree(plan->d_twp);
    if (plan->d_rot) cudaFree(plan->d_rot);
    delete plan;
}

skei_status skei_plan_geometry(const skei_plan *plan, skei_geometry *out) {
    if (!plan || !out) return SKEI_ERR_ARG;
    out->n = plan->n;
    out->n_det = plan->n_det;
    out->n_full = plan->n_full;
    out->fft_len = plan->fft_len;
    return SKEI_OK;
}

size_t skei_workspace_bytes(const skei_plan *plan, int32_t batch, int32_t m) {
    if (!plan || batch < 1 || m < 1) return 0;
    return ws_layout(plan, batch, m).total;
}

skei_status skei_draw(uint64_t seed, uint64_t iter, uint64_t image, int32_t n_full, int32_t m,
                      int32_t mode, int32_t *g_deg, int32_t *angle_idx) {
    if (!g_deg || !angle_idx) return SKEI_ERR_ARG;
    if (n_full < 1 || m < 1 || m > n_full) return SKEI_ERR_CONFIG;
    if (mode != 0 && mode != 1) return SKEI_ERR_CONFIG;
    if (mode == 0 && n_full % m != 0) return SKEI_ERR_CONFIG;
    return host_draw(seed, iter, image, n_full, m, mode, g_deg, angle_idx) == 0
               ? SKEI_OK
               : SKEI_ERR_CONFIG;
}

skei_status skei_draw_device(uint64_t seed, uint64_t iter, uint64_t image0, int32_t count,
                             int32_t shared, int32_t n_full, int32_t m, int32_t mode,
                             int32_t *g_dev, int32_t *idx_dev, skei_stream stream) {
    if (!g_dev || !idx_dev) return SKEI_ERR_ARG;
    if (count < 1 || (shared && count != 1)) return SKEI_ERR_ARG;
    if (n_full < 1 || n_full > 16384 || m < 1 || m > n_full) return SKEI_ERR_CONFIG;
    if (mode != 0 && mode != 1) return SKEI_ERR_CONFIG;
    if (mode == 0 && n_full % m != 0) return SKEI_ERR_CONFIG;
    SKEI_CUDA(launch_draw(seed, iter, image0, count, shared, n_full, m, mode, g_dev, idx_dev,
                          (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_rotate(const skei_plan *plan, const float *x, float *out, int32_t B,
                        const int32_t *g_deg, int32_t g_stride, skei_stream stream) {
    if (!plan || !x || !out || !g_deg) return SKEI_ERR_ARG;
    if (B < 1) return SKEI_ERR_SHAPE;
    if (g_stride != 0 && g_stride != 1) return SKEI_ERR_ARG;
    if (x == out) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    SKEI_CUDA(launch_rotate(plan, x, out, B, g_deg, g_stride, (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_rotate_adjoint(const skei_plan *plan, const float *y, float *out, int32_t B,
                                const int32_t *g_deg, int32_t g_stride, skei_stream stream) {
    if (!plan || !y || !out || !g_deg) return SKEI_ERR_ARG;
    if (B < 1) return SKEI_ERR_SHAPE;
    if (g_stride != 0 && g_stride != 1) return SKEI_ERR_ARG;
    if (y == out) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    SKEI_CUDA(launch_rotate_adj(plan, y, out, B, g_deg, g_stride, (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_radon_fwd(const skei_plan *plan, const float *x, float *p, int32_t B,
                           const int32_t *idx, int32_t m, int32_t idx_stride, void *ws,
                           size_t ws_bytes, skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!x || !p || !ws) return SKEI_ERR_ARG;
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    const WsLayout w = ws_layout(plan, B, m);
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *ctr = reinterpret_cast<unsigned *>(ws_f(ws, w.ctr));
    float *xc = xc_slot(ws, w.pack[1], B, idx_stride);
    RotPackJob pj{x, nullptr, nullptr, 0, ws_f(ws, w.pack[0]), xc, ctr};
    SKEI_CUDA(launch_rotate_pack(plan, &pj, 1, B, fwd_bb(B, idx_stride), s));
    FwdJob job{ws_f(ws, w.pack[0]), xc, p, nullptr, nullptr};
    const FwdScratch scr{ctr + 2, ws_f(ws, w.fscr)};
    SKEI_CUDA(launch_radon_fwd(plan, &job, 1, B, idx, m, idx_stride, scr, s));
    return SKEI_OK;
}

skei_status skei_radon_adj(const skei_plan *plan, const float *p, float *x, int32_t B,
                           const int32_t *idx, int32_t m, int32_t idx_stride, float scale,
                           skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!x || !p) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    AdjJob job{p, x, scale};
    SKEI_CUDA(launch_radon_adj(plan, &job, 1, B, idx, m, idx_stride, (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_ramp_filter(const skei_plan *plan, const float *p, float *q, int32_t rows,
                             skei_stream stream) {
    if (!plan || !p || !q) return SKEI_ERR_ARG;
    if (rows < 1) return SKEI_ERR_SHAPE;
    DeviceGuard guard(plan->device);
    SKEI_CUDA(launch_ramp(plan, p, q, rows, (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_fbp(const skei_plan *plan, const float *p, float *x, int32_t B,
                     const int32_t *idx, int32_t m, int32_t idx_stride, int32_t m_total,
                     void *ws, size_t ws_bytes, skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!x || !p || !ws) return SKEI_ERR_ARG;
    if (m_total < m) return SKEI_ERR_ARG;
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    float *q = ws_f(ws, ws_layout(plan, B, m).q);
    cudaStream_t s = (cudaStream_t)stream;
    SKEI_CUDA(launch_ramp(plan, p, q, B * m, s));
    AdjJob job{q, x, (float)(M_PI / (2.0 * (double)m_total))};
    SKEI_CUDA(launch_radon_adj(plan, &job, 1, B, idx, m, idx_stride, s));
    return SKEI_OK;
}

skei_status skei_ei_grad(const skei_plan *plan, int32_t B, const float *x2, const float *x3,
                         const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                         int32_t idx_stride, float *grad, void *ws, size_t ws_bytes,
                         skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!x2 || !x3 || !g_deg || !grad || !ws) return SKEI_ERR_ARG;
    if (g_stride != 0 && g_stride != 1) return SKEI_ERR_ARG;
    if (grad == x2 || grad == x3) return SKEI_ERR_ARG;
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    const WsLayout wl = ws_layout(plan, B, m);
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *ctr = reinterpret_cast<unsigned *>(ws_f(ws, wl.ctr));
    // d = 2 (x2 - x3), packed for the forward projector (pack[0..1]) and written (pack[2])
    float *d = ws_f(ws, wl.pack[2]), *u = ws_f(ws, wl.pack[3]);
    float *xc = xc_slot(ws, wl.pack[1], B, idx_stride);
    RotPackJob pj{x2, d, nullptr, 0, ws_f(ws, wl.pack[0]), xc, ctr, x3, 2.0f};
    SKEI_CUDA(launch_rotate_pack(plan, &pj, 1, B, fwd_bb(B, idx_stride), s));
    // M d = (pi/2m) A_S^T ramp(A_S d); u = d - M d
    float *p = ws_f(ws, wl.ri);  // A_S d (the interleaved-r region is free outside the pass)
    FwdJob fj{ws_f(ws, wl.pack[0]), xc, p, nullptr, nullptr};
    const FwdScratch scr{ctr + 2, ws_f(ws, wl.fscr)};
    SKEI_CUDA(launch_radon_fwd(plan, &fj, 1, B, idx, m, idx_stride, scr, s));
    const bool il = fwd_bb(B, idx_stride) == 4 && pick_bb(B, idx_stride) == 4;
    float *q = ws_f(ws, wl.q), *qi = il ? ws_f(ws, wl.qi) : nullptr;
    SKEI_CUDA(launch_ramp(plan, p, q, B * m, s, qi, m, 4));
    AdjJob aj{q, u, (float)(-M_PI / (2.0 * (double)m)), qi, d};
    SKEI_CUDA(launch_radon_adj(plan, &aj, 1, B, idx, m, idx_stride, s));
    // grad = T_g^T u
    SKEI_CUDA(launch_rotate_adj(plan, u, grad, B, g_deg, g_stride, s));
    return SKEI_OK;
}

skei_status skei_backproject_band(const skei_plan *plan, int32_t B, const float *q,
                                  const float *r, const int32_t *idx, int32_t m,
                                  int32_t idx_stride, int32_t m_total, const float *x2,
                                  int32_t row0, int32_t rows, float *xfbp_band,
                                  float *grad_band, float *ei_band, void *ws, size_t ws_bytes,
                                  skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!q || !r || !x2 || !xfbp_band || !grad_band || !ei_band || !ws) return SKEI_ERR_ARG;
    if (m_total < m) return SKEI_ERR_ARG;
    if (row0 < 0 || rows < 1 || row0 + rows > plan->n) return SKEI_ERR_SHAPE;
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    const WsLayout wl = ws_layout(plan, B, m);
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *ctr = reinterpret_cast<unsigned *>(ws_f(ws, wl.ctr));
    SKEI_CUDA(cudaMemsetAsync(ctr + 1, 0, sizeof(unsigned), s));  // the ei completion counter
    AdjJob aj[2] = {{q, xfbp_band, (float)(M_PI / (2.0 * (double)m_total))}, {r, grad_band, 2.0f}};
    AdjEi eif{x2, ws_f(ws, wl.eipart), ctr + 1, ei_band};
    SKEI_CUDA(launch_radon_adj(plan, aj, 2, B, idx, m, idx_stride, s, &eif, row0, rows));
    return SKEI_OK;
}

namespace {
// row band of `rank` when n rows are split over `world` ranks (dist.batch_range)
void band_of(int n, int rank, int world, int *row0, int *rows) {
    const int q = n / world, rem = n - q * world;
    *row0 = rank * q + (rank < rem ? rank : rem);
    *rows = q + (rank < rem ? 1 : 0);
}
}  // namespace

size_t skei_rs_recv_floats(const skei_plan *plan, int32_t B, int32_t world) {
    if (!plan || B < 1 || world < 1) return 0;
    const size_t bmax = ((size_t)plan->n + world - 1) / world;
    return (size_t)world * 2 * B * bmax * plan->n;
}

skei_status skei_backproject_scatter(const skei_plan *plan, int32_t B, const float *q,
                                     const float *r, const int32_t *idx, int32_t m,
                                     int32_t idx_stride, int32_t m_total,
                                     float *const *peer_recv, int32_t world, int32_t rank,
                                     skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!q || !r || !peer_recv || m_total < m) return SKEI_ERR_ARG;
    if (world < 1 || world > kMaxRsPeers || rank < 0 || rank >= world || world > plan->n)
        return SKEI_ERR_ARG;
    AdjRs rs;
    rs.world = world;
    rs.bmax = (plan->n + world - 1) / world;
    const size_t slot = (size_t)2 * B * rs.bmax * plan->n;
    for (int o = 0; o < kMaxRsPeers; ++o) {
        rs.peer[o] = o < world ? peer_recv[o] : nullptr;
        if (o < world && !rs.peer[o]) return SKEI_ERR_ARG;
        if (o < world) rs.peer[o] += (size_t)rank * slot;  // this rank's slot
    }
    DeviceGuard guard(plan->device);
    AdjJob aj[2] = {{q, nullptr, (float)(M_PI / (2.0 * (double)m_total))}, {r, nullptr, 2.0f}};
    SKEI_CUDA(launch_radon_adj(plan, aj, 2, B, idx, m, idx_stride, (cudaStream_t)stream, nullptr,
                               0, -1, false, &rs));
    return SKEI_OK;
}

skei_status skei_band_reduce(const skei_plan *plan, int32_t B, const float *recv, int32_t world,
                             int32_t rank, const float *x2, float *xfbp_band, float *grad_band,
                             float *ei_band, void *ws, size_t ws_bytes, skei_stream stream) {
    if (!plan || !recv || !x2 || !xfbp_band || !grad_band || !ei_band || !ws) return SKEI_ERR_ARG;
    if (B < 1) return SKEI_ERR_SHAPE;
    if (world < 1 || world > kMaxRsPeers || rank < 0 || rank >= world || world > plan->n)
        return SKEI_ERR_ARG;
    if (ws_bytes < skei_workspace_bytes(plan, B, 1)) return SKEI_ERR_ARG;
    int row0, rows;
    band_of(plan->n, rank, world, &row0, &rows);
    DeviceGuard guard(plan->device);
    const WsLayout wl = ws_layout(plan, B, 1);
    SKEI_CUDA(launch_band_reduce(recv, world, B, (plan->n + world - 1) / world, plan->n, row0,
                                 rows, x2, xfbp_band, grad_band, ei_band, ws_f(ws, wl.eipart),
                                 (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_sketch_deviation(const skei_plan *plan, int32_t B, const int32_t *idx,
                                  int32_t m, int32_t idx_stride, int32_t iters, float *v,
                                  float *lambda, void *ws, size_t ws_bytes, skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!v || !lambda || !ws || iters < 1) return SKEI_ERR_ARG;
    const int nf = plan->n_full;
    if (ws_bytes < skei_workspace_bytes(plan, B, nf)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    const WsLayout w = ws_layout(plan, B, nf);  // sized for the full angle set
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *ctr = reinterpret_cast<unsigned *>(ws_f(ws, w.ctr));
    int32_t *all = reinterpret_cast<int32_t *>(ws_f(ws, w.aux));
    double *npart = reinterpret_cast<double *>((char *)ws + w.aux +  // norm partials
                                               align256(sizeof(int32_t) * (size_t)nf));
    float *pf = ws_f(ws, w.q), *ps = ws_f(ws, w.ri);
    float *u = ws_f(ws, w.pack[2]), *dv = ws_f(ws, w.pack[3]);
    const long per = (long)plan->n * plan->n;
    SKEI_CUDA(launch_iota(all, nf, s));
    // v <- v / ||v||
    SKEI_CUDA(launch_sumsq(v, B, per, npart, s));
    SKEI_CUDA(launch_normalise(v, v, B, per, npart, nullptr, plan->num_sms, s));
    const FwdScratch scr{ctr + 2, ws_f(ws, w.fscr)};
    // the packed layout follows each forward's image grouping: per-image sketches (B even)
    // group differently from the shared full angle set, so v is packed again for A_S v
    const bool repack = fwd_bb(B, idx_stride) != fwd_bb(B, 0);
    for (int it = 0; it < iters; ++it) {
        float *xc = xc_slot(ws, w.pack[1], B, 0);
        RotPackJob pj{v, nullptr, nullptr, 0, ws_f(ws, w.pack[0]), xc, ctr};
        SKEI_CUDA(launch_rotate_pack(plan, &pj, 1, B, fwd_bb(B, 0), s));
        FwdJob ff{ws_f(ws, w.pack[0]), xc, pf, nullptr, nullptr};
        SKEI_CUDA(launch_radon_fwd(plan, &ff, 1, B, all, nf, 0, scr, s));   // A v
        if (repack) {
            xc = xc_slot(ws, w.pack[1], B, idx_stride);
            RotPackJob ps_{v, nullptr, nullptr, 0, ws_f(ws, w.pack[0]), xc, ctr};
            SKEI_CUDA(launch_rotate_pack(plan, &ps_, 1, B, fwd_bb(B, idx_stride), s));
        }
        FwdJob fs{ws_f(ws, w.pack[0]), xc, ps, nullptr, nullptr};
        SKEI_CUDA(launch_radon_fwd(plan, &fs, 1, B, idx, m, idx_stride, scr, s));  // A_S v
        AdjJob a1{pf, u, -1.0f};  // u = -A^T A v
        SKEI_CUDA(launch_radon_adj(plan, &a1, 1, B, all, nf, 0, s));
        AdjJob a2{ps, dv, (float)((double)nf / m), nullptr, u};  // D v = u + (n_full/m) A_S^T A_S v
        SKEI_CUDA(launch_radon_adj(plan, &a2, 1, B, idx, m, idx_stride, s));
        SKEI_CUDA(launch_sumsq(dv, B, per, npart, s));
        SKEI_CUDA(launch_normalise(dv, v, B, per, npart, lambda, plan->num_sms, s));
    }
    return SKEI_OK;
}

skei_status skei_ramp_allgather(const skei_plan *plan, int32_t B, const float *p,
                                const float *r, int32_t m_local, int32_t row0, int32_t m_total,
                                float *q_local, float *const *peer_q, float *const *peer_r,
                                int32_t n_peers, skei_stream stream) {
    if (!plan || !p || !r || !q_local || !peer_q || !peer_r) return SKEI_ERR_ARG;
    if (B < 1 || m_local < 1 || row0 < 0 || row0 + m_local > m_total) return SKEI_ERR_SHAPE;
    if (n_peers < 1 || n_peers > kMaxPeers) return SKEI_ERR_ARG;
    RampPeers pr;
    pr.n = n_peers;
    for (int g = 0; g < kMaxPeers; ++g) {
        pr.q[g] = g < n_peers ? peer_q[g] : nullptr;
        pr.r[g] = g < n_peers ? peer_r[g] : nullptr;
        if (g < n_peers && (!pr.q[g] || !pr.r[g])) return SKEI_ERR_ARG;
    }
    pr.m_local = m_local;
    pr.row0 = row0;
    pr.m_total = m_total;
    DeviceGuard guard(plan->device);
    SKEI_CUDA(launch_ramp(plan, p, q_local, B * m_local, (cudaStream_t)stream, nullptr, 0, 0, r,
                          nullptr, 1.f, &pr));
    return SKEI_OK;
}

skei_status skei_fbp_adjoint(const skei_plan *plan, const float *x, float *p, int32_t B,
                             const int32_t *idx, int32_t m, int32_t idx_stride, int32_t m_total,
                             void *ws, size_t ws_bytes, skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!x || !p || !ws) return SKEI_ERR_ARG;
    if (m_total < m) return SKEI_ERR_ARG;
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    const WsLayout w = ws_layout(plan, B, m);
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *ctr = reinterpret_cast<unsigned *>(ws_f(ws, w.ctr));
    float *xc = xc_slot(ws, w.pack[1], B, idx_stride);
    RotPackJob pj{x, nullptr, nullptr, 0, ws_f(ws, w.pack[0]), xc, ctr};
    SKEI_CUDA(launch_rotate_pack(plan, &pj, 1, B, fwd_bb(B, idx_stride), s));
    float *ax = ws_f(ws, w.q);  // A_S x
    FwdJob job{ws_f(ws, w.pack[0]), xc, ax, nullptr, nullptr};
    const FwdScratch scr{ctr + 2, ws_f(ws, w.fscr)};
    SKEI_CUDA(launch_radon_fwd(plan, &job, 1, B, idx, m, idx_stride, scr, s));
    // p = (pi / 2 m_total) ramp(A_S x): the scale folded into the ramp's spectrum
    SKEI_CUDA(launch_ramp(plan, ax, p, B * m, s, nullptr, 0, 0, nullptr, nullptr,
                          (float)(M_PI / (2.0 * (double)m_total))));
    return SKEI_OK;
}

skei_status skei_ei_residual(const skei_plan *plan, const float *p1, const float *y,
                             const int32_t *idx, int32_t m, int32_t idx_stride,
                             const float *x2, const float *x3, int32_t B, float *mc,
                             float *ei, float *r, void *ws, size_t ws_bytes,
                             skei_stream stream) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    const bool do_mc = p1 || y || mc, do_ei = x2 || x3 || ei;
    if (!ws || (!do_mc && !do_ei)) return SKEI_ERR_ARG;
    if (do_mc && (!p1 || !y || !mc)) return SKEI_ERR_ARG;  // the MC part needs all three
    if (do_ei && (!x2 || !x3 || !ei)) return SKEI_ERR_ARG;  // the EI part needs all three
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    void *w = ws_f(ws, ws_layout(plan, B, m).res);
    SKEI_CUDA(launch_residual(plan, do_mc ? p1 : nullptr, y, idx, m, idx_stride,
                              do_ei ? x2 : nullptr, x3, B, do_mc ? mc : nullptr,
                              do_ei ? ei : nullptr, do_mc ? r : nullptr, w, (cudaStream_t)stream));
    return SKEI_OK;
}

namespace {

// REI: the FBP of the EI branch sees p2 + sigma eps (rei.cu)
struct ReiNoise {
    float sigma;
    uint64_t seed, iter, image0;
};

skei_status run_pass(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                     const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                     int32_t idx_stride, const float *x3_in, const skei_pass_outputs *o,
                     void *ws, size_t ws_bytes, cudaEvent_t const *ev, cudaStream_t s,
                     const ReiNoise *rei = nullptr, const skei_draw_spec *draw = nullptr,
                     bool y_sketched = false) {
    skei_status st = check_idx_args(plan, B, idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (!x1 || !y || !g_deg || !o || !ws) return SKEI_ERR_ARG;
    if (!o->x2 || !o->p1 || !o->p2 || !o->q || !o->xfbp || !o->r || !o->grad || !o->mc ||
        !o->ei)
        return SKEI_ERR_ARG;
    if (g_stride != 0 && g_stride != 1) return SKEI_ERR_ARG;
    if (ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    const WsLayout wl = ws_layout(plan, B, m);
    void *wres = ws_f(ws, wl.res);
    // Under stream capture the stage events become external event-record nodes of the
    // graph, so every replay records them (and their elapsed times stay meaningful).
    unsigned ev_flags = cudaEventRecordDefault;
    if (ev) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        SKEI_CUDA(cudaStreamIsCapturing(s, &cs));
        if (cs == cudaStreamCaptureStatusActive) ev_flags = cudaEventRecordExternal;
    }
    auto mark = [&](int i) -> cudaError_t {  // NULL slots are skipped
        return (ev && ev[i]) ? cudaEventRecordWithFlags(ev[i], s, ev_flags) : cudaSuccess;
    };
    const float fbp_scale = (float)(M_PI / (2.0 * m));

    SKEI_CUDA(mark(0));
    // a1 (skei_pass_draw): the draw kernel, followed programmatically by rotate + pack, whose
    // x1 packing overlaps the draw (only the rotation job waits for g)
    if (draw)
        SKEI_CUDA(launch_draw(draw->seed, draw->iter, draw->image0, draw->shared ? 1 : B,
                              draw->shared, plan->n_full, m, draw->mode,
                              const_cast<int32_t *>(g_deg), const_cast<int32_t *>(idx), s));
    unsigned *ctr = reinterpret_cast<unsigned *>(ws_f(ws, wl.ctr));
    // a2: x2 = T_g x1, fused with packing x1 and x2 for the forward projector (and zeroing
    // the completion counters of the fused reductions below)
    // Images that cannot be grouped (per-image sketches, odd B) are projected job-fused: an
    // image's x1 and x2 share its sketch, so they are the two slots of one group of the
    // forward (one set of per-(bin, line) geometry for both), packed together: the fused
    // row-packed copy spans pack[0..1], the column-packed one pack[2..3]
    // Groups of 4 pack only the row-lines copy of x1 and x2: the forward stages the column
    // class from it through a transposing tensor map (half the packing traffic)
    const bool fuse = fwd_bb(B, idx_stride) == 1;
    const bool one = SKEI_PACK_ONE && fwd_bb(B, idx_stride) == 4;
    RotPackJob rj[2] = {
        {x1, nullptr, nullptr, 0, ws_f(ws, wl.pack[0]), one ? nullptr : ws_f(ws, wl.pack[fuse ? 2 : 1]), ctr},
        {x1, o->x2, g_deg, g_stride, ws_f(ws, wl.pack[fuse ? 0 : 2]),
         one ? nullptr : ws_f(ws, wl.pack[fuse ? 2 : 3]), nullptr}};
    SKEI_CUDA(launch_rotate_pack(plan, rj, 2, B, fwd_bb(B, idx_stride), s, draw != nullptr, fuse));
    SKEI_CUDA(mark(1));
    // a3 + a7 (MC part): p1 = A_S x1 with r = p1 - y_S and mc = ||r||^2 fused into its
    // epilogue, and p2 = A_S x2, in one launch
    // with image groups of 4, q and r are also written in the backprojector's interleaved
    // padded layout (its windows are then one bulk copy per angle)
    // (job-fused pass: q and r of an image interleaved as the two slots of one row, one buffer)
    const bool il = fwd_bb(B, idx_stride) == 4 && pick_bb(B, idx_stride) == 4;
    float *qi = il || fuse ? ws_f(ws, wl.qi) : nullptr;
    float *ri = il ? ws_f(ws, wl.ri) : fuse ? qi : nullptr;
    FwdJob fj[2] = {{ws_f(ws, wl.pack[0]), one ? nullptr : ws_f(ws, wl.pack[fuse ? 2 : 1]), o->p1, y, o->r,
                     y_sketched},
                    {ws_f(ws, wl.pack[2]), one ? nullptr : ws_f(ws, wl.pack[3]), o->p2, nullptr, nullptr}};
    FwdMc mcr{ws_f(ws, wl.mcpart), ctr, o->mc};
    const FwdScratch scr{ctr + 2, ws_f(ws, wl.fscr)};
    SKEI_CUDA(launch_radon_fwd(plan, fj, 2, B, idx, m, idx_stride, scr, s, &mcr, fuse));
    SKEI_CUDA(mark(2));
    // a4: q = ramp(p2); the same launch also copies r into the interleaved layout.  REI:
    // q = ramp(p2 + sigma eps), the noisy copy in the workspace (p2 stays noise-free)
    const float *pin = o->p2;
    if (rei) {
        float *pn = ws_f(ws, wl.q);
        SKEI_CUDA(launch_rei_noise(o->p2, pn, B, m, plan->n_det, rei->sigma, rei->seed,
                                   rei->iter, rei->image0, plan->num_sms, s));
        pin = pn;
    }
    SKEI_CUDA(launch_ramp(plan, pin, o->q, B * m, s, qi, m, fuse ? 2 : 4, o->r, ri, 1.f, nullptr, fuse));
    SKEI_CUDA(mark(3));
    // a5 + a8 (+ a7 EI part when x3 is the identity network's x_fbp): x_fbp = (pi/2m) A_S^T q
    // and grad = 2 A_S^T r in one launch, ei = ||x2 - x_fbp||^2 fused into its epilogue
    AdjJob aj[2] = {{o->q, o->xfbp, fbp_scale, qi}, {o->r, o->grad, 2.0f, ri}};
    AdjEi eif{o->x2, ws_f(ws, wl.eipart), ctr + 1, o->ei};
    SKEI_CUDA(launch_radon_adj(plan, aj, 2, B, idx, m, idx_stride, s, x3_in ? nullptr : &eif, 0, -1,
                               fuse));
    SKEI_CUDA(mark(4));
    if (x3_in)  // a7 (EI part) against a caller-provided x3
        SKEI_CUDA(launch_residual(plan, nullptr, nullptr, idx, m, idx_stride, o->x2, x3_in, B,
                                  nullptr, o->ei, nullptr, wres, s));
    SKEI_CUDA(mark(5));
    return SKEI_OK;
}

}  // namespace

skei_status skei_pass(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                      const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                      int32_t idx_stride, const float *x3_in, const skei_pass_outputs *o,
                      void *ws, size_t ws_bytes, skei_stream stream) {
    return run_pass(plan, B, x1, y, g_deg, g_stride, idx, m, idx_stride, x3_in, o, ws, ws_bytes,
                    nullptr, (cudaStream_t)stream);
}

skei_status skei_pass_rei(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                          const int32_t *g_deg, int32_t g_stride, const int32_t *idx, int32_t m,
                          int32_t idx_stride, float sigma, uint64_t noise_seed,
                          uint64_t noise_iter, uint64_t image0, const skei_pass_outputs *out,
                          void *ws, size_t ws_bytes, skei_stream stream) {
    if (!(sigma >= 0.f)) return SKEI_ERR_ARG;
    const ReiNoise rei{sigma, noise_seed, noise_iter, image0};
    return run_pass(plan, B, x1, y, g_deg, g_stride, idx, m, idx_stride, nullptr, out, ws,
                    ws_bytes, nullptr, (cudaStream_t)stream, &rei);
}

skei_status skei_pass_profiled(const skei_plan *plan, int32_t B, const float *x1,
                               const float *y, const int32_t *g_deg, int32_t g_stride,
                               const int32_t *idx, int32_t m, int32_t idx_stride,
                               const skei_pass_outputs *out, void *ws, size_t ws_bytes,
                               void *const *events, int32_t n_events, skei_stream stream) {
    if (!events || n_events < 6) return SKEI_ERR_ARG;
    return run_pass(plan, B, x1, y, g_deg, g_stride, idx, m, idx_stride, nullptr, out, ws,
                    ws_bytes, (cudaEvent_t const *)events, (cudaStream_t)stream);
}

skei_status skei_pass_draw(const skei_plan *plan, int32_t B, const float *x1, const float *y,
                           const skei_draw_spec *draw, int32_t m, int32_t *g_dev,
                           int32_t *idx_dev, const skei_pass_outputs *out, void *ws,
                           size_t ws_bytes, void *const *events, int32_t n_events,
                           skei_stream stream) {
    if (!plan || !draw || !g_dev || !idx_dev) return SKEI_ERR_ARG;
    if (events && n_events < 6) return SKEI_ERR_ARG;
    if (B < 1) return SKEI_ERR_SHAPE;
    if (draw->shared != 0 && draw->shared != 1) return SKEI_ERR_ARG;
    const int n_full = plan->n_full;
    if (m < 1 || m > n_full) return SKEI_ERR_SHAPE;
    if (draw->mode != 0 && draw->mode != 1) return SKEI_ERR_CONFIG;
    if (draw->mode == 0 && n_full % m != 0) return SKEI_ERR_CONFIG;
    const int stride = draw->shared ? 0 : 1;
    return run_pass(plan, B, x1, y, g_dev, stride, idx_dev, m, stride ? m : 0, nullptr, out, ws,
                    ws_bytes, (cudaEvent_t const *)events, (cudaStream_t)stream, nullptr, draw);
}

skei_status skei_smem_probe(float *sink, int32_t blocks, int32_t iters, skei_stream stream) {
    if (!sink || blocks < 1 || iters < 1) return SKEI_ERR_ARG;
    SKEI_CUDA(launch_smem_probe(sink, blocks, iters, (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_l2_probe(const float *buf, int64_t n_floats, float *sink, int32_t blocks,
                          int32_t iters, skei_stream stream) {
    if (!buf || !sink || blocks < 1 || iters < 1 || n_floats < 4 * 1024 || n_floats % 4)
        return SKEI_ERR_ARG;
    if (((uintptr_t)buf & 15) != 0) return SKEI_ERR_ARG;
    SKEI_CUDA(launch_l2_probe(buf, (long)n_floats, sink, blocks, iters, (cudaStream_t)stream));
    return SKEI_OK;
}

skei_status skei_pass_host(const skei_plan *plan, int32_t B, const float *h_x1,
                           const float *h_y, const int32_t *h_g, int32_t g_stride,
                           const int32_t *h_idx, int32_t m, int32_t idx_stride, float *d_x1,
                           float *d_y, int32_t *d_g, int32_t *d_idx,
                           const skei_pass_outputs *o, float *h_mc, float *h_ei,
                           float *h_ystage, void *ws, size_t ws_bytes, skei_stream stream) {
    if (!plan || !h_x1 || !h_y || !h_g || !h_idx || !d_x1 || !d_y || !d_g || !d_idx || !o ||
        !h_mc || !h_ei)
        return SKEI_ERR_ARG;
    skei_status st = check_idx_args(plan, B, h_idx, m, idx_stride);
    if (st != SKEI_OK) return st;
    if (g_stride != 0 && g_stride != 1) return SKEI_ERR_ARG;
    // everything run_pass would reject is rejected here, before the first copy
    if (!ws || ws_bytes < skei_workspace_bytes(plan, B, m)) return SKEI_ERR_ARG;
    if (!o->x2 || !o->p1 || !o->p2 || !o->q || !o->xfbp || !o->r || !o->grad || !o->mc ||
        !o->ei)
        return SKEI_ERR_ARG;
    for (long i = 0; i < (long)m * (idx_stride ? B : 1); ++i)  // host indices: checked here
        if (h_idx[i] < 0 || h_idx[i] >= plan->n_full) return SKEI_ERR_ARG;
    DeviceGuard guard(plan->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t nn = (size_t)plan->n * plan->n, ny = (size_t)plan->n_full * plan->n_det;
    SKEI_CUDA(cudaMemcpyAsync(d_x1, h_x1, sizeof(float) * B * nn, cudaMemcpyHostToDevice, s));
    const int n_det = plan->n_det;
    // Only the m sketched rows of each image's y cross the link, into d_y as y_S
    // [B][m][n_det] (the pass then reads y_S row k of image b for angle idx_b[k]).  With a
    // staging buffer each image's rows (its own sketch when idx_stride = m) are gathered
    // into it and sent as one copy; without one, a shared sketch uses one strided copy of B
    // row blocks per run of consecutive angle indices and per-image sketches copy all of y.
    // Equispaced sketches (uniform mode: idx[k] = idx[0] + k d) need no host gather: the rows
    // of y_S are a pitched sub-array of y, so the copy engine reads them in place — one 3-D
    // copy for a shared sketch (d | n_full: the image stride is a whole number of pitches),
    // one 2-D copy per image for per-image sketches.  The host then only enqueues.
    auto stride_of = [&](const int32_t *ib) -> int {
        if (m < 2) return 0;
        const int d = ib[1] - ib[0];
        if (d < 1) return 0;
        for (int k = 2; k < m; ++k)
            if (ib[k] - ib[k - 1] != d) return 0;
        return d;
    };
    bool pitched = true;
    for (int b = 0; b < (idx_stride ? B : 1) && pitched; ++b) {
        const int d = stride_of(h_idx + (size_t)b * idx_stride);
        pitched = d > 0 && (idx_stride != 0 || plan->n_full % d == 0);
    }
    // small transfers with a staging buffer keep the gather (cfg2, 0.4 MB of rows: the pitched
    // copy's per-row cost on the copy engine outweighs a 30 us gather — e2e 6700 vs 3800
    // passes/s; cfg3, 4.2 MB: host enqueue 0.34 -> 0.05 ms per step at the same step time)
    if (h_ystage && sizeof(float) * (size_t)B * m * n_det < ((size_t)2 << 20)) pitched = false;
    if (const char *e = std::getenv("SKEI_HOST_PITCHED"))  // A/B knob: 0 = always gather
        if (e[0] == '0') pitched = false;
    const bool y_sk = idx_stride == 0 || h_ystage || pitched;
    if (pitched && idx_stride == 0) {
        const int d = stride_of(h_idx);
        cudaMemcpy3DParms cp = {};
        cp.srcPtr = make_cudaPitchedPtr(const_cast<float *>(h_y) + (size_t)h_idx[0] * n_det,
                                        sizeof(float) * d * n_det, sizeof(float) * n_det,
                                        (size_t)(plan->n_full / d));
        cp.dstPtr = make_cudaPitchedPtr(d_y, sizeof(float) * n_det, sizeof(float) * n_det, (size_t)m);
        cp.extent = make_cudaExtent(sizeof(float) * n_det, (size_t)m, (size_t)B);
        cp.kind = cudaMemcpyHostToDevice;
        SKEI_CUDA(cudaMemcpy3DAsync(&cp, s));
    } else if (pitched) {
        for (int b = 0; b < B; ++b) {
            const int32_t *ib = h_idx + (size_t)b * idx_stride;
            SKEI_CUDA(cudaMemcpy2DAsync(d_y + (size_t)b * m * n_det, sizeof(float) * n_det,
                                        h_y + (size_t)b * ny + (size_t)ib[0] * n_det,
                                        sizeof(float) * stride_of(ib) * n_det,
                                        sizeof(float) * n_det, (size_t)m, cudaMemcpyHostToDevice, s));
        }
    } else if (h_ystage) {
        auto gather = [=](int b0, int b1) {
            for (int b = b0; b < b1; ++b) {
                const int32_t *ib = h_idx + (size_t)b * idx_stride;
                for (int k = 0; k < m;) {
                    int e = k + 1;
                    while (e < m && ib[e] == ib[e - 1] + 1) ++e;
                    std::memcpy(h_ystage + ((size_t)b * m + k) * n_det,
                                h_y + (size_t)b * ny + (size_t)ib[k] * n_det,
                                sizeof(float) * (e - k) * n_det);
                    k = e;
                }
            }
        };
        // large batches (cfg4: 33 MB of rows) are gathered by a few host threads
        const size_t bytes = sizeof(float) * (size_t)B * m * n_det;
        const int nt = (int)std::min<size_t>({(size_t)B, (size_t)8, bytes / (4u << 20) + 1});
        if (nt <= 1) {
            gather(0, B);
        } else {
            std::vector<std::thread> th;
            for (int t = 1; t < nt; ++t)
                th.emplace_back(gather, (int)((long)B * t / nt), (int)((long)B * (t + 1) / nt));
            gather(0, B / nt);
            for (auto &t : th) t.join();
        }
        SKEI_CUDA(cudaMemcpyAsync(d_y, h_ystage, bytes, cudaMemcpyHostToDevice, s));
    } else if (y_sk) {
        for (int k = 0; k < m;) {
            int e = k + 1;
            while (e < m && h_idx[e] == h_idx[e - 1] + 1) ++e;
            SKEI_CUDA(cudaMemcpy2DAsync(d_y + (size_t)k * n_det, sizeof(float) * m * n_det,
                                        h_y + (size_t)h_idx[k] * n_det, sizeof(float) * ny,
                                        sizeof(float) * (e - k) * n_det, B,
                                        cudaMemcpyHostToDevice, s));
            k = e;
        }
    } else {
        SKEI_CUDA(cudaMemcpyAsync(d_y, h_y, sizeof(float) * B * ny, cudaMemcpyHostToDevice, s));
    }
    SKEI_CUDA(cudaMemcpyAsync(d_g, h_g, sizeof(int32_t) * (g_stride ? B : 1),
                              cudaMemcpyHostToDevice, s));
    SKEI_CUDA(cudaMemcpyAsync(d_idx, h_idx, sizeof(int32_t) * (size_t)m * (idx_stride ? B : 1),
                              cudaMemcpyHostToDevice, s));
    st = run_pass(plan, B, d_x1, d_y, d_g, g_stride, d_idx, m, idx_stride, nullptr, o, ws,
                  ws_bytes, nullptr, s, nullptr, nullptr, y_sk);
    if (st != SKEI_OK) return st;
    SKEI_CUDA(cudaMemcpyAsync(h_mc, o->mc, sizeof(float) * B, cudaMemcpyDeviceToHost, s));
    SKEI_CUDA(cudaMemcpyAsync(h_ei, o->ei, sizeof(float) * B, cudaMemcpyDeviceToHost, s));
    return SKEI_OK;
}

}  // extern "C"
