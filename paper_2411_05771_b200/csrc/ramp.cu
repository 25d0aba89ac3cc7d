// ramp.cu — a4: q = h2 (*) p row by row (doubled Ram-Lak kernel, R8), as the
// north_star's "batched zero-padded real FFT-multiply kernel".
//
// Two real rows are packed into one complex sequence z = p_a + i p_b, zero-padded to
// P >= 2 n_det - 1 (so the circular convolution equals the linear one on the first n_det
// outputs).  Because the spectrum R[k] is real and even,
// IFFT(R . FFT(z)) = (h2 (*) p_a) + i (h2 (*) p_b): no un-packing twiddles.
//
// The FFT is a Stockham autosort transform of radix-16 passes plus one final pass of the
// remaining factor (8, 4 or 2); each thread holds 16 complex values (one radix-16
// butterfly, or 16/R radix-R butterflies) in registers:
//   pass (R, Ns): for j < P/R, k = j mod Ns: v_r = z[j + r P/R] w^(r k), w = e^(-2 pi i /
//   (R Ns)); y = DFT_R(v); z'[(j - k) R + k + q Ns] = y_q.
// One CTA = one packed pair of rows, P/16 threads.  Passes exchange through one padded
// shared-memory buffer in place (element e at e + e/16: conflict-free for the strides of
// every pass); the first pass reads the rows straight from global memory, the spectrum is
// multiplied by R[k]/P as the inverse transform loads it, and the last inverse pass writes
// the two output rows straight to global memory.  Twiddles w^(rk) come from per-pass plan
// tables computed in fp64 and rounded once (no recurrences, no fast intrinsics), stored
// r-major so a warp's loads are coalesced; the in-register DFT uses the exact 16th roots of
// unity as literals.  Each pass's mode and direction are template parameters.
#include "internal.h"

namespace skei {
namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ int pad(int e) { return e + (e >> 4); }

// cos / sin of 2 pi t / 16, t = 0..7
__device__ __constant__ float kC16[8] = {1.0f, 0.92387953251128674f, 0.70710678118654757f,
                                         0.38268343236508978f, 0.0f, -0.38268343236508978f,
                                         -0.70710678118654757f, -0.92387953251128674f};
__device__ __constant__ float kS16[8] = {0.0f, 0.38268343236508978f, 0.70710678118654757f,
                                         0.92387953251128674f, 1.0f, 0.92387953251128674f,
                                         0.70710678118654757f, 0.38268343236508978f};

// In-register DFT of size R: y_q = sum_r v_r exp(-+2 pi i q r / R) (iterative radix-2,
// bit-reversed inputs, natural-order outputs).
template <int R, bool inverse>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
    constexpr int L = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        int r = 0;
#pragma unroll
        for (int b = 0; b < L; ++b) r |= ((i >> b) & 1) << (L - 1 - b);
        if (r > i) {
            const float2 t = v[i];
            v[i] = v[r];
            v[r] = t;
        }
    }
#pragma unroll
    for (int s = 1; s <= L; ++s) {
        const int m = 1 << s, h = m >> 1;
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
            const int t = jj * (16 / m);  // angle 2 pi t / 16
            const float wr = kC16[t];
            const float wi = inverse ? kS16[t] : -kS16[t];
#pragma unroll
            for (int k = 0; k < R; k += m) {
                const float2 a = v[k + jj], b = v[k + jj + h];
                float2 tb;
                if (jj == 0) {
                    tb = b;
                } else if (4 * jj == m) {  // w = -+i
                    tb = inverse ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
                } else {
                    tb = make_float2(fmaf(b.x, wr, -b.y * wi), fmaf(b.x, wi, b.y * wr));
                }
                v[k + jj] = make_float2(a.x + tb.x, a.y + tb.y);
                v[k + jj + h] = make_float2(a.x - tb.x, a.y - tb.y);
            }
        }
    }
}

struct RampArgs {
    const float *p;
    float *q;
    int rows, n_det, P;
    const float *R;    // [P] spectrum / P
    float rscale;      // output scale (folded into the spectrum as it is applied; 1 = none)
    const float2 *tw;  // per-pass twiddle tables [k][r], k < Ns, r < R
    int npass;
    // optional interleaved copy for the backprojector's bulk window copies:
    // row (b, k) of q -> qi[b / BB][k][kAdjPad + j][b % BB], zero pads of kAdjPad bins on
    // both sides (rows of width wp = n_det + 2 kAdjPad)
    float *qi;
    int m, bb, wp;
    // fused (the job-fused pass, one image per group): q and r of image b are the two slots of
    // one interleaved row, qi[b][k][kAdjPad + j][slot] (slot 0 = q, 1 = r), rows of even width
    // wp so that every 16-byte-aligned window start is an even bin
    int fused;
    // optional: CTAs nramp.. copy the residual r [B][m][n_det] into the same interleaved
    // layout (one CTA per (image group of 4, angle): 16-byte stores)
    const float *rs;
    float *ri;
    int nramp;
    // optional peer outputs (the fused all-gather of the single-image angle split, SURVEY
    // §8(f) #2): local row (b, k) of q — and, by CTAs nramp.., of rs — is also stored into
    // row (b, row0 + k) of every peer's [B][m_total][n_det] buffer (P2P stores over
    // NVLink; one of the peers is this GPU's own buffer)
    float *pq[kMaxPeers];
    float *pr[kMaxPeers];
    int npeer, m_local, row0, m_total;
};
__device__ __forceinline__ float *il_row(const RampArgs &a, int row) {
    const int b = row / a.m, k = row - b * a.m;
    if (a.fused) return a.qi + ((long)row * a.wp + kAdjPad) * 2;  // slot 0 of row (b, k)
    return a.qi + ((long)((b / a.bb) * a.m + k) * a.wp + kAdjPad) * a.bb + b % a.bb;
}

// One Stockham pass (in place on z): J = 16/R butterflies per thread.  Compile-time mode
// flags (with the direction, so each pass instance carries only its own branches):
// kIn = read the two input rows from global (first forward pass), kScale = multiply by
// R[i] as loaded (first inverse pass), kOut = write the two output rows to global (last
// inverse pass); otherwise smem -> smem.
constexpr int kIn = 1, kScale = 2, kOut = 4;
template <int R, bool PEERS, int mode, bool inverse>
__device__ __forceinline__ void pass(float2 *z, const RampArgs &a, int ip,
                                     const float *pa, const float *pb, float *qa, float *qb, float *ia, float *ib,
                                     long peer_a, long peer_b) {
    constexpr int J = 16 / R;
    // every pass before `ip` is radix 16: Ns = 16^ip, table offset = sum_{i<ip} 16 * 16^i
    const int Ns = 1 << (4 * ip), stride = a.P / R;
    const float2 *tw = a.tw + 16 * (Ns - 1) / 15;
    float2 v[J][R];
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        const int j = threadIdx.x + jj * blockDim.x;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = j + r * stride;
            if (mode & kIn) {
                v[jj][r] = i < a.n_det ? make_float2(__ldg(pa + i), pb ? __ldg(pb + i) : 0.f)
                                       : make_float2(0.f, 0.f);
            } else {
                v[jj][r] = z[pad(i)];
                if (mode & kScale) {
                    const float s = __ldg(a.R + i) * a.rscale;
                    v[jj][r].x *= s;
                    v[jj][r].y *= s;
                }
            }
        }
    }
    if (!(mode & kIn)) __syncthreads();  // every read of this pass precedes every write
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        const int j = threadIdx.x + jj * blockDim.x;
        const int k = j & (Ns - 1);
        if (Ns > 1) {  // twiddles r-major: a warp's consecutive k load consecutive entries
            const float2 *t = tw + k;
#pragma unroll
            for (int r = 1; r < R; ++r)
                v[jj][r] = inverse ? cmulc(v[jj][r], __ldg(t + (long)r * Ns))
                                   : cmul(v[jj][r], __ldg(t + (long)r * Ns));
        }
        dft<R, inverse>(v[jj]);
        const int d = (j - k) * R + k;
        if (mode & kOut) {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int o = d + q * Ns;
                if (o < a.n_det) {
                    qa[o] = v[jj][q].x;
                    if (qb) qb[o] = v[jj][q].y;
                    if (ia) {
                        ia[(long)o * a.bb] = v[jj][q].x;
                        if (ib) ib[(long)o * a.bb] = v[jj][q].y;
                    }
                    if constexpr (PEERS) {
#pragma unroll 1
                        for (int g = 0; g < a.npeer; ++g) {
                            a.pq[g][peer_a + o] = v[jj][q].x;
                            if (qb) a.pq[g][peer_b + o] = v[jj][q].y;
                        }
                    }
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < R; ++q) z[pad(d + q * Ns)] = v[jj][q];
        }
    }
    if (!(mode & kOut)) __syncthreads();
}

// MAXT: P/16 <= MAXT threads; MINB: resident CTAs per SM the register budget must allow
template <int RL, int MAXT, int MINB, bool PEERS>
__global__ void __launch_bounds__(MAXT, MINB) k_ramp(RampArgs a) {
    extern __shared__ float2 z[];
    // global row of local row `row` in the peers' [B][m_total][n_det] buffers
    auto peer_off = [&](int row) -> long {
        const int b = row / a.m_local, k = row - b * a.m_local;
        SKEI_DCHECK(a.row0 + k < a.m_total && a.row0 >= 0, "ramp peer row");
        return ((long)b * a.m_total + a.row0 + k) * a.n_det;
    };
    if (PEERS && (int)blockIdx.x >= a.nramp) {  // copy local r row u to every peer
        const int u = blockIdx.x - a.nramp;
        const float *src = a.rs + (long)u * a.n_det;
        const long off = peer_off(u);
        for (int j = threadIdx.x; j < a.n_det; j += blockDim.x) {
            const float v = __ldg(src + j);
#pragma unroll 1
            for (int g = 0; g < a.npeer; ++g) a.pr[g][off + j] = v;
        }
        return;
    }
    if ((int)blockIdx.x >= a.nramp && a.fused) {  // r row u into slot 1 of the fused rows
        const int u = blockIdx.x - a.nramp;
        const float *src = a.rs + (long)u * a.n_det;
        float *dst = a.ri + (long)u * a.wp * 2 + 1;
        for (int o = threadIdx.x; o < a.wp; o += blockDim.x) {
            const int j = o - kAdjPad;
            dst[(long)o * 2] = (j >= 0 && j < a.n_det) ? __ldg(src + j) : 0.f;
        }
        return;
    }
    if ((int)blockIdx.x >= a.nramp) {  // interleave r: group g = u / m of 4 images, angle k
        const int u = blockIdx.x - a.nramp, g = u / a.m, k = u - g * a.m;
        const long stride = (long)a.m * a.n_det;  // between images
        const float *src = a.rs + ((long)(4 * g) * a.m + k) * a.n_det;
        float4 *dst = reinterpret_cast<float4 *>(a.ri) + (long)u * a.wp;
        for (int o = threadIdx.x; o < a.wp; o += blockDim.x) {
            const int j = o - kAdjPad;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (j >= 0 && j < a.n_det)
                v = make_float4(__ldg(src + j), __ldg(src + stride + j), __ldg(src + 2 * stride + j),
                                __ldg(src + 3 * stride + j));
            dst[o] = v;
        }
        return;
    }
    const int ra = 2 * blockIdx.x, rb = ra + 1;
    const bool has_b = rb < a.rows;
    const float *pa = a.p + (long)ra * a.n_det;
    const float *pb = has_b ? a.p + (long)rb * a.n_det : nullptr;
    float *qa = a.q + (long)ra * a.n_det;
    float *qb = has_b ? a.q + (long)rb * a.n_det : nullptr;
    float *ia = a.qi ? il_row(a, ra) : nullptr;
    float *ib = a.qi && has_b ? il_row(a, rb) : nullptr;
    const long pa_off = PEERS ? peer_off(ra) : 0, pb_off = PEERS && has_b ? peer_off(rb) : 0;
    const int last = a.npass - 1;
#define SKEI_PASS(RV, MODE, INV, IP) \
    pass<RV, PEERS, MODE, INV>(z, a, IP, pa, pb, qa, qb, ia, ib, pa_off, pb_off)
    if (last == 0) {  // a single pass each way (P <= 16)
        SKEI_PASS(RL, kIn, false, 0);
        SKEI_PASS(RL, kOut | kScale, true, 0);
    } else {
        // forward: radix-16 passes (the first reads the rows from global) then the RL pass
        SKEI_PASS(16, kIn, false, 0);
        for (int ip = 1; ip < last; ++ip) SKEI_PASS(16, 0, false, ip);
        SKEI_PASS(RL, 0, false, last);
        // inverse of R . FFT(z): the first pass scales by R[k], the last writes the rows
        SKEI_PASS(16, kScale, true, 0);
        for (int ip = 1; ip < last; ++ip) SKEI_PASS(16, 0, true, ip);
        SKEI_PASS(RL, kOut, true, last);
    }
#undef SKEI_PASS
    if (ia) {  // the zero pads of the interleaved rows (fused rows: up to the even width)
        const int npad = a.wp - a.n_det;
        for (int t = threadIdx.x; t < npad; t += blockDim.x) {
            const int o = t < kAdjPad ? t - kAdjPad : a.n_det + (t - kAdjPad);
            ia[(long)o * a.bb] = 0.f;
            if (ib) ib[(long)o * a.bb] = 0.f;
        }
    }
}

}  // namespace

// Pass plan of a P-point transform (P a power of two >= 16): radix-16 passes, then one
// pass of the remaining factor 8, 4 or 2.  Twiddle table offsets are in complex entries.
void fft_plan(int P, int *npass, int *radix, int *ns, int *twoff, int *twtotal) {
    int n = 0, Ns = 1, off = 0;
    int rem = P;
    while (rem >= 16) {
        radix[n] = 16;
        ns[n] = Ns;
        twoff[n] = off;
        off += 16 * Ns;
        Ns *= 16;
        rem /= 16;
        ++n;
    }
    if (rem > 1) {  // final pass of 8, 4 or 2
        radix[n] = rem;
        ns[n] = Ns;
        twoff[n] = off;
        off += rem * Ns;
        ++n;
    }
    *npass = n;
    *twtotal = off;
}

cudaError_t launch_ramp(const skei_plan *plan, const float *p, float *q, int rows,
                        cudaStream_t s, float *qi, int m, int bb, const float *rs, float *ri,
                        float rscale, const RampPeers *peers, bool fused) {
    RampArgs a;
    a.fused = fused ? 1 : 0;
    a.npeer = peers ? peers->n : 0;
    for (int g = 0; g < kMaxPeers; ++g) {
        a.pq[g] = peers && g < peers->n ? peers->q[g] : nullptr;
        a.pr[g] = peers && g < peers->n ? peers->r[g] : nullptr;
    }
    a.m_local = peers ? peers->m_local : 1;
    a.row0 = peers ? peers->row0 : 0;
    a.m_total = peers ? peers->m_total : 1;
    a.rs = rs;
    a.ri = ri;
    a.qi = qi;
    a.m = m > 0 ? m : 1;
    a.bb = bb > 0 ? bb : 1;
    a.wp = fused ? adj_fused_wp(plan) : plan->n_det + 2 * kAdjPad;
    if (fused) a.bb = 2;
    a.p = p;
    a.q = q;
    a.rows = rows;
    a.n_det = plan->n_det;
    a.P = plan->fft_len;
    a.R = plan->d_ramp;
    a.rscale = rscale;
    a.tw = plan->d_twp;
    a.npass = plan->fft_npass;
    const int RL = plan->fft_radix[plan->fft_npass - 1];
    const size_t smem = sizeof(float2) * (size_t)(a.P + a.P / 16);
    const int threads = a.P / 16;
    a.nramp = (rows + 1) / 2;
    // + the interleaving CTAs of r (rows / m images in groups of 4, m angles each), or with
    // peers the CTAs that copy each local r row to the peers
    const bool pe = peers && peers->n > 0;
    const int grid = a.nramp + (pe ? (rs ? rows : 0)
                                   : (ri && rs ? (fused ? rows : (rows / a.m / 4) * a.m) : 0));
    cudaError_t e = cudaSuccess;
#define SKEI_RAMP_LAUNCH4(RLV, MT, MB, PE)                                                      \
    do {                                                                                        \
        if (smem > 48 * 1024)                                                                   \
            e = cudaFuncSetAttribute(k_ramp<RLV, MT, MB, PE>,                                   \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
        if (e == cudaSuccess) k_ramp<RLV, MT, MB, PE><<<grid, threads, smem, s>>>(a);          \
    } while (0)
#define SKEI_RAMP_LAUNCH3(RLV, MT, MB)                  \
    do {                                                \
        if (pe)                                         \
            SKEI_RAMP_LAUNCH4(RLV, MT, MB, true);       \
        else                                            \
            SKEI_RAMP_LAUNCH4(RLV, MT, MB, false);      \
    } while (0)
    // small transforms (P <= 2048, <= 128 threads): <= 64 registers so 8 CTAs fit an SM
#define SKEI_RAMP_LAUNCH(RLV)                      \
    do {                                           \
        if (threads <= 128)                        \
            SKEI_RAMP_LAUNCH3(RLV, 128, 6);        \
        else                                       \
            SKEI_RAMP_LAUNCH3(RLV, 512, 1);        \
    } while (0)
    switch (RL) {
        case 16: SKEI_RAMP_LAUNCH(16); break;
        case 8: SKEI_RAMP_LAUNCH(8); break;
        case 4: SKEI_RAMP_LAUNCH(4); break;
        default: SKEI_RAMP_LAUNCH(2); break;
    }
#undef SKEI_RAMP_LAUNCH
#undef SKEI_RAMP_LAUNCH3
#undef SKEI_RAMP_LAUNCH4
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace skei
