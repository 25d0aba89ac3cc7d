// tma_transpose_probe.cu — diagnostic: can the forward projector stage its COLUMN-class line
// blocks from the ROW-packed copy with a 4-D TMA tensor map (16-byte innermost runs, a
// transposing box), so that rotate + pack writes one packed copy per image instead of two?
// Compares L2 -> shared staging throughput of (a) the current contiguous bulk copies and
// (b) the transposing tensor-map loads, and checks (b)'s layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tp tools/tma_transpose_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

constexpr int N = 512, R = 8, NB = N / R, G = 4;  // 4 image groups of 4 images
constexpr int BLK_B = N * 128;                     // one packed block (8 lines x 4 images)

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(b)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void bar_tx(uint64_t *b, unsigned n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned ph) {
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su(b)),
        "r"(ph)
        : "memory");
}

// a CTA's stream: blocks b = blockIdx.x + j gridDim.x (mod nblocks), iters passes; 3 buffers,
// block j + 3 issued into the buffer of block j once every thread has read it
template <bool TMAP>
__device__ void stream(const char *src, const CUtensorMap *tm, int nblocks, int iters, float *sink,
                       float *dump, int dump_block) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[3];
    const int per = (nblocks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int total = per * iters;
    auto blk = [&](int j) { return (int)blockIdx.x + (j % per) * (int)gridDim.x; };
    auto issue = [&](int j) {
        const int s = j % 3, b = blk(j);
        bar_tx(&bar[s], BLK_B);
        if (TMAP) {
            const int q = b / NB, cb = b % NB;
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
                    su(sm + s * BLK_B)),
                "l"(tm), "r"(0), "r"(cb * 8), "r"(0), "r"(q * NB), "r"(su(&bar[s]))
                : "memory");
        } else {
            for (int off = 0; off < BLK_B; off += 32768)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        su(sm + s * BLK_B + off)),
                    "l"(src + (long)b * BLK_B + off), "r"(32768), "r"(su(&bar[s]))
                    : "memory");
        }
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) bar_init(&bar[i]);
        for (int j = 0; j < 3 && j < total; ++j) issue(j);
    }
    __syncthreads();
    float acc = 0.f;
    for (int j = 0; j < total; ++j) {
        const int s = j % 3;
        bar_wait(&bar[s], (j / 3) & 1);
        acc += ((float *)(sm + s * BLK_B))[threadIdx.x];
        if (dump && j < per && blk(j) == dump_block)
            for (int i = threadIdx.x; i < BLK_B / 4; i += blockDim.x) dump[i] = ((float *)(sm + s * BLK_B))[i];
        __syncthreads();
        if (threadIdx.x == 0 && j + 3 < total) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(j + 3);
        }
    }
    if (acc == 12345.f) *sink = acc;
}
__global__ void k_bulk(const char *src, int nblocks, int iters, float *sink) {
    stream<false>(src, nullptr, nblocks, iters, sink, nullptr, -1);
}
__global__ void k_tmap(const __grid_constant__ CUtensorMap tm, int nblocks, int iters, float *sink,
                       float *dump, int dump_block) {
    stream<true>(nullptr, &tm, nblocks, iters, sink, dump, dump_block);
}

int main() {
    const size_t bytes = (size_t)G * NB * BLK_B;  // 16.8 MB: one class copy of 4 groups
    // row-packed: value(q, b, c, l, img) at ((q NB + b) N + c) 32 + l 4 + img
    std::vector<float> h(bytes / 4);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000003);
    char *d;
    float *sink, *dump;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMalloc(&dump, BLK_B));
    CK(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult qr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &qr));
    CUtensorMap tm;
    // dims innermost first: img (4 floats), column c (N, stride 128 B), line l (8, stride 16 B),
    // row block (G NB, stride N 128 B)
    cuuint64_t dims[4] = {4, (cuuint64_t)N, 8, (cuuint64_t)G * NB};
    cuuint64_t strides[3] = {128, 16, (cuuint64_t)N * 128};
    cuuint32_t box[4] = {4, 8, 8, (cuuint32_t)NB};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("cuTensorMapEncodeTiled (decreasing strides) -> %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;

    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int smem = 3 * BLK_B;
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_tmap, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int nblocks = G * NB, iters = 40;  // 40 x 16.8 MB = 671 MB staged (~ one forward's)
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int rep = 0; rep < 3; ++rep) {
        float ms;
        CK(cudaEventRecord(e0));
        k_bulk<<<nsm, 256, smem>>>(d, nblocks, iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("bulk   : %.1f us, %.2f TB/s\n", ms * 1e3, (double)bytes * iters / ms / 1e9);
        CK(cudaEventRecord(e0));
        k_tmap<<<nsm, 256, smem>>>(tm, nblocks, iters, sink, dump, 2 * NB + 17);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("tensor : %.1f us, %.2f TB/s\n", ms * 1e3, (double)bytes * iters / ms / 1e9);
    }
    CK(cudaGetLastError());
    // layout check: column block (q = 5 / NB... ) dump_block = q NB + cb with q = 5 / 64 -> use q, cb
    std::vector<float> hd(BLK_B / 4);
    CK(cudaMemcpy(hd.data(), dump, BLK_B, cudaMemcpyDeviceToHost));
    const int qd = (2 * NB + 17) / NB, cbd = (2 * NB + 17) % NB;
    long bad = 0;
    for (int rr = 0; rr < N; ++rr)
        for (int cc = 0; cc < 8; ++cc)
            for (int im = 0; im < 4; ++im) {
                // shared [r][col][img] <- row-packed (q, b = r / 8, c = 8 cb + col, l = r % 8, img)
                const size_t src = ((size_t)(qd * NB + rr / 8) * N + (8 * cbd + cc)) * 32 + (rr % 8) * 4 + im;
                if (hd[((size_t)rr * 8 + cc) * 4 + im] != h[src]) ++bad;
            }
    printf("layout check: %ld mismatches of %d\n", bad, N * 32);
    return 0;
}
