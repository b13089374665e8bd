// Experiment: HBM read bandwidth of streaming patterns on B200 (decode GEMM weight stream).
//  mode 0: TMA 2D boxes {64 K, 256 rows} over a row-major [rows, 4096] bf16 matrix,
//          K blocks fastest inside a 256-row tile (the w1/w3 swap GEMM's access order)
//  mode 1: 1D bulk copies of contiguous 32 KB chunks (a pre-tiled weight layout)
//  mode 2: plain 16-byte LDG grid-stride read (sum)
//  mode 4: TMA 2D boxes {64 K, 128 rows} over a row-major [rows, 14336] bf16 matrix (the
//          w2 layout: 28 KB row stride), 56 K blocks per tile (split-K 4), 16 KB stages
//  mode 3: as mode 0 but whole 2 MB tiles per CTA (tile t -> CTA t % 148), 896 tiles:
//          the decode w1/w3 GEMM's work split (tail: 8 CTAs run a 7th tile)
// 148 persistent CTAs, S-stage mbarrier ring of 32 KB stages (modes 0/1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(n)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n)); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(su(b)), "r"(ph));
}
constexpr int SMAX = 7, STAGE = 32768;
__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap m, int mode, const uint8_t* base,
                                                int64_t nchunks, int nkb, float* sink, int stage_bytes = STAGE,
                                                int box_rows = 256, int nkb_row = 64, int S = 6, int delay = 0) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[SMAX];
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    int64_t i0 = blockIdx.x;
    int issued = 0, done = 0;
    uint32_t acc = 0;
    auto issue = [&](int64_t c) {
        const int st = issued % S;
        expect_tx(&full[st], stage_bytes);
        if (mode == 0 || mode == 3 || mode == 4) {
            // chunk c -> (tile, kb); a tile = box_rows rows x nkb K blocks; tiles walk
            // (row block, K range) with K ranges of nkb blocks inside rows of nkb_row blocks
            const int64_t tile = c / nkb;
            const int kb = (int)(c % nkb);
            const int kr = nkb_row / nkb;  // K ranges per row block
            const int row = (int)(tile / kr) * box_rows, kcol = (int)(tile % kr) * nkb + kb;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(su(smem + st * STAGE)), "l"((uint64_t)&m), "r"(su(&full[st])), "r"(kcol * 64), "r"(row) : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(smem + st * STAGE)), "l"(base + c * stage_bytes), "r"(stage_bytes), "r"(su(&full[st])) : "memory");
        }
        ++issued;
    };
    // chunk sequence of this CTA: mode 3 -> tiles t = blockIdx.x + j*gridDim.x, all nkb chunks each
    const int64_t ntiles = nchunks / nkb;
    const int64_t my_tiles = mode == 3 ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int64_t my_n = mode == 3 ? my_tiles * nkb : (nchunks - i0 + gridDim.x - 1) / gridDim.x;
    auto chunk_of = [&](int64_t j) -> int64_t {
        if (mode == 3) return (blockIdx.x + (j / nkb) * gridDim.x) * nkb + (j % nkb);
        return i0 + j * gridDim.x;
    };
    int64_t j = 0;
    for (int p = 0; p < S && j < my_n; ++p, ++j) issue(chunk_of(j));
    while (done < issued) {
        const int st = done % S;
        wait(&full[st], (done / S) & 1);
        acc += smem[st * STAGE + 7];
        if (delay) {  // emulate the MMA hold time of a stage before it is released
            const long long t0 = clock64();
            while (clock64() - t0 < delay) {}
        }
        ++done;
        if (j < my_n) { issue(chunk_of(j)); ++j; }
    }
    if (acc == 0x12345678) sink[0] = acc;
}
__global__ void k_ldg(const uint4* p, int64_t n, float* sink) {
    uint32_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}
typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const int64_t K = 4096, rows = 256 * 1024;  // 2 GiB bf16
    const int64_t bytes = rows * K * 2;
    uint8_t* d;
    float* sink;
    cudaMalloc(&d, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(d, 1, bytes);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 256}, es[2] = {1, 1};
    ((enc_t)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, SMAX * STAGE + 1024);
    const int nkb = (int)(K / 64);
    const int64_t nchunks = bytes / STAGE;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    CUtensorMap m2;
    const int64_t K2 = 14336, rows2 = bytes / (K2 * 2) / 128 * 128;
    cuuint64_t dims2[2] = {(cuuint64_t)K2, (cuuint64_t)rows2}, str2[1] = {(cuuint64_t)K2 * 2};
    cuuint32_t box2[2] = {64, 128};
    ((enc_t)fn)(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims2, str2, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char* names[6] = {"TMA 2D box {64,256} (GEMM order)", "1D bulk 32 KB contiguous", "LDG.128 grid-stride",
                            "TMA 2D, whole 2 MB tiles per CTA", "TMA 2D {64,128} w2 layout (28KB stride)",
                            "1D bulk 16 KB contiguous"};
    for (int mode = 0; mode < 6; ++mode)
        for (int grid_mul = 1; grid_mul <= (mode == 2 ? 4 : 1); grid_mul *= 2) {
            float best = 1e9;
            for (int rep = 0; rep < 8; ++rep) {
                cudaEventRecord(a);
                if (mode < 2) k_tma<<<148, 128, SMAX * STAGE + 1024>>>(m, mode, d, nchunks, nkb, sink);
                else if (mode == 3) k_tma<<<148, 128, SMAX * STAGE + 1024>>>(m, mode, d, 896LL * nkb, nkb, sink);
                else if (mode == 4) k_tma<<<148, 128, SMAX * STAGE + 1024>>>(m2, 4, d, rows2 / 128 * 224, 56, sink, 16384, 128, 224);
                else if (mode == 5) k_tma<<<148, 128, SMAX * STAGE + 1024>>>(m, 5, d, bytes / 16384, nkb, sink, 16384);
                else k_ldg<<<148 * 8 * grid_mul, 256>>>((const uint4*)d, bytes / 16, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            const double by = mode == 3 ? 896.0 * nkb * STAGE : mode == 4 ? (double)rows2 * K2 * 2 : (double)bytes;
            printf("%-36s grid x%d: %.3f ms  %.1f GB/s  (%s)\n", names[mode], grid_mul, best, by / best / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    // stage-depth / hold-time sweep on the contiguous 32 KB chunk stream (mode 1)
    for (int S = 2; S <= SMAX; ++S)
        for (int delay : {0, 500, 1000}) {
            float best = 1e9;
            for (int rep = 0; rep < 6; ++rep) {
                cudaEventRecord(a);
                k_tma<<<148, 128, SMAX * STAGE + 1024>>>(m, 1, d, nchunks, nkb, sink, STAGE, 256, 64, S, delay);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("mode1 S=%d hold=%4d cycles: %.1f GB/s\n", S, delay, bytes / best / 1e6);
        }
    return 0;
}
