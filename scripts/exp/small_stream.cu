// Experiment: efficiency of SHORT single-wave weight streams (the per-rank decode GEMMs at
// EP8 / TP8: 112 CTAs x one 2 MB weight tile each, ~40 us). G CTAs each stream a contiguous
// region of B bytes with 1D bulk copies of 32 KB (S-stage mbarrier ring, like the GEMMs'
// producer); the consumer releases stages immediately. Prints time and GB/s per (G, B), so
// the fixed cost (launch, first-byte latency, tail) can be read off as the intercept.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o small_stream small_stream.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int S = 6, STAGE = 32768;
__global__ void __launch_bounds__(64, 1) k_stream(const uint8_t* base, int64_t per_cta, float* sink, int interleave) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[S];
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    // contiguous: CTA i owns bytes [i * per_cta, (i+1) * per_cta); interleaved: CTA i reads
    // chunks i, i + G, i + 2G, ... (the CTAs sweep one region together)
    const uint8_t* src = interleave ? base + blockIdx.x * (int64_t)STAGE : base + blockIdx.x * per_cta;
    const int64_t step = interleave ? (int64_t)gridDim.x * STAGE : STAGE;
    const int64_t n = per_cta / STAGE;
    int64_t issued = 0, done = 0;
    uint32_t acc = 0;
    auto issue = [&]() {
        const int st = issued % S;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(STAGE));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su(smem + st * STAGE)), "l"(src + issued * step), "r"(STAGE), "r"(su(&full[st])) : "memory");
        ++issued;
    };
    while (issued < n && issued < S) issue();
    while (done < n) {
        const int st = done % S;
        const uint32_t ph = (done / S) & 1;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(su(&full[st])), "r"(ph));
        acc += smem[st * STAGE + 7];
        ++done;
        if (issued < n) issue();
    }
    if (acc == 0x12345678) sink[0] = acc;
}
int main() {
    const int64_t bytes = 3LL << 30;
    uint8_t* d;
    float* sink;
    cudaMalloc(&d, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(d, 1, bytes);
    uint8_t* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, S * STAGE + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int il = 0; il < 2; ++il)
    for (int G : {112, 128, 148})
        for (int64_t mb : {1, 2, 4, 8, 16}) {
            const int64_t per = mb << 20;
            float best = 1e9;
            for (int rep = 0; rep < 10; ++rep) {
                cudaMemsetAsync(flush, rep, 256 << 20);  // evict the previous pass from L2
                const int64_t off = ((rep % 3) * (int64_t)G * per) % (bytes - G * per);
                cudaEventRecord(a);
                k_stream<<<G, 64, S * STAGE + 1024>>>(d + off / 4096 * 4096, per, sink, il);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("%s G=%3d per_cta=%2lld MB total=%5lld MB: %8.2f us  %7.1f GB/s  (%s)\n", il ? "interleaved" : "contiguous ", G, (long long)mb,
                   (long long)(G * mb), best * 1e3, G * per / best / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
