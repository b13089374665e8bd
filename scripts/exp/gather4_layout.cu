// Experiment: layout check of TMA tile::gather4 with a 2D map, box {64, 1},
// SWIZZLE_128B. Gathers rows {5,2,9,0} and {7,7,3,1} of a [16, 128] bf16 matrix
// (element value = row*1000+col as u16) into a 1024-byte aligned tile and prints
// the position of each 16-byte chunk, to confirm row r of the tile lands at
// r*128 with chunk j at ((j ^ (r & 7)) * 16) -- the layout UMMA's SW128 K-major
// descriptor expects.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, uint16_t* out) {
    __shared__ __align__(1024) uint16_t buf[8 * 64];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(1024));
        int rows[8] = {5, 2, 9, 0, 7, 7, 3, 1};
        for (int g = 0; g < 2; ++g)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su(buf + g * 256)),
                "l"(reinterpret_cast<uint64_t>(&m)), "r"(su(&bar)), "r"(64), "r"(rows[4 * g]), "r"(rows[4 * g + 1]),
                "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3])
                : "memory");
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(su(&bar)));
        for (int i = 0; i < 512; ++i) out[i] = buf[i];
    }
}
typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const int R = 16, K = 128;
    std::vector<uint16_t> h(R * K);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < K; ++c) h[r * K + c] = (uint16_t)(r * 1000 + c);
    uint16_t *d, *o;
    cudaMalloc(&d, h.size() * 2);
    cudaMalloc(&o, 1024);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[2] = {K, R}, str[1] = {K * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult rc = ((enc_t)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)rc);
    k<<<1, 32>>>(m, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<uint16_t> out(512);
    cudaMemcpy(out.data(), o, 1024, cudaMemcpyDeviceToHost);
    int rows[8] = {5, 2, 9, 0, 7, 7, 3, 1};
    int bad = 0;
    for (int r = 0; r < 8; ++r)
        for (int j = 0; j < 8; ++j) {
            const int slot = r * 64 + ((j ^ (r & 7)) * 8);
            for (int u = 0; u < 8; ++u)
                if (out[slot + u] != (uint16_t)(rows[r] * 1000 + 64 + j * 8 + u)) ++bad;
        }
    printf("row0 raw:");
    for (int i = 0; i < 64; i += 8) printf(" %u", out[i]);
    printf("\nSW128 layout mismatches: %d\n", bad);
    return bad != 0;
}
