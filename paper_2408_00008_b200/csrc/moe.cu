// moe.cu -- libmoe: the C ABI of include/moe.h (context, validation, workspace,
// TMA-descriptor cache, launch sequence, instrumentation, NCCL variants).
//
// Launch sequence of one forward (single GPU; SURVEY.md Sec. 3 "S1"):
//   K1 moe_router_kernel   (logits, top-k, gates, histogram, scan)     [a2-a5]
//   K2 moe_permute_kernel  (stable positions, 16-B row scatter)        [a6]
//   K3 moe_gemm_kernel<G1> (w1/w3 grouped GEMM + fused SwiGLU)         [a7]
//   K4 moe_gemm_kernel<G2> (w2 grouped GEMM, fp32 out / split-K)       [a8]
//   K5 moe_combine_kernel  (gate-weighted un-permute, bf16 RNE)        [a9]
// chained with programmatic dependent launch; no host synchronisation.

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/moe.h"
#include "gemm_sm100.cuh"
#include "ffn_fused.cuh"
#include "kernels.cuh"
#include "nvls.h"

using namespace moe;

namespace {

thread_local std::string g_init_error;

enum Slot { kSlotRouter = 0, kSlotPermute, kSlotGemm1, kSlotGemm2, kSlotCombine, kSlotDispatch, kSlotExchange, kSlotPack };

// ------------------------------------------------------------------ NCCL (dlopen)
typedef int ncclResult_t;
typedef void* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { ncclInt8 = 0, ncclInt32 = 2, ncclFloat32 = 7, ncclBfloat16 = 9 };
enum { ncclSum = 0 };
struct NcclApi {
    bool loaded = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AlltoAll)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);  // optional (>= 2.28)
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl(std::string& err) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.loaded) return true;
    const char* env = getenv("MOE_NCCL_LIB");
    const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* c : cands) {
        if (!c) continue;
        h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) { err = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return false; }
#define LOADSYM(field, name)                                                     \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));    \
    if (!g_nccl.field) { err = "missing NCCL symbol " name; return false; }
    // ncclAlltoAll exists only from NCCL 2.28 (the system libnccl here is 2.27): optional,
    // comm_alltoall falls back to grouped ncclSend / ncclRecv with the same counts
    g_nccl.AlltoAll = reinterpret_cast<decltype(g_nccl.AlltoAll)>(dlsym(h, "ncclAlltoAll"));
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(AllReduce, "ncclAllReduce");
    LOADSYM(ReduceScatter, "ncclReduceScatter");
    LOADSYM(AllGather, "ncclAllGather");
    LOADSYM(Send, "ncclSend");
    LOADSYM(Recv, "ncclRecv");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(GetErrorString, "ncclGetErrorString");
#undef LOADSYM
    g_nccl.loaded = true;
    return true;
}

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_t get_encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    });
    return fn;
}

typedef CUresult (*PFN_waitValue64_t)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
PFN_waitValue64_t get_wait64_fn() {
    static PFN_waitValue64_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_waitValue64_t>(p);
    });
    return fn;
}

typedef CUresult (*PFN_writeValue64_t)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
PFN_writeValue64_t get_write64_fn() {
    static PFN_writeValue64_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_writeValue64_t>(p);
    });
    return fn;
}

// rank-2 [rows, K] or rank-3 [batch, rows, K] bf16, K innermost; box {64, box_rows(, 1)}; 128B swizzle.
bool encode_map(CUtensorMap* m, const void* base, int rank, uint64_t K, uint64_t rows, uint64_t batch,
                uint32_t box_rows) {
    PFN_encodeTiled_t fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {K, rows, batch};
    cuuint64_t strides[2] = {K * 2, K * 2 * rows};
    cuuint32_t box[3] = {64, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Store map of a row-major [rows, cols] output (h: bf16, y: fp32) for the CTA-pair epilogue:
// box {128 B of columns, 32 rows}, 128-byte swizzle (gemm_sm100.cuh kPairOutBytes).
bool encode_store_map(CUtensorMap* m, const void* base, bool fp32, uint64_t cols, uint64_t rows) {
    PFN_encodeTiled_t fn = get_encode_fn();
    if (!fn) return false;
    const uint64_t eb = fp32 ? 4 : 2;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * eb};
    cuuint32_t box[2] = {(cuuint32_t)(128 / eb), 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Tiled bf16 weights (moe_pack_weights): 4D {64, tile_rows, K/64, tiles_per_expert * E}, each
// [tile_rows][64] chunk contiguous; box {64, box_rows, 1, box_tiles}; 128B swizzle.
bool encode_wmap(CUtensorMap* m, const void* base, uint64_t K, uint64_t tile_rows, uint64_t ntiles_total,
                 uint32_t box_rows, uint32_t box_tiles) {
    PFN_encodeTiled_t fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {64, tile_rows, K / 64, ntiles_total};
    cuuint64_t strides[3] = {128, tile_rows * 128, (K / 64) * tile_rows * 128};
    cuuint32_t box[4] = {64, box_rows, 1, box_tiles};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// rank-3 [batch, rows, K] fp8 (1 byte), box {64, box_rows, 1}, 64-byte swizzle (FP8 weights)
bool encode_map_fp8(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint64_t batch, uint32_t box_rows,
                    uint32_t box_k = 64) {
    PFN_encodeTiled_t fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {K, rows, batch};
    cuuint64_t strides[2] = {K, K * rows};
    cuuint32_t box[3] = {box_k, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, box_k == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Tiled FP8 weights (moe_pack_weights_fp8): 4D {128 B, tile_rows, K/128, tiles_total}, each
// [tile_rows][128 B] chunk contiguous; box {128, tile_rows, 1, 1}; 128B swizzle.
bool encode_wmap_u8(CUtensorMap* m, const void* base, uint64_t K, uint64_t tile_rows, uint64_t ntiles_total) {
    PFN_encodeTiled_t fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {128, tile_rows, K / 128, ntiles_total};
    cuuint64_t strides[3] = {128, tile_rows * 128, (K / 128) * tile_rows * 128};
    cuuint32_t box[4] = {128, (cuuint32_t)tile_rows, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
int next_pow2(int v) { int p = 1; while (p < v) p <<= 1; return p; }

}  // namespace

struct moe_ctx {
    moe_config cfg{};
    int device = 0;
    int num_sms = 148;
    int d = 0, f = 0, E = 0, k = 0, G = 1, rank = 0;
    int E_local = 0, e_lo = 0, f_local = 0, f_off = 0;
    int ep_world = 1, ep_rank = 0, tp_world = 1, tp_rank = 0;  // G = ep_world * tp_world
    float* lb_scratch = nullptr;  // loopback all-reduce scratch (test transport)
    size_t lb_scratch_elems = 0;
    int max_T = 0, nblk_max = 0;
    int64_t cap = 0;          // rows of the permuted buffers (tiled path)
    int64_t cap_swap = 0;     // rows used by the swap (decode) path
    // Tuning (moe_config.tuning, include/moe.h moe_tuning; defaults below). Measurements
    // behind each default: DESIGN.md section 12 and profiles/r01/experiments/.
    // Decode (swap-AB) GEMMs while the mean rows per local expert T*k/E_l <= this: the
    // weight stream dominates up to ~2 token tiles of 128 per expert (r01: 32-layer
    // T=575 stack 18.5 ms swap vs 20.8 ms CTA-pair tiles). For the w2 GEMM an isolated
    // layer favours CTA pairs from ~40 rows per expert, but inside the 32-layer stack the
    // swap kernel's weight prefetch under PDL wins (17.85 vs 18.5-18.7 ms).
    int swap_rows_per_expert = 256;   // w1/w3 GEMM
    int swap2_rows_per_expert = 256;  // w2 GEMM
    int max_splits = 8;       // split-K partial buffers are sized for this many splits
    int64_t split_stride = 0; // elements between split-K partial buffers of this forward
    bool fp8 = false;             // MOE_FLAG_FP8_WEIGHTS
    moe_expert_weights cur_w{};   // weights of the current forward
    int pair_tune = 0;        // prefill tile-order override (tuning.pair_order)
    // prefill tile orders (pair_decode). G1: bands of 16 token tiles (ncu DRAM sweep r01).
    // G2: bands of 8 weight tiles, weight tiles fastest (tiled weights, interleaved A/B on
    // two boxes: 18.57/18.52 and 18.30/18.11 ms per step vs 19.14/19.04 and 18.36/18.48 ms
    // for weight-tiles-fastest; DRAM 17.2 vs 17.6 GB per launch, scripts/sweep_order.sh)
    int g1_raster = 2, g1_band = 16, g2_raster = 3, g2_band = 8;
    // weight blocks (256 columns) per CTA-pair tile: 2 = 256 x 512 tiles with a
    // single-buffered TMEM accumulator (gemm_sm100.cuh PairCfg), 1 = 256 x 256 tiles
    // with two accumulators. G2 band counts wide tiles when 2.
    int pair_nblk = 2;
    int swap_nb_cap = 0;      // cap of the swap-path token tile (tuning; see run_gemms)
    int tune_g1_nb = 0, tune_g2_nb = 0;  // forced swap-path token tiles (tuning g1_nb / g2_nb; 0 = auto)
    int pair_hints = 0;                  // prefill L2 policies (tuning.pair_hints; see pair_hint())
    // CUDA-core router (2 tokens / block, 32 blocks at T = 64) for T <= this.
    // r01 64-token decode, interleaved: 0.4335 vs 0.4312 ms with the mma.sync router (4 blocks)
    int router_cc_max_T = 0;
    // FP8 weights (moe_gemm_fp8x_kernel, both GEMMs on 8-bit MMAs): tokens as two E4M3
    // terms with a per-row scale, h as two E4M3 terms with UE8M0 block scales
    float* tok_scale = nullptr;   // [cap] 2^-s of each permuted row
    uint8_t* h8 = nullptr;        // [2][cap][f_local] E4M3 terms of h (w1/w3 epilogue -> w2 GEMM)
    uint8_t* h_sf = nullptr;      // [cap/NB][f_local/128][2 NB * 4 B] their UE8M0 scales (GemmParams::h_sf)
    int fp8_nb2 = 0;              // token tile of this forward's FP8 w2 GEMM (sets the scale layout)
    CUtensorMap tm_h8[3]{};       // h8 planes, box {128, NB}, NB = 32, 64, 128
    CUtensorMap tm_x8[3]{};       // x_perm as [2][cap][d] E4M3 planes, box {128, NB}, NB = 32, 64, 128
    // workspace (device)
    int32_t *topk_idx = nullptr, *pos = nullptr, *blockcount = nullptr, *blockoff = nullptr;
    int32_t *counts = nullptr, *offsets = nullptr;
    float* topk_w = nullptr;
    unsigned int* done = nullptr;
    unsigned int* fold_epoch = nullptr;   // folded EP dispatch: scan publications (monotonic)
    int ep_fold_mode = 0;                 // tuning.ep_fold: 2 on (EP P2P, T <= 64), 0 / 1 off
    __nv_bfloat16 *x_perm = nullptr, *h = nullptr;
    int32_t* src_row = nullptr;  // gather mode: [cap + 512] token of each permuted row
    int w13_nt = 0, w2_nt = 0;   // tiles per expert of the tiled bf16 weight layout (256 / 128 rows)
    bool gather = false;         // MOE_FLAG_GATHER: tile::gather4 token fetch
    bool gather_now = false;     // the current forward gathers (set per call)
    // Decode speculative L2 weight prefetch (K blocks per CTA, 0 = off): the router and
    // permute kernels trigger their PDL dependents early, so the w1/w3 GEMM launches
    // while routing runs and prefetches the first K blocks of the weight tile it will
    // most likely own (every expert holding one token tile) into L2.
    // Only for 16 <= T <= 128 (one token tile per expert, all experts likely used).
    // 48 after the grid change (ab_spec2.log, 3/3 rounds: 0.4121 ms at 48, 0.4127 at 32,
    // 0.4132 at 16 and off; first sweep on 148-CTA grids: ab_spec_l2.log).
    int spec_l2 = 48;
    bool spec_now = false;       // the current forward prefetches speculatively (set per call)
    // Persistent grid of the bf16 swap GEMMs (run_gemms; tuning g1_grid / g2_grid override,
    // 0 = auto). Auto, when every expert fits one token tile (decode): the w1/w3 GEMM runs
    // (f_l/128) * floor(SMs / (f_l/128)) CTAs -- Mixtral: 112, so CTA m streams weight tile
    // m of every expert -- and the w2 GEMM ceil(U / ceil(U / SMs)) CTAs for U units (256 ->
    // 128: two equal waves). r01 interleaved sweep at the 64-token decode
    // (profiles/r01/experiments/ab_grid*.log): w1/w3 grid 148 -> 282.4 us, 136 -> 296,
    // 128 -> ~283, 120 -> 278.7, 112 -> 266.8 (7.06 TB/s), 104 -> 274, 96 -> 286; w2 grid
    // 148 -> 154.8 us, 136 -> 146, 128 -> 142.7, 112 -> 207; step 0.4340 -> 0.4124 ms.
    // These two rules are bf16 only: the FP8 kernels are slower on them (ab_grid_fp8.log:
    // w1/w3 165 -> 184 us at 112, w2 94 -> 105 us at 128); the FP8 w1/w3 GEMM takes equal
    // waves instead (run_gemms), the FP8 w2 GEMM one CTA per SM.
    int g1_grid = 0, g2_grid = 0;
    int g1_grid_now = 0, g2_grid_now = 0;  // the current forward's choice
    // Fused decode FFN (moe_ffn_fused_kernel, ffn_fused.cuh): w1/w3 + SwiGLU and w2 tiles in
    // one persistent launch (tuning.fused: 0 auto, 1 off, 2 on where the shape allows;
    // tuning.fused_splits: K splits of its w2 tiles, 0 = auto)
    int fused_mode = 0, fused_splits = 0, fused_stages = 0, fused_uniform = 0;
    bool fused_now = false;              // the current forward ran the fused kernel
    int32_t* fused_sched = nullptr;      // [2] claim / exit counters (zero between launches)
    int32_t* fused_ready = nullptr;      // [E_local * f_local / 128] finished h tiles
    int32_t* fused_arrive = nullptr;     // [d / 256] finished w2 tiles per slice (in-kernel combine)
    int32_t* fused_chain = nullptr;      // [fused_chain_n] splits stored per w2 output tile (split chaining)
    int64_t fused_chain_n = 0;
    int fused_chain_mode = 0;            // tuning.fused_chain: 1 on, 0 off (S partial buffers, default)
    int fused_half_mode = 0;             // tuning.fused_half: 0 auto, 1 off, 2 on (128-row w1/w3 tiles)
    bool fused_half_now = false;
    int combine_vec = 0;                 // tuning.combine_vec: K5 column groups per thread (0 auto, 1, 4)
    // in-kernel combine of the fused FFN (single GPU, no TP / EP; tuning.fused_combine 1 = on):
    // set by forward_impl before run_gemms, taken by the fused launch (fcomb_done)
    struct FusedCombine {
        bool on = false;
        int T = 0;
        const void* x = nullptr;
        void* out = nullptr;
        float* out_f32 = nullptr;
    } fcomb;
    bool fcomb_done = false;
    int fused_combine_mode = 0;  // tuning.fused_combine: 0 auto (host output), 1 always, 2 never
    bool host_out_now = false;   // moe_forward_host: this forward's output is mapped host memory
    CUtensorMap tm_src{};        // gather map over the current call's tokens [T, d], box {64, 1}
    float* y = nullptr;
    int64_t y_elems = 0;
    __nv_bfloat16 *stage_in = nullptr, *stage_out = nullptr;  // moe_forward_host staging (2 input slots)
    cudaStream_t copy_stream = nullptr;                        // moe_forward_host uploads
    cudaEvent_t slot_free[2]{}, slot_loaded[2]{};
    int host_slot = 0;
    uint64_t swap_w_hint = 0;    // L2 policy of the decode GEMMs' weight stream (set per forward)
    int swap_hint_mode = 0;      // tuning.weight_hint: 0 auto, 1 evict-first, 2 normal, 3 evict-last
    int swap_pair_mode = 0;      // tuning.swap_pair: 0 auto, 1 off, 2 on where the shape allows
    bool host_zero_copy = true;  // moe_forward_host: combine writes pinned output directly (tuning.host_stage: copy)
    moe_nvls::State* nvls = nullptr;  // MOE_FLAG_NVLS: symmetric window + device communicator (nvls.cu)
    int nvls_blocks = 0;              // grid bound of the fused TP combine (its LSA barrier count)
    float* tp_partial = nullptr;                               // TP: fp32 partial [max_T, d]
    float* tp_scatter = nullptr;                               // TP: reduce-scatter result
    // EP staging
    __nv_bfloat16 *ep_send = nullptr, *ep_recv = nullptr;
    float *ep_ysend = nullptr, *ep_yrecv = nullptr;
    int32_t *ep_meta_send = nullptr, *ep_meta_recv = nullptr;
    int32_t *ep_ridx = nullptr, *ep_rpos = nullptr;
    float* ep_rw = nullptr;
    int32_t* ep_rcounts = nullptr;    // device: rows each peer sends me (exact mode)
    int32_t* h_counts = nullptr;      // pinned host: [0,64) my send counts, [64,128) receive counts
    int64_t ep_exact_bytes = 32ll << 20;  // exact mode when a capacity exchange would move more bf16 bytes
    // peer-memory transport (MOE_FLAG_P2P, p2p.cuh)
    bool p2p = false;             // flag given at init: symmetric region allocated
    bool p2p_ready = false;       // moe_p2p_connect done
    int p2p_world = 1, p2p_rank = 0;
    uint8_t* sym = nullptr;       // this rank's symmetric region
    size_t sym_bytes = 0;
    struct SymLayout {
        int64_t ep_rows = 0, ep_meta = 0, ep_yret = 0;      // EP: [G*cap, d] bf16, [G*cap] i32, [G*cap, d] f32
        int64_t tp_slots = 0, tp_keep16 = 0, tp_keep32 = 0; // TP: [G][shard_max, d] f32, [max_T, d] bf16 / f32
        int64_t sig = 0;                                    // 4 u64 arrival counters
    } so;
    int tp_shard_max = 0;
    uint8_t** d_peers = nullptr;  // device [p2p_world] region bases (own included)
    unsigned int* p2p_tickets = nullptr;  // device [4] last-block tickets of the producing kernels
    std::vector<void*> p2p_opened;  // IPC mappings to close at destroy
    // TMA descriptors: workspace operands
    CUtensorMap tm_x_tiled{}, tm_h_tiled{};
    CUtensorMap tm_h_store{}, tm_y_store{};       // CTA-pair epilogue TMA stores
    CUtensorMap tm_x_swap[6]{}, tm_h_swap[6]{};  // box rows 32, 64, 128, 256, 192, 96 (96: CTA-pair NB 192)
    // weight descriptor cache (keyed by pointer)
    struct WeightMaps {
        const void* w13 = nullptr;
        const void* w2 = nullptr;
        uint64_t tick = 0;
        CUtensorMap tm_w13{}, tm_w13_pair{}, tm_w2_tiled{}, tm_w2_swap{}, tm_w13_h{};
    };
    static constexpr size_t kWeightMapCache = 64;
    std::vector<WeightMaps> wmaps;
    uint64_t use_tick = 0;
    CUtensorMap tm_w13{}, tm_w13_pair{}, tm_w2_tiled{}, tm_w2_swap{}, tm_w13_h{};  // maps of the current call
    // instrumentation
    bool profiling = false;
    struct Ev { int slot; cudaEvent_t a, b; };
    std::vector<Ev> pending;
    std::vector<cudaEvent_t> ev_pool;
    double ms[MOE_NUM_KERNEL_SLOTS]{};
    int64_t launches[MOE_NUM_KERNEL_SLOTS]{};
    int64_t launch_count = 0;
    bool poisoned = false;
    std::string err;
};

namespace {

moe_status fail(moe_ctx* c, moe_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        // CUDA faults are sticky; a failed NCCL call may leave a group open or peers
        // blocked in a collective, so no later forward on this context may start one
        if (s == MOE_ERR_CUDA || s == MOE_ERR_NCCL) c->poisoned = true;
    } else {
        g_init_error = buf;
    }
    return s;
}

#define CUDA_TRY(ctx, expr)                                                                          \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess)                                                                       \
            return fail(ctx, MOE_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),   \
                        __FILE__, __LINE__);                                                         \
    } while (0)

cudaEvent_t take_event(moe_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Launch helper: cudaLaunchKernelEx with PDL + optional profiling events.
template <typename... KArgs, typename... Args>
moe_status launch(moe_ctx* c, int slot, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                  cudaStream_t st, Args&&... args) {
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (c->profiling) {
        ea = take_event(c);
        eb = take_event(c);
        cudaEventRecord(ea, st);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (c->cfg.flags & MOE_FLAG_NO_PDL) ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) return fail(c, MOE_ERR_CUDA, "kernel launch (slot %d) failed: %s", slot, cudaGetErrorString(e));
    c->launch_count++;
    if (c->profiling) {
        cudaEventRecord(eb, st);
        c->pending.push_back({slot, ea, eb});
    }
    return MOE_OK;
}

template <int NB>
moe_status set_fp8x_attr(moe_ctx* c) {
    CUDA_TRY(c, cudaFuncSetAttribute(moe_gemm_fp8x_kernel<kG1Swap, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Fp8xCfg<kG1Swap, NB>::kSmemBytes));
    CUDA_TRY(c, cudaFuncSetAttribute(moe_gemm_fp8x_kernel<kG2Swap, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Fp8xCfg<kG2Swap, NB>::kSmemBytes));
    return MOE_OK;
}

template <int KIND, int NBLK>
moe_status set_pair_attr(moe_ctx* c) {
    CUDA_TRY(c, cudaFuncSetAttribute(moe_gemm_pair_kernel<KIND, NBLK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     PairCfg<NBLK>::kSmemBytes));
    return MOE_OK;
}

template <int NB>
moe_status set_spair_attr(moe_ctx* c) {
    CUDA_TRY(c, cudaFuncSetAttribute(moe_gemm_swap_pair_kernel<kG1Swap, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SwapPairCfg<kG1Swap, NB>::kSmemBytes));
    CUDA_TRY(c, cudaFuncSetAttribute(moe_gemm_swap_pair_kernel<kG2Swap, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SwapPairCfg<kG2Swap, NB>::kSmemBytes));
    return MOE_OK;
}

template <int NB>
moe_status set_fused_attr(moe_ctx* c) {
    CUDA_TRY(c, cudaFuncSetAttribute(moe_ffn_fused_kernel<NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     FusedCfg<NB, false>::kSmemBytes));
    CUDA_TRY(c, cudaFuncSetAttribute(moe_ffn_fused_kernel<NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     FusedCfg<NB, true>::kSmemBytes));
    if constexpr (NB == 32)
        CUDA_TRY(c, cudaFuncSetAttribute(moe_ffn_fused_kernel<32, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, FusedCfg<32, false, true>::kSmemBytes));
    return MOE_OK;
}

template <int KIND, int NB>
moe_status set_gemm_attr(moe_ctx* c) {
    CUDA_TRY(c, cudaFuncSetAttribute(moe_gemm_kernel<KIND, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     GemmCfg<KIND, NB>::kSmemBytes));
    return MOE_OK;
}

template <int KIND, int NBLK>
moe_status launch_gemm_pair(moe_ctx* c, int slot, const GemmParams& p, const CUtensorMap& a, const CUtensorMap& b,
                            const CUtensorMap& out, int nclusters, cudaStream_t st) {
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (c->profiling) {
        ea = take_event(c);
        eb = take_event(c);
        cudaEventRecord(ea, st);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * nclusters);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = PairCfg<NBLK>::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (c->cfg.flags & MOE_FLAG_NO_PDL) ? 0 : 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, moe_gemm_pair_kernel<KIND, NBLK>, p, a, b, out);
    if (e != cudaSuccess) return fail(c, MOE_ERR_CUDA, "pair kernel launch (slot %d) failed: %s", slot, cudaGetErrorString(e));
    c->launch_count++;
    if (c->profiling) {
        cudaEventRecord(eb, st);
        c->pending.push_back({slot, ea, eb});
    }
    return MOE_OK;
}

// Swap-AB GEMM on CTA pairs: `nclusters` clusters of 2 CTAs
template <int KIND, int NB>
moe_status launch_swap_pair(moe_ctx* c, int slot, const GemmParams& p, const CUtensorMap& a, const CUtensorMap& b,
                            int nclusters, cudaStream_t st) {
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (c->profiling) {
        ea = take_event(c);
        eb = take_event(c);
        cudaEventRecord(ea, st);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * nclusters);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = SwapPairCfg<KIND, NB>::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (c->cfg.flags & MOE_FLAG_NO_PDL) ? 0 : 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, moe_gemm_swap_pair_kernel<KIND, NB>, p, a, b);
    if (e != cudaSuccess)
        return fail(c, MOE_ERR_CUDA, "swap pair kernel launch (slot %d) failed: %s", slot, cudaGetErrorString(e));
    c->launch_count++;
    if (c->profiling) {
        cudaEventRecord(eb, st);
        c->pending.push_back({slot, ea, eb});
    }
    return MOE_OK;
}

template <int KIND, int NB>
moe_status launch_gemm(moe_ctx* c, int slot, const GemmParams& p, const CUtensorMap& a, const CUtensorMap& b,
                       int grid, cudaStream_t st) {
    return launch(c, slot, moe_gemm_kernel<KIND, NB>, dim3(grid), dim3(kGemmThreads),
                  (size_t)GemmCfg<KIND, NB>::kSmemBytes, st, p, a, b);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Parallel layout of a config: G ranks = ep_world x tp_world; rank = ep_rank * tp_world + tp_rank.
struct ParShape {
    int G = 1, ep_world = 1, tp_world = 1, ep_rank = 0, tp_rank = 0;
    int E_local = 0, e_lo = 0, f_local = 0, f_off = 0;
};

ParShape par_shape(const moe_config* cfg) {
    ParShape ps;
    ps.G = cfg->par == MOE_PAR_NONE ? 1 : cfg->world_size;
    if (cfg->par == MOE_PAR_EP) { ps.ep_world = ps.G; ps.ep_rank = cfg->rank; }
    if (cfg->par == MOE_PAR_TP) { ps.tp_world = ps.G; ps.tp_rank = cfg->rank; }
    if (cfg->par == MOE_PAR_HYBRID) {
        ps.tp_world = cfg->tp_size > 0 ? cfg->tp_size : 1;
        ps.ep_world = ps.G / ps.tp_world;
        ps.ep_rank = cfg->rank / ps.tp_world;
        ps.tp_rank = cfg->rank % ps.tp_world;
    }
    ps.E_local = cfg->num_experts / ps.ep_world;
    ps.e_lo = ps.ep_rank * ps.E_local;
    ps.f_local = cfg->ffn / ps.tp_world;
    ps.f_off = ps.tp_rank * ps.f_local;
    return ps;
}

moe_status validate_cfg(const moe_config* cfg, moe_ctx* c) {
    if (!cfg) return fail(c, MOE_ERR_INVALID, "cfg is NULL");
    if (cfg->hidden <= 0 || cfg->hidden % 64) return fail(c, MOE_ERR_INVALID, "hidden must be a positive multiple of 64");
    if (cfg->num_experts < 1 || cfg->num_experts > 32) return fail(c, MOE_ERR_INVALID, "num_experts must be in [1,32]");
    if (cfg->top_k < 1 || cfg->top_k > 2 || cfg->top_k > cfg->num_experts)
        return fail(c, MOE_ERR_INVALID, "top_k must be 1 or 2 and <= num_experts");
    if (cfg->max_tokens < 1) return fail(c, MOE_ERR_INVALID, "max_tokens must be >= 1");
    if (cfg->par < MOE_PAR_NONE || cfg->par > MOE_PAR_HYBRID) return fail(c, MOE_ERR_INVALID, "bad par");
    const int G = cfg->par == MOE_PAR_NONE ? 1 : cfg->world_size;
    if (G < 1 || cfg->rank < 0 || cfg->rank >= G) return fail(c, MOE_ERR_INVALID, "bad world_size/rank");
    if (cfg->par == MOE_PAR_NONE && (cfg->world_size > 1 || cfg->rank != 0))
        return fail(c, MOE_ERR_INVALID, "MOE_PAR_NONE needs world_size 1, rank 0");
    if (cfg->par == MOE_PAR_HYBRID && (cfg->tp_size < 1 || G % cfg->tp_size))
        return fail(c, MOE_ERR_INVALID, "MOE_PAR_HYBRID needs tp_size >= 1 dividing world_size");
    if (cfg->par != MOE_PAR_HYBRID && (cfg->tp_size != 0 || cfg->tp_comm))
        return fail(c, MOE_ERR_INVALID, "tp_size / tp_comm are for MOE_PAR_HYBRID only");
    const ParShape ps = par_shape(cfg);
    if (cfg->ffn <= 0 || cfg->ffn % (128 * ps.tp_world))
        return fail(c, MOE_ERR_INVALID, "ffn / tp_world must be a positive multiple of 128");
    if (cfg->num_experts % ps.ep_world) return fail(c, MOE_ERR_INVALID, "num_experts % ep_world != 0");
    if (cfg->par == MOE_PAR_TP && cfg->hidden % (4 * G))
        return fail(c, MOE_ERR_INVALID, "TP needs hidden % (4*world) == 0 (reduce-scatter shards)");
    const bool p2p = (cfg->flags & MOE_FLAG_P2P) != 0;
    if (p2p && cfg->par == MOE_PAR_HYBRID)
        return fail(c, MOE_ERR_UNSUPPORTED, "MOE_FLAG_P2P supports MOE_PAR_EP and MOE_PAR_TP");
    if (p2p && cfg->par == MOE_PAR_NONE) return fail(c, MOE_ERR_INVALID, "MOE_FLAG_P2P needs MOE_PAR_EP or MOE_PAR_TP");
    if (p2p && G > 32) return fail(c, MOE_ERR_UNSUPPORTED, "MOE_FLAG_P2P supports groups of at most 32 ranks");
    if ((cfg->flags & MOE_FLAG_NVLS) && (cfg->par != MOE_PAR_TP || p2p || !cfg->nccl_comm))
        return fail(c, MOE_ERR_INVALID, "MOE_FLAG_NVLS needs MOE_PAR_TP with an NCCL communicator (no MOE_FLAG_P2P)");
    if (!p2p && (cfg->par == MOE_PAR_EP || cfg->par == MOE_PAR_HYBRID) && !cfg->nccl_comm)
        return fail(c, MOE_ERR_INVALID, "nccl_comm (EP group) required");
    if (!p2p && cfg->par == MOE_PAR_TP && G > 1 && !cfg->nccl_comm) return fail(c, MOE_ERR_INVALID, "nccl_comm required");
    if (cfg->par == MOE_PAR_HYBRID && ps.tp_world > 1 && !cfg->tp_comm)
        return fail(c, MOE_ERR_INVALID, "tp_comm (TP group) required");
    if (cfg->split_k < 0 || cfg->split_k > 8) return fail(c, MOE_ERR_INVALID, "split_k must be in [0,8]");
    if ((cfg->flags & MOE_FLAG_FP8_WEIGHTS) && cfg->hidden % 128)
        return fail(c, MOE_ERR_UNSUPPORTED, "MOE_FLAG_FP8_WEIGHTS needs hidden % 128 == 0 (128-byte E4M3 K chunks)");
    for (int i = 0; i < 2; ++i)
        if (cfg->reserved[i]) return fail(c, MOE_ERR_INVALID, "reserved fields must be zero");
    if (const moe_tuning* tu = cfg->tuning) {
        for (int i = 0; i < 8; ++i)
            if (tu->reserved[i]) return fail(c, MOE_ERR_INVALID, "tuning.reserved fields must be zero");
        if (tu->g1_swap_rows < 0 || tu->g2_swap_rows < 0 || tu->g1_grid < 0 || tu->g2_grid < 0 ||
            tu->swap_nb_cap < 0 || tu->router_cc_max_T < 0 || tu->pair_order < 0)
            return fail(c, MOE_ERR_INVALID, "tuning fields must be >= 0 (spec_l2 may be < 0: off)");
        if (tu->pair_nblk < 0 || tu->pair_nblk > 2) return fail(c, MOE_ERR_INVALID, "tuning.pair_nblk must be 0, 1 or 2");
        if (tu->swap_pair < 0 || tu->swap_pair > 2) return fail(c, MOE_ERR_INVALID, "tuning.swap_pair must be 0, 1 or 2");
        if (tu->fused < 0 || tu->fused > 2) return fail(c, MOE_ERR_INVALID, "tuning.fused must be 0, 1 or 2");
        if (tu->fused_splits < 0 || tu->fused_splits > 8)
            return fail(c, MOE_ERR_INVALID, "tuning.fused_splits must be in [0, 8]");
        if (tu->ep_fold < 0 || tu->ep_fold > 2) return fail(c, MOE_ERR_INVALID, "tuning.ep_fold must be 0, 1 or 2");
        if (tu->combine_vec != 0 && tu->combine_vec != 1 && tu->combine_vec != 4)
            return fail(c, MOE_ERR_INVALID, "tuning.combine_vec must be 0, 1 or 4");
        if (tu->fused_half < 0 || tu->fused_half > 2)
            return fail(c, MOE_ERR_INVALID, "tuning.fused_half must be 0, 1 or 2");
        if (tu->fused_chain < 0 || tu->fused_chain > 1)
            return fail(c, MOE_ERR_INVALID, "tuning.fused_chain must be 0 or 1");
        if (tu->fused_combine < 0 || tu->fused_combine > 2)
            return fail(c, MOE_ERR_INVALID, "tuning.fused_combine must be 0, 1 or 2");
        if (tu->fused_uniform < 0 || tu->fused_uniform > 4)
            return fail(c, MOE_ERR_INVALID, "tuning.fused_uniform must be 0..4");
        if (tu->fused_stages < 0 || tu->fused_stages > 8)
            return fail(c, MOE_ERR_INVALID, "tuning.fused_stages must be in [0, 8]");
        if (tu->weight_hint < 0 || tu->weight_hint > 3) return fail(c, MOE_ERR_INVALID, "tuning.weight_hint must be 0..3");
        if (tu->swap_nb_cap && tu->swap_nb_cap != 32 && tu->swap_nb_cap != 64 && tu->swap_nb_cap != 128)
            return fail(c, MOE_ERR_INVALID, "tuning.swap_nb_cap must be 0, 32, 64 or 128");
        auto nb_ok = [](int v, bool g2) { return v == 0 || v == 32 || v == 64 || v == 128 || v == 192 || (g2 && v == 256); };
        if (!nb_ok(tu->g1_nb, false) || !nb_ok(tu->g2_nb, true))
            return fail(c, MOE_ERR_INVALID, "tuning.g1_nb must be 0/32/64/128/192, g2_nb also 256");
    }
    if ((cfg->flags & MOE_FLAG_FORCE_SWAP) && (cfg->flags & MOE_FLAG_FORCE_TILED))
        return fail(c, MOE_ERR_INVALID, "FORCE_SWAP and FORCE_TILED are exclusive");
    return MOE_OK;
}

moe_status ensure_weight_maps(moe_ctx* c, const moe_expert_weights* w) {
    c->use_tick++;
    for (auto& m : c->wmaps)
        if (m.w13 == w->w13 && m.w2 == w->w2) {
            m.tick = c->use_tick;
            c->tm_w13 = m.tm_w13; c->tm_w13_pair = m.tm_w13_pair;
            c->tm_w2_tiled = m.tm_w2_tiled; c->tm_w2_swap = m.tm_w2_swap; c->tm_w13_h = m.tm_w13_h;
            return MOE_OK;
        }
    moe_ctx::WeightMaps m;
    m.w13 = w->w13;
    m.w2 = w->w2;
    m.tick = c->use_tick;
    if (c->fp8) {  // tiled E4M3 weights: only the decode (swap-AB) maps exist
        if (!encode_wmap_u8(&m.tm_w13, w->w13, c->d, 256, (uint64_t)c->E_local * c->w13_nt) ||
            !encode_wmap_u8(&m.tm_w2_swap, w->w2, c->f_local, 128, (uint64_t)c->E_local * (c->d / 128)))
            return fail(c, MOE_ERR_CUDA, "cuTensorMapEncodeTiled(fp8 weights) failed");
    } else {
        // tiled layout: W13 in 256-row tiles, W2 in 128-row tiles (rows padded to 256)
        const uint64_t nt13 = (uint64_t)c->E_local * c->w13_nt, nt2 = (uint64_t)c->E_local * c->w2_nt;
        if (!encode_wmap(&m.tm_w13, w->w13, c->d, 256, nt13, 256, 1) ||
            !encode_wmap(&m.tm_w13_pair, w->w13, c->d, 256, nt13, 128, 1) ||
            !encode_wmap(&m.tm_w13_h, w->w13, c->d, 256, nt13, 64, 1))
            return fail(c, MOE_ERR_CUDA, "cuTensorMapEncodeTiled(w13) failed");
        if (!encode_wmap(&m.tm_w2_tiled, w->w2, c->f_local, 128, nt2, 128, 2) ||
            !encode_wmap(&m.tm_w2_swap, w->w2, c->f_local, 128, nt2, 128, 1))
            return fail(c, MOE_ERR_CUDA, "cuTensorMapEncodeTiled(w2) failed");
    }
    if (c->wmaps.size() >= moe_ctx::kWeightMapCache) {
        size_t lru = 0;
        for (size_t i = 1; i < c->wmaps.size(); ++i)
            if (c->wmaps[i].tick < c->wmaps[lru].tick) lru = i;
        c->wmaps[lru] = m;
    } else {
        c->wmaps.push_back(m);
    }
    c->tm_w13 = m.tm_w13; c->tm_w13_pair = m.tm_w13_pair;
    c->tm_w2_tiled = m.tm_w2_tiled; c->tm_w2_swap = m.tm_w2_swap; c->tm_w13_h = m.tm_w13_h;
    return MOE_OK;
}

// Decode (swap-AB) GEMM1 with token tile NB: bf16 weights, or FP8 weights widened in
// TMEM (NB <= 64) / in shared memory (NB = 128).
template <int NB>
moe_status run_swap_g1(moe_ctx* c, int nbi, const moe_expert_weights* w, cudaStream_t st) {
    GemmParams p1{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->h, 0};
    p1.hint_a = c->swap_w_hint;
    p1.w_tr = 256;
    p1.w_nt = c->w13_nt;
    if (c->gather_now) {
        p1.src_row = c->src_row;
        return launch_gemm<kG1Swap, NB>(c, kSlotGemm1, p1, c->tm_w13, c->tm_src, c->num_sms, st);
    }
    if constexpr (NB >= 32 && NB <= 128)
        if (c->fp8) {  // h -> two E4M3 planes + block scales for the block-scaled w2 GEMM
            p1.spec_l2 = c->spec_now ? c->spec_l2 : 0;  // early-triggered grid: counts after the wait
            p1.out = c->h8;
            p1.h_sf = c->h_sf;
            p1.plane_rows = c->cap;
            p1.sf_nb = c->fp8_nb2;  // scale blocks laid out for the w2 GEMM's token tile
            return launch(c, kSlotGemm1, moe_gemm_fp8x_kernel<kG1Swap, NB>, dim3(c->g1_grid_now), dim3(kGemmThreads),
                          (size_t)Fp8xCfg<kG1Swap, NB>::kSmemBytes, st, p1, static_cast<const float*>(w->w13_scale),
                          static_cast<const float*>(c->tok_scale), c->tm_w13, c->tm_x8[nbi]);
        }
    if (c->spec_now) p1.spec_l2 = c->spec_l2;
    return launch_gemm<kG1Swap, NB>(c, kSlotGemm1, p1, c->tm_w13, c->tm_x_swap[nbi],
                                    c->g1_grid_now, st);
}

template <int NB>
moe_status run_swap_g2(moe_ctx* c, int nbi, const moe_expert_weights* w, int splits, cudaStream_t st) {
    GemmParams p2{c->counts, c->offsets, c->E_local, c->d, c->f_local, splits, c->y, c->split_stride};
    p2.hint_a = c->swap_w_hint;
    p2.w_tr = 128;
    p2.w_nt = c->w2_nt;
    if constexpr (NB >= 32 && NB <= 128)
        if (c->fp8) {  // block-scaled 8-bit MMAs on the two E4M3 planes of h
            p2.h_sf = c->h_sf;
            p2.plane_rows = c->cap;
            p2.sf_nb = NB;
            return launch(c, kSlotGemm2, moe_gemm_fp8x_kernel<kG2Swap, NB>, dim3(c->g2_grid_now), dim3(kGemmThreads),
                          (size_t)Fp8xCfg<kG2Swap, NB>::kSmemBytes, st, p2, static_cast<const float*>(w->w2_scale),
                          static_cast<const float*>(nullptr), c->tm_w2_swap, c->tm_h8[nbi]);
        }
    return launch_gemm<kG2Swap, NB>(c, kSlotGemm2, p2, c->tm_w2_swap, c->tm_h_swap[nbi],
                                    c->g2_grid_now, st);
}

// Swap-AB GEMMs on CTA pairs (moe_gemm_swap_pair_kernel): token map with NB/2-row boxes
int half_box_index(int nb) { return nb == 128 ? 1 : nb == 192 ? 5 : 2; }  // 64 / 96 / 128 rows
template <int NB>
moe_status run_spair_g1(moe_ctx* c, int nclusters, cudaStream_t st) {
    GemmParams p1{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->h, 0};
    p1.hint_a = c->swap_w_hint;
    p1.w_tr = 256;
    p1.w_nt = c->w13_nt;
    return launch_swap_pair<kG1Swap, NB>(c, kSlotGemm1, p1, c->tm_w13, c->tm_x_swap[half_box_index(NB)], nclusters, st);
}
template <int NB>
moe_status run_spair_g2(moe_ctx* c, int splits, int nclusters, cudaStream_t st) {
    GemmParams p2{c->counts, c->offsets, c->E_local, c->d, c->f_local, splits, c->y, c->split_stride};
    p2.hint_a = c->swap_w_hint;
    p2.w_tr = 128;
    p2.w_nt = c->w2_nt;
    return launch_swap_pair<kG2Swap, NB>(c, kSlotGemm2, p2, c->tm_w2_swap, c->tm_h_swap[half_box_index(NB)], nclusters,
                                         st);
}

// One routing + permutation pass (K1 + K2) over `T` rows of `x`.
struct RouteSpec {
    const void* x = nullptr;     // [T, d] bf16 rows
    int T = 0, k = 0;
    const void* router_w = nullptr;       // router mode
    const int32_t* in_idx = nullptr;      // routed mode
    const float* in_w = nullptr;
    int allow_neg = 0;
    int key_lo = 0, key_div = 1, nkeys = 0, seg_align = kSegAlign;
    float* logits = nullptr;
    int32_t* topk_idx = nullptr;
    float* topk_w = nullptr;
    int32_t* pos = nullptr;
    int32_t* pos_aux = nullptr;
    void* dst_rows = nullptr;    // x_perm (normal) or EP send buffer (dispatch); nullptr: gather mode
    int32_t* src_row = nullptr;  // gather mode: token of each permuted row
    int cap = 0;                 // > 0: EP dispatch buckets of `cap` rows per key
    int32_t* meta = nullptr;
    uint8_t* const* peers = nullptr;  // P2P dispatch: rows / meta into the destinations' regions
    int64_t peer_rows_off = 0, peer_meta_off = 0;
    int my_rank = 0;
    bool early = false;          // spec_l2: router and permute trigger their dependents early
    // EP P2P dispatch folded into the router (CUDA-core router, every block does the permute's
    // work for its tokens after the scan, no permute / fill launch): peers + cap + my_rank above,
    // completion through ticket / sig like moe_ep_p2p_fill_kernel
    bool fold = false;
    unsigned int* fold_ticket = nullptr;
    int64_t fold_sig_off = 0;
};

moe_status route_and_permute(moe_ctx* c, const RouteSpec& r, cudaStream_t st) {
    // Router variant: E <= 8 -> tensor-core router (mma.sync, N = E = 8); 16 tokens
    // per block with K split over 8 warps for small batches (latency), 128 tokens
    // per block for large ones (throughput). Routed mode / E > 8 -> CUDA-core
    // router, 2 tokens per block.
    const bool mma = r.in_idx == nullptr && c->E <= 8 && r.T > c->router_cc_max_T;
    const int KS = r.T >= 2048 ? 1 : 8;
    const int TB = mma ? 16 * (8 / KS) : 2;
    const int nblk = (r.T + TB - 1) / TB;
    RouteParams rp{};
    rp.x = static_cast<const __nv_bfloat16*>(r.x);
    rp.wg = static_cast<const __nv_bfloat16*>(r.router_w);
    rp.in_idx = r.in_idx;
    rp.in_w = r.in_w;
    rp.T = r.T; rp.d = c->d; rp.E = c->E; rp.k = r.k;
    rp.key_lo = r.key_lo; rp.key_div = r.key_div; rp.nkeys = r.nkeys; rp.seg_align = r.seg_align;
    rp.allow_neg = r.allow_neg;
    rp.logits = r.logits;
    rp.topk_idx = r.topk_idx; rp.topk_w = r.topk_w;
    rp.rank = r.pos;
    rp.blockcount = c->blockcount; rp.blockoff = c->blockoff;
    rp.counts = c->counts; rp.offsets = c->offsets; rp.done = c->done;
    rp.early_trigger = r.early;
    if (r.fold) {
        rp.scan_epoch = c->fold_epoch;
        rp.peers = r.peers;
        rp.peer_rows_off = r.peer_rows_off;
        rp.peer_meta_off = r.peer_meta_off;
        rp.sig_off = r.fold_sig_off;
        rp.cap = r.cap;
        rp.my_rank = r.my_rank;
        rp.pos_aux = r.pos_aux;
        rp.p2p_ticket = r.fold_ticket;
    }
    moe_status s;
    const dim3 rg(nblk);
    if (mma && KS == 1) s = launch(c, kSlotRouter, moe_router_mma_kernel<1>, rg, dim3(256), 0, st, rp);
    else if (mma) s = launch(c, kSlotRouter, moe_router_mma_kernel<8>, rg, dim3(256), 0, st, rp);
    else if (c->E <= 8) s = launch(c, kSlotRouter, moe_router_kernel<8, 2>, rg, dim3(kRouteThreads), 0, st, rp);
    else if (c->E <= 16) s = launch(c, kSlotRouter, moe_router_kernel<16, 2>, rg, dim3(kRouteThreads), 0, st, rp);
    else s = launch(c, kSlotRouter, moe_router_kernel<32, 2>, rg, dim3(kRouteThreads), 0, st, rp);
    if (s) return s;
    if (r.fold) return MOE_OK;  // the router blocks did the dispatch

    PermuteParams pp{};
    pp.x = rp.x; pp.topk_idx = r.topk_idx; pp.blockoff = c->blockoff; pp.offsets = c->offsets;
    pp.T = r.T; pp.d = c->d; pp.k = r.k;
    pp.key_lo = r.key_lo; pp.key_div = r.key_div; pp.nkeys = r.nkeys;
    pp.cap = r.cap; pp.meta = r.meta;
    pp.TB = TB;
    pp.PT = r.T <= 1024 ? 2 : 8;
    pp.pos = r.pos; pp.pos_aux = r.pos_aux; pp.x_perm = static_cast<__nv_bfloat16*>(r.dst_rows);
    pp.src_row = r.src_row;
    pp.early_trigger = r.early;
    pp.peers = r.peers; pp.peer_rows_off = r.peer_rows_off; pp.peer_meta_off = r.peer_meta_off; pp.my_rank = r.my_rank;
    if (c->fp8 && r.cap == 0 && r.dst_rows == c->x_perm) {  // FP8 weights: two E4M3 token terms
        pp.x8 = reinterpret_cast<uint8_t*>(c->x_perm);
        pp.tok_scale = c->tok_scale;
        pp.plane_rows = c->cap;
    }
    return launch(c, kSlotPermute, moe_permute_kernel, dim3((r.T + pp.PT - 1) / pp.PT), dim3(kPermuteThreads), 0,
                  st, pp);
}

// K3 + K4 over the expert segments described by the device-side counts/offsets.
// rows_bound: upper bound of the rows of any one local expert (picks the swap-path
// token tile NB so one tile covers the whole expert at decode); rows_total: bound
// of all permuted rows (sizes the split-K partial buffers).
// Which GEMM family runs each GEMM: the swap-AB (decode) kernels while the rows of a
// local expert stay small, the tokens-as-M tiles (CTA pairs) beyond. The two GEMMs
// switch at different sizes: the w2 swap tile reads its token operand (h, NB rows)
// from L2 for every 128 weight rows, which costs more than the w1/w3 tile (256
// weight rows per token tile) -- r01 sweep, scripts/exp/stack_breakdown.py.
struct GemmPaths {
    bool swap1, swap2;
};
GemmPaths gemm_paths(const moe_ctx* c, int64_t rows_expected) {
    if ((c->cfg.flags & MOE_FLAG_FORCE_SWAP) || c->fp8) return {true, true};  // fp8 weights: decode GEMMs only
    if (c->cfg.flags & MOE_FLAG_FORCE_TILED) return {false, false};
    return {rows_expected <= (int64_t)c->swap_rows_per_expert * c->E_local,
            rows_expected <= (int64_t)c->swap2_rows_per_expert * c->E_local};
}

// K3 + K4 over the expert segments described by the device-side counts/offsets.
// rows_bound: upper bound of the rows of any one local expert (picks the swap-path
// token tile NB so one tile covers the whole expert at decode); rows_total: bound
// of all permuted rows (sizes the split-K partial buffers).
// L2 policy of field i (2 bits) of tuning.pair_hints: 0 evict-normal, 1 evict-first, 2 evict-last.
uint64_t pair_hint(int hints, int i) {
    const int v = (hints >> (2 * i)) & 3;
    return v == 1 ? ptx::kEvictFirst : v == 2 ? ptx::kEvictLast : ptx::kEvictNormal;
}

// Smallest supported swap-AB token tile >= n (GEMM1: 32, 64, 128, 192; GEMM2 adds 256).
int swap_nb_ceil(int n, bool g2) {
    if (n <= 32) return 32;
    if (n <= 64) return 64;
    if (n <= 128) return 128;
    if (n <= 192 || !g2) return 192;
    return 256;
}

// K splits of the fused kernel's w2 tiles: enough 256-row w2 units that the w2 phase is
// not a single short wave at the end of the stream
int fused_auto_splits(const moe_ctx* c, int64_t need, int nb) {
    (void)need; (void)nb;
    // bulk w2 tiles (256 rows, splits 0..S-2) + tail tiles (128 rows, split S-1): 4 splits
    // while the expert count gives >= 64 256-row units, else 8 (EP ranks holding few experts)
    return (int64_t)c->E_local * (c->d / 256) >= 64 ? 4 : 8;
}

moe_status run_gemms(moe_ctx* c, GemmPaths gp, int64_t rows_bound, int64_t rows_total, int64_t rows_expected,
                     int* splits_out, cudaStream_t st) {
    moe_status s;
    int splits = 1;
    c->split_stride = 0;
    // Token tile NB of the swap kernels: one tile covers an expert's rows when possible
    // (the weight tile then streams once from HBM and once from L2). rows_bound (an exact
    // bound: no expert gets more rows than tokens) <= 128: the power of two above it
    // (decode). Beyond, a statistical bound on the busiest expert, mean + 4 sqrt(mean)
    // of the expected rows per local expert (T = 575 stack: 144 + 48 -> 192; an expert
    // with more rows just runs a second token tile), capped at 192 for the w1/w3 GEMM
    // (a and b accumulators of 192 columns: single-buffered TMEM) and 256 for w2.
    int nb1, nb2;
    int64_t need = rows_bound;  // rows the busiest local expert is expected to hold (at most)
    if (rows_bound <= 128) {
        nb1 = nb2 = std::max(32, next_pow2((int)rows_bound));
    } else {
        const double mean = (double)std::max<int64_t>(1, rows_expected) / c->E_local;
        need = std::min<int64_t>(rows_bound, (int64_t)(mean + 4.0 * std::sqrt(mean)) + 1);
        nb1 = swap_nb_ceil((int)std::min<int64_t>(need, 192), false);
        nb2 = swap_nb_ceil((int)std::min<int64_t>(need, 256), true);
    }
    if (c->tune_g1_nb) nb1 = c->tune_g1_nb;
    if (c->tune_g2_nb) nb2 = c->tune_g2_nb;
    if (c->gather_now) nb1 = std::min(nb1, 128);  // tile::gather4 token fetch: up to 128 rows (4 per lane)
    if (c->fp8) nb1 = nb2 = std::min(nb1, 128);  // FP8 kernels: token tiles up to 128
    // tuning.swap_nb_cap: cap the swap-path token tile below the
    // worst-case bound; an expert with more rows then takes several token tiles
    // (device-side tile count: still correct), re-streaming its weights per tile
    // FP8 (fp8x) decode: a 32-token tile while the mean rows per expert is <= 16 (64-token
    // decode: per-expert counts ~ Bin(64, 1/4), P(> 32) ~ 1e-6; a larger expert just runs
    // two token tiles). The smaller B stages leave room for a 5th pipeline stage
    // (r01 A/B: 0.2744 -> 0.2686 ms per step).
    if (c->fp8 && rows_total <= 16LL * c->E_local) {
        nb1 = std::min(nb1, 32);
        nb2 = std::min(nb2, 32);
    }
    if (c->swap_nb_cap >= 32) {
        nb1 = std::min(nb1, c->swap_nb_cap);
        nb2 = std::min(nb2, c->swap_nb_cap);
    }
    if (c->fp8) {  // the w1/w3 epilogue lays the h scales out for the w2 GEMM's token tile
        nb2 = nb1;
        c->fp8_nb2 = nb2;
    }
    // weight tiles re-read by a second token tile of the same expert (rows > NB) should
    // survive in L2 between the passes: evict-normal then, evict-first otherwise (r01
    // stack T=575, interleaved: 17.97 / 17.84 ms vs 18.38 / 18.61 ms all-evict-first)
    c->swap_w_hint = c->swap_hint_mode == 1 ? ptx::kEvictFirst
                   : c->swap_hint_mode == 2 ? ptx::kEvictNormal
                   : c->swap_hint_mode == 3 ? ptx::kEvictLast
                   : (need > nb1 ? ptx::kEvictNormal : ptx::kEvictFirst);
    const bool pair = !(c->cfg.flags & MOE_FLAG_NO_PAIR);
    // Swap-AB tiles on CTA pairs (token tile split over the pair) for token tiles of >= 128
    // rows -- the mid-size batches where the token operand crowds the single-CTA stage ring
    // (tuning.swap_pair: 1 off, 2 also forced tiles). bf16 only, not in gather mode; the
    // w1/w3 pair unit is two 256-row W13 tiles (f_local % 256 == 0). The w1/w3 tile then
    // takes up to 256 token rows (a and b accumulators of 256 columns in the pair's TMEM).
    const bool sp_ok = pair && !c->fp8 && !c->gather_now && !c->spec_now && c->swap_pair_mode != 1;
    bool sp1 = sp_ok && gp.swap1 && c->f_local % 256 == 0 && (nb1 >= 128 || c->swap_pair_mode == 2);
    bool sp2 = sp_ok && gp.swap2 && (nb2 >= 128 || c->swap_pair_mode == 2);
    // w1/w3 on CTA pairs only where the pair units (E_l x f_l/256) fill the clusters: below one
    // wave (EP8 / TP8 ranks of the T=575 layer, 56 units on 74 clusters) the single-CTA tiles run
    // 112 units on 148 SMs (TP8 rank 51.6 vs 53.3 us, profiles/r03/experiments/ab_tp8_stack_rank.txt;
    // r02 shards_stack_pair.md: EP8 50.9 vs 51.9 us); the w2 GEMM stays on pairs there
    if (sp1 && c->swap_pair_mode != 2 && (int64_t)c->E_local * (c->f_local / 256) < c->num_sms / 2) sp1 = false;
    if (sp1 && !c->tune_g1_nb && rows_bound > 128) {
        nb1 = swap_nb_ceil((int)std::min<int64_t>(need, 256), true);
        if (c->swap_nb_cap >= 32) nb1 = std::min(nb1, c->swap_nb_cap);
    }
    sp1 = sp1 && nb1 >= 128;
    sp2 = sp2 && nb2 >= 128;
    // CTA-pair (cta_group::2) 256x256 tiles, one cluster of 2 CTAs per TPC; tile order
    // per GEMM (see pair_decode); env MOE_PAIR_TUNE overrides for experiments:
    // bits 0-1 G1 order, 2-3 G2 order, 4-9 G1 band, 10-15 G2 band
    int r1 = c->g1_raster, r2 = c->g2_raster, b1 = c->g1_band, b2 = c->g2_band;
    if (c->pair_tune) {
        r1 = c->pair_tune & 3; r2 = (c->pair_tune >> 2) & 3;
        b1 = std::max(1, (c->pair_tune >> 4) & 63); b2 = std::max(1, (c->pair_tune >> 10) & 63);
    }
    // Fused decode FFN: both GEMMs in one persistent launch (ffn_fused.cuh) where the shape
    // allows -- bf16, one token tile size <= 128 rows for both GEMMs, d a multiple of 256.
    c->fused_now = false;
    {
        // FP8 weights: the 32-row token tile of the FP8 decode only (moe_gemm_fp8x_kernel's tiles)
        const bool shape_ok = gp.swap1 && gp.swap2 && !c->gather_now && nb1 == nb2 && nb1 <= 128 &&
                              (!c->fp8 || nb1 == 32) && c->d % 256 == 0 && c->f_local % 128 == 0 &&
                              c->E_local <= 32;
        // auto: where the w1/w3 tiles give >= 3 waves over the SMs (single GPU, EP2 / TP2 ranks)
        // and the token tile is <= 64 rows (64-token decode: 0.4055-0.4064 vs 0.4094-0.4102 ms,
        // 3 of 3 interleaved rounds; EP4 / TP4 / EP8 / TP8 ranks measured slower fused:
        // profiles/r03/fused_ab.md)
        const int64_t U1 = (int64_t)c->E_local * (c->f_local / 128);
        const bool want = c->fused_mode == 2 ||
                          (c->fused_mode == 0 && !sp1 && !sp2 && nb1 <= 64 && U1 >= 3 * (int64_t)c->num_sms);
        // FP8 weights included since its w2 tiles run 128 rows x two K chunks per stage (one
        // block-scaled MMA per K step, 32 KB of weights per stage): 0.2281-0.2334 vs 0.2350-0.2357
        // ms for the two FP8 kernels, 3 of 3 rounds (256-row w2 tiles were slower: 0.255-0.261;
        // profiles/r03/fused_ab.md)
        if (shape_ok && want) {
            const int64_t rows_needed = round_up(rows_total + (int64_t)c->E_local * (kSegAlign - 1), kSegAlign);
            const int wt = c->f_local / 128;
            int S = c->fused_splits ? c->fused_splits : c->cfg.split_k ? c->cfg.split_k : fused_auto_splits(c, need, nb1);
            S = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)S, (int64_t)c->max_splits, (int64_t)wt,
                                                            c->y_elems / (rows_needed * c->d)}));
            c->split_stride = rows_needed * c->d;
            const int grid = c->g1_grid > 0 ? std::min(c->g1_grid, c->num_sms) : c->num_sms;
            FusedParams fp{};
            fp.g = GemmParams{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->h, 0};
            fp.g.hint_a = c->swap_w_hint;
            fp.g.w_tr = 256;
            fp.g.w_nt = c->w13_nt;
            fp.g.spec_l2 = c->spec_now ? c->spec_l2 : 0;
            if (c->fp8) {  // two E4M3 h planes + UE8M0 block scales (the FP8 w2 tiles' B operand)
                // weights evict-first, as moe_gemm_fp8x_kernel: the 32-row token tile is below the
                // 64-row bound, so the auto rule would pick evict-normal, and the weight stream then
                // pushes the token planes (re-read by every w1/w3 tile) out of L2
                fp.g.hint_a = c->swap_hint_mode ? c->swap_w_hint : ptx::kEvictFirst;
                fp.g.out = c->h8;
                fp.g.h_sf = c->h_sf;
                fp.g.plane_rows = c->cap;
                fp.g.sf_nb = 32;
                fp.w13_scale = static_cast<const float*>(c->cur_w.w13_scale);
                fp.w2_scale = static_cast<const float*>(c->cur_w.w2_scale);
                fp.tok_scale = c->tok_scale;
            }
            fp.y = c->y;
            fp.y_split_stride = c->split_stride;
            fp.splits = S;
            fp.w2_nt = c->w2_nt;
            fp.sched = c->fused_sched;
            fp.ready = c->fused_ready;
            fp.stages = c->fused_stages;
            // split chaining (tuning.fused_chain = 1): needs room for every output tile of one split.
            // Off by default: the combine gets cheaper (8.0 vs 10.2-10.7 us eager) but the fused
            // kernel slower (411 vs 402-404 us; step 0.4149-0.4156 vs 0.4076-0.4108 ms, 3 of 3
            // interleaved rounds, profiles/r03/fused_ab.md): the last split's tiles wait for the
            // previous split of their output tile
            {
                int64_t nt_sum = c->E_local;
                nt_sum += (rows_total + nb1 - 1) / nb1;
                if (c->fused_chain_mode == 1 && !c->fp8 && !MOE_FUSED_BF16_G2_128 && S > 1 &&
                    nt_sum * (c->d / 256) <= c->fused_chain_n)
                    fp.chain = c->fused_chain;
            }
            const bool comb = c->fcomb.on && c->d / 256 <= grid;  // every combine task claimed by some CTA
            if (comb) {
                fp.combine_T = c->fcomb.T;
                fp.k = c->k;
                fp.pos = c->pos;
                fp.topk_w = c->topk_w;
                fp.x_res = static_cast<const __nv_bfloat16*>(c->fcomb.x);
                fp.out = static_cast<__nv_bfloat16*>(c->fcomb.out);
                fp.out_f32 = c->fcomb.out_f32;
                fp.arrive = c->fused_arrive;
                // tokens per combine task: at most one task per CTA (grid / (d/256) chunks per slice)
                const int per_slice = std::max(1, grid / (c->d / 256));
                fp.comb_chunk = (c->fcomb.T + per_slice - 1) / per_slice;
            }
            // split boundaries in ffn tiles: uniform (tuning fused_uniform 1: the two-kernel path's
            // split of whole tiles) or tapered so the stream ends on the shortest w2 tiles: split i
            // weighted 2^(S-1-i) (fused_uniform 4; 4 splits: 8/15, 4/15, 2/15, 1/15 of K), S - i (2)
            // or (S-i)^2 (3); default (0): geometric for bf16 where one split's w2 tiles (at least
            // E_local * d/256) cover half the grid, else linear -- with few tiles per split the
            // first split's long tiles run on a few CTAs (EP8 rank, forced fused: 99.7 vs 73 us).
            // 64-token decode: 0.4052-0.4054 ms geometric vs 0.4063-0.4071 linear vs 0.4065-0.4070
            // quadratic (4 of 4 interleaved rounds); FP8: 0.2250 linear vs 0.2255-0.2268 geometric
            // (3 of 3; profiles/r03/fused_ab.md)
            {
                const bool geo = !c->fp8 && 2LL * c->E_local * (c->d / 256) >= grid;
                const int mode = c->fused_uniform ? c->fused_uniform : geo ? 4 : 2;
                auto weight = [&](int i) -> int64_t {
                    return mode == 1 ? 1 : mode == 2 ? S - i : mode == 3 ? (int64_t)(S - i) * (S - i)
                                                                         : (int64_t)1 << (S - 1 - i);
                };
                int64_t wsum = 0, acc = 0;
                for (int i = 0; i < S; ++i) wsum += weight(i);
                fp.split_j[0] = 0;
                for (int i = 0; i < S; ++i) {
                    acc += weight(i);
                    int j = (int)((wt * acc + wsum / 2) / wsum);
                    if (mode == 1) j = (int)(wt * acc / wsum);
                    fp.split_j[i + 1] = std::max(fp.split_j[i] + 1, std::min(j, wt - (S - 1 - i)));
                }
                fp.split_j[S] = wt;
            }
            c->g1_grid_now = c->g2_grid_now = grid;
            const int i = nb1 == 32 ? 0 : nb1 == 64 ? 1 : 2;
            // 128-row w1/w3 tiles where the 256-row ones do not fill the SMs (tuning.fused_half)
            const bool half = !c->fp8 && (c->fused_half_mode == 2 || (c->fused_half_mode == 0 && U1 < (int64_t)c->num_sms));
            c->fused_half_now = half;
            const CUtensorMap& tw = half ? c->tm_w13_h : c->tm_w13;
            auto go = [&](auto kern, size_t smem) {
                return launch(c, kSlotGemm1, kern, dim3(grid), dim3(kGemmThreads), smem, st, fp, tw, c->tm_x_swap[i],
                              (MOE_FUSED_BF16_G2_128 && !half) ? c->tm_w2_swap : c->tm_w2_tiled, c->tm_h_swap[i]);
            };
            if (c->fp8)
                s = launch(c, kSlotGemm1, moe_ffn_fused_kernel<32, false, true>, dim3(grid), dim3(kGemmThreads),
                           (size_t)FusedCfg<32, false, true>::kSmemBytes, st, fp, c->tm_w13, c->tm_x8[0], c->tm_w2_swap,
                           c->tm_h8[0]);
            else if (nb1 == 32)
                s = half ? go(moe_ffn_fused_kernel<32, true>, (size_t)FusedCfg<32, true>::kSmemBytes)
                         : go(moe_ffn_fused_kernel<32, false>, (size_t)FusedCfg<32, false>::kSmemBytes);
            else if (nb1 == 64)
                s = half ? go(moe_ffn_fused_kernel<64, true>, (size_t)FusedCfg<64, true>::kSmemBytes)
                         : go(moe_ffn_fused_kernel<64, false>, (size_t)FusedCfg<64, false>::kSmemBytes);
            else
                s = half ? go(moe_ffn_fused_kernel<128, true>, (size_t)FusedCfg<128, true>::kSmemBytes)
                         : go(moe_ffn_fused_kernel<128, false>, (size_t)FusedCfg<128, false>::kSmemBytes);
            if (s) return s;
            c->fused_now = true;
            c->fcomb_done = comb;
            *splits_out = fp.chain ? 1 : S;  // chained: the w2 tiles summed the splits into buffer 0
            return MOE_OK;
        }
    }
    const int ncl = c->num_sms / 2;
    {
        // bf16, one token tile per expert: the expert-stride grid where it also balances the
        // waves (all experts used; Mixtral single GPU: 896 units on 112 CTAs), else equal
        // waves over the units (TP4: 224 units -> 112 CTAs of 2 instead of 76 CTAs doing a
        // second unit while 72 idle; TP8 / EP8: 112 units -> 112 CTAs)
        const int wt = c->f_local / 128, ns = c->num_sms;
        const int gs = wt <= ns ? wt * (ns / wt) : ns;
        const int64_t U1 = (int64_t)c->E_local * wt, wv1 = (U1 + ns - 1) / ns;
        c->g1_grid_now = c->g1_grid > 0 ? std::min(c->g1_grid, ns)
                       : (c->fp8 || need > nb1) ? ns
                       : (wt <= ns && U1 % gs == 0) ? gs : (int)std::min<int64_t>(ns, (U1 + wv1 - 1) / wv1);
        // FP8 w1/w3 (fp8x) at the 32-token tile (mean <= 16 rows per expert): equal waves
        // over the E_l * wt one-tile-per-expert units (896 -> 128 CTAs; ab_grid_fp8_2.log:
        // 165.6 -> 164.2 us, step 0.2685 -> 0.2668 ms)
        if (c->g1_grid <= 0 && c->fp8 && rows_total <= 16LL * c->E_local) {
            const int64_t U1 = (int64_t)c->E_local * wt, w1 = (U1 + ns - 1) / ns;
            c->g1_grid_now = (int)std::min<int64_t>(ns, (U1 + w1 - 1) / w1);
        }
    }
    if (sp1) {
        // equal waves over the pair units (E_l x f_l/256 x token tiles) on <= SMs/2 clusters
        const int64_t U = (int64_t)c->E_local * (c->f_local / 256) * std::max<int64_t>(1, (need + nb1 - 1) / nb1);
        const int64_t waves = (U + ncl - 1) / ncl;
        const int g = c->g1_grid > 0 ? std::max(1, std::min(c->g1_grid, c->num_sms) / 2)
                                     : (int)std::min<int64_t>(ncl, (U + waves - 1) / waves);
        c->g1_grid_now = 2 * g;
        if (nb1 == 128) s = run_spair_g1<128>(c, g, st);
        else if (nb1 == 192) s = run_spair_g1<192>(c, g, st);
        else s = run_spair_g1<256>(c, g, st);
        if (s) return s;
    } else if (gp.swap1) {
        const int i1 = nb1 == 32 ? 0 : nb1 == 64 ? 1 : nb1 == 128 ? 2 : 4;
        if (nb1 == 32) s = run_swap_g1<32>(c, i1, &c->cur_w, st);
        else if (nb1 == 64) s = run_swap_g1<64>(c, i1, &c->cur_w, st);
        else if (nb1 == 128) s = run_swap_g1<128>(c, i1, &c->cur_w, st);
        else s = run_swap_g1<192>(c, i1, &c->cur_w, st);
        if (s) return s;
    } else if (pair) {
        const int nblk = c->gather_now ? 1 : c->pair_nblk;  // gather4 token fetch: 256 x 256 tiles only
        const int64_t mt_max = rows_total / 256 + c->E_local;
        const int g1 = (int)std::min<int64_t>(ncl, mt_max * ((c->f_local / 128 + nblk - 1) / nblk));
        GemmParams p1{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->h, 0, r1, b1,
                      pair_hint(c->pair_hints, 0), pair_hint(c->pair_hints, 1), c->gather_now ? c->src_row : nullptr};
        p1.w_tr = 256;
        p1.w_nt = c->w13_nt;
        const CUtensorMap& ta = c->gather_now ? c->tm_src : c->tm_x_tiled;
        s = nblk == 2 ? launch_gemm_pair<kG1Pair, 2>(c, kSlotGemm1, p1, ta, c->tm_w13_pair, c->tm_h_store, g1, st)
                      : launch_gemm_pair<kG1Pair, 1>(c, kSlotGemm1, p1, ta, c->tm_w13_pair, c->tm_h_store, g1, st);
        if (s) return s;
    } else {
        const int64_t mt_max = rows_total / 128 + c->E_local;
        const int g1 = (int)std::min<int64_t>(c->num_sms, mt_max * (c->f_local / 128));
        GemmParams p1{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->h, 0};
        p1.w_tr = 256;
        p1.w_nt = c->w13_nt;
        p1.src_row = c->gather_now ? c->src_row : nullptr;
        if ((s = launch_gemm<kG1Tiled, 256>(c, kSlotGemm1, p1, c->gather_now ? c->tm_src : c->tm_x_tiled, c->tm_w13,
                                            g1, st)))
            return s;
    }
    if (gp.swap2) {
        const int64_t rows_needed = round_up(rows_total + (int64_t)c->E_local * (kSegAlign - 1), kSegAlign);
        // split-K of the decode w2 GEMM (fixed-order fp32 partials summed by the combine).
        // r01 interleaved A/B (tiled weights): 64-token decode 0.4298 ms at 1 split vs
        // 0.434 at 2 and 0.442 at 4 (each tile's K range is one contiguous region and
        // >= 108 SMs stay busy in the last wave); the T=575 stack 17.4 ms at 2 vs 18.2 at
        // 1 and 17.4 at 4; FP8 0.2917 ms at 4 vs 0.2970 at 2.
        // Few weight units (EP / hybrid ranks holding E/G experts): split K until the units
        // cover the SMs -- EP8 at decode has 32 units of 128 W2 rows (21.6 % of 148 SMs),
        // 4 splits -> 128 units (SURVEY 8(d) wave table); EP4 64 -> 2 splits.
        const int64_t U0 = (int64_t)c->E_local * ((c->d + 127) / 128);
        // r02 (shard sweeps, profiles/r02): with one token tile per expert (NB 192 at the
        // T = 575 stack) 1 split beats 2 -- stack layer 527 vs 535 us, TP8 stack rank 94.6 vs
        // 104.8 us; the 32-layer stack is unchanged (14.97 vs 14.93 ms)
        int auto_splits = c->fp8 ? 4 : 1;
        if (need <= nb2 && 4 * U0 < 3 * (int64_t)c->num_sms)
            auto_splits = std::max<int>(auto_splits, (int)std::min<int64_t>(std::min(4, c->max_splits), c->num_sms / U0));
        splits = c->cfg.split_k ? c->cfg.split_k : auto_splits;
        splits = (int)std::max<int64_t>(1, std::min<int64_t>(splits, c->y_elems / (rows_needed * c->d)));
        splits = std::min(splits, c->f_local / (c->fp8 ? 128 : kBK));  // >= 1 K block per split
        c->split_stride = rows_needed * c->d;
        {
            const int64_t U = (int64_t)c->E_local * ((c->d + 127) / 128) * splits;
            const int ns = c->num_sms;
            const int64_t waves = (U + ns - 1) / ns;
            c->g2_grid_now = c->g2_grid > 0 ? std::min(c->g2_grid, ns)
                           : (!c->fp8 && need <= nb2) ? (int)std::min<int64_t>(ns, (U + waves - 1) / waves) : ns;
        }
        if (sp2) {
            const int64_t U = (int64_t)c->E_local * ((c->d + 255) / 256) * splits;
            const int64_t waves = (U + ncl - 1) / ncl;
            const int g = c->g2_grid > 0 ? std::max(1, std::min(c->g2_grid, c->num_sms) / 2)
                                         : (int)std::min<int64_t>(ncl, (U + waves - 1) / waves);
            c->g2_grid_now = 2 * g;
            if (nb2 == 128) s = run_spair_g2<128>(c, splits, g, st);
            else if (nb2 == 192) s = run_spair_g2<192>(c, splits, g, st);
            else s = run_spair_g2<256>(c, splits, g, st);
        } else if (nb2 == 32) s = run_swap_g2<32>(c, 0, &c->cur_w, splits, st);
        else if (nb2 == 64) s = run_swap_g2<64>(c, 1, &c->cur_w, splits, st);
        else if (nb2 == 128) s = run_swap_g2<128>(c, 2, &c->cur_w, splits, st);
        else if (nb2 == 192) s = run_swap_g2<192>(c, 4, &c->cur_w, splits, st);
        else s = run_swap_g2<256>(c, 3, &c->cur_w, splits, st);
        if (s) return s;
    } else if (pair) {
        const int nblk = c->pair_nblk;
        const int64_t mt_max = rows_total / 256 + c->E_local;
        const int g2 = (int)std::min<int64_t>(ncl, mt_max * (((c->d + 255) / 256 + nblk - 1) / nblk));
        GemmParams p2{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->y, 0, r2,
                      nblk == 2 && !c->pair_tune ? std::max(1, b2 / 2) : b2, pair_hint(c->pair_hints, 2),
                      pair_hint(c->pair_hints, 3)};
        p2.w_tr = 128;
        p2.w_nt = c->w2_nt;
        s = nblk == 2 ? launch_gemm_pair<kG2Pair, 2>(c, kSlotGemm2, p2, c->tm_h_tiled, c->tm_w2_swap, c->tm_y_store, g2, st)
                      : launch_gemm_pair<kG2Pair, 1>(c, kSlotGemm2, p2, c->tm_h_tiled, c->tm_w2_swap, c->tm_y_store, g2, st);
        if (s) return s;
    } else {
        const int64_t mt_max = rows_total / 128 + c->E_local;
        const int g2 = (int)std::min<int64_t>(c->num_sms, mt_max * ((c->d + 255) / 256));
        GemmParams p2{c->counts, c->offsets, c->E_local, c->d, c->f_local, 1, c->y, 0};
        p2.w_tr = 128;
        p2.w_nt = c->w2_nt;
        if ((s = launch_gemm<kG2Tiled, 256>(c, kSlotGemm2, p2, c->tm_h_tiled, c->tm_w2_tiled, g2, st))) return s;
    }
    *splits_out = splits;
    return MOE_OK;
}

// K5 launch: 1 column group per thread below 256 tokens (4x the blocks), 4 above
// (tuning.combine_vec overrides: 1 or 4)
moe_status launch_combine(moe_ctx* c, const CombineParams& cp, int T, cudaStream_t st) {
    const int vec = c->combine_vec ? c->combine_vec : (T <= 256 ? 1 : 4);
    if (vec == 1)
        return launch(c, kSlotCombine, moe_combine_kernel<1>, dim3((unsigned)((c->d + 1023) / 1024 * (int64_t)T)),
                      dim3(256), 0, st, cp);
    return launch(c, kSlotCombine, moe_combine_kernel<4>, dim3((unsigned)((c->d + 4095) / 4096 * (int64_t)T)),
                  dim3(256), 0, st, cp);
}

moe_status copy_aux(moe_ctx* c, const moe_aux* aux, int T, cudaStream_t st) {
    if (!aux || T <= 0) return MOE_OK;
    if (aux->topk_idx)
        CUDA_TRY(c, cudaMemcpyAsync(aux->topk_idx, c->topk_idx, sizeof(int32_t) * T * c->k, cudaMemcpyDeviceToDevice, st));
    if (aux->topk_w)
        CUDA_TRY(c, cudaMemcpyAsync(aux->topk_w, c->topk_w, sizeof(float) * T * c->k, cudaMemcpyDeviceToDevice, st));
    return MOE_OK;
}

moe_status copy_aux_segments(moe_ctx* c, const moe_aux* aux, cudaStream_t st) {
    if (!aux) return MOE_OK;
    if (aux->expert_counts)
        CUDA_TRY(c, cudaMemcpyAsync(aux->expert_counts, c->counts, sizeof(int32_t) * c->E_local, cudaMemcpyDeviceToDevice, st));
    if (aux->expert_offsets)
        CUDA_TRY(c, cudaMemcpyAsync(aux->expert_offsets, c->offsets, sizeof(int32_t) * (c->E_local + 1), cudaMemcpyDeviceToDevice, st));
    return MOE_OK;
}

// profiling of non-kernel steps (NCCL) on the launch stream
struct StepTimer {
    moe_ctx* c; int slot; cudaStream_t st; cudaEvent_t a = nullptr;
    StepTimer(moe_ctx* c_, int slot_, cudaStream_t st_) : c(c_), slot(slot_), st(st_) {
        if (c->profiling) { a = take_event(c); cudaEventRecord(a, st); }
    }
    void done() {
        if (c->profiling && a) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, st);
            c->pending.push_back({slot, a, b});
            a = nullptr;
        }
    }
};

// P2P exchange completion: counter `idx` of every rank's region += 1 after the
// producing kernel (device-side release), then this rank's stream waits until all
// G ranks have arrived for this epoch (no SM is held while waiting).
moe_status p2p_wait(moe_ctx* c, int idx, cudaStream_t st);

#define NCCL_TRY(ctx, expr)                                                                          \
    do {                                                                                             \
        ncclResult_t _r = (expr);                                                                    \
        if (_r != 0) return fail(ctx, MOE_ERR_NCCL, "%s failed: %s", #expr, g_nccl.GetErrorString(_r)); \
    } while (0)

// ncclGroupStart / ncclGroupEnd bracket that is closed on every path: an early error
// return inside the group still ends it (the NCCL group depth is per host thread and
// would otherwise swallow the caller's next NCCL calls).
struct NcclGroup {
    bool active = false;
    ncclResult_t start(bool use) {
        if (!use) return 0;
        ncclResult_t r = g_nccl.GroupStart();
        active = r == 0;
        return r;
    }
    ncclResult_t end() {
        if (!active) return 0;
        active = false;
        return g_nccl.GroupEnd();
    }
    ~NcclGroup() { end(); }
};

// ------------------------------------------------------------------ collectives
// Two transports behind the same three collectives: NCCL (production; one process
// per GPU) and a loopback group (TEST ONLY: G contexts in one process on one
// device, each driven by its own host thread; host barrier + device copies),
// which lets the EP/TP device path be parity-tested at G = 2..8 on one GPU.
__global__ void moe_loopback_add_kernel(float* dst, const float* src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

struct LoopbackGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t generation = 0;
    std::vector<const void*> ptr;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};
struct LoopbackRank {
    uint32_t magic = 0x4C4F4F50u;  // "LOOP"
    LoopbackGroup* g = nullptr;
    int rank = 0;
};

LoopbackRank* as_loopback(void* comm) {
    LoopbackRank* r = static_cast<LoopbackRank*>(comm);
    return (r && r->magic == 0x4C4F4F50u) ? r : nullptr;
}

moe_status lb_sync(moe_ctx* c, cudaStream_t st) {
    CUDA_TRY(c, cudaStreamSynchronize(st));
    return MOE_OK;
}

// A communicator of the context: NCCL handle or loopback rank handle, its size and
// this process's rank in it (EP group, TP group).
struct CommRef {
    void* comm;
    int world, rank;
};

// all-to-all: peer p's block `rank` -> my block p (count elements per peer)
moe_status comm_alltoall(moe_ctx* c, CommRef cm, const void* send, void* recv, size_t count, int nccl_type,
                         size_t esize, cudaStream_t st) {
    if (LoopbackRank* lr = as_loopback(cm.comm)) {
        moe_status s;
        if ((s = lb_sync(c, st))) return s;
        LoopbackGroup* g = lr->g;
        g->ptr[lr->rank] = send;
        g->barrier();
        const size_t b = count * esize;
        for (int p = 0; p < g->world; ++p)
            CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(recv) + p * b,
                                        static_cast<const char*>(g->ptr[p]) + lr->rank * b, b,
                                        cudaMemcpyDeviceToDevice, st));
        if ((s = lb_sync(c, st))) return s;
        g->barrier();
        return MOE_OK;
    }
    if (g_nccl.AlltoAll) {
        NCCL_TRY(c, g_nccl.AlltoAll(send, recv, count, nccl_type, cm.comm, st));
        return MOE_OK;
    }
    // NCCL < 2.28: the same exchange as grouped point-to-point calls
    const size_t b = count * esize;
    NcclGroup grp;
    NCCL_TRY(c, grp.start(true));
    for (int p = 0; p < cm.world; ++p) {
        NCCL_TRY(c, g_nccl.Send(static_cast<const char*>(send) + p * b, count, nccl_type, p, cm.comm, st));
        NCCL_TRY(c, g_nccl.Recv(static_cast<char*>(recv) + p * b, count, nccl_type, p, cm.comm, st));
    }
    NCCL_TRY(c, grp.end());
    return MOE_OK;
}

moe_status comm_reduce_scatter_f32(moe_ctx* c, CommRef cm, const float* send, float* recv, size_t cnt,
                                   cudaStream_t st) {
    if (LoopbackRank* lr = as_loopback(cm.comm)) {
        moe_status s;
        if ((s = lb_sync(c, st))) return s;
        LoopbackGroup* g = lr->g;
        g->ptr[lr->rank] = send;
        g->barrier();
        for (int p = 0; p < g->world; ++p) {
            const float* src = static_cast<const float*>(g->ptr[p]) + lr->rank * cnt;
            if (p == 0) CUDA_TRY(c, cudaMemcpyAsync(recv, src, cnt * 4, cudaMemcpyDeviceToDevice, st));
            else moe_loopback_add_kernel<<<c->num_sms, 256, 0, st>>>(recv, src, (int64_t)cnt);
        }
        if ((s = lb_sync(c, st))) return s;
        g->barrier();
        return MOE_OK;
    }
    NCCL_TRY(c, g_nccl.ReduceScatter(send, recv, cnt, ncclFloat32, ncclSum, cm.comm, st));
    return MOE_OK;
}

// in-place fp32 sum over the group (hybrid EP x TP: the expert outputs of the ffn slices)
moe_status comm_allreduce_f32(moe_ctx* c, CommRef cm, float* buf, size_t cnt, cudaStream_t st) {
    if (LoopbackRank* lr = as_loopback(cm.comm)) {
        moe_status s;
        if ((s = lb_sync(c, st))) return s;
        LoopbackGroup* g = lr->g;
        g->ptr[lr->rank] = buf;
        g->barrier();
        // every rank forms the same ascending-rank sum in a scratch copy, then all
        // ranks meet again before anyone overwrites its buffer
        float* tmp = c->lb_scratch;
        if (!tmp || c->lb_scratch_elems < cnt) {
            if (tmp) cudaFree(tmp);
            CUDA_TRY(c, cudaMalloc(reinterpret_cast<void**>(&c->lb_scratch), cnt * 4));
            c->lb_scratch_elems = cnt;
            tmp = c->lb_scratch;
        }
        for (int p = 0; p < g->world; ++p) {
            const float* src = static_cast<const float*>(g->ptr[p]);
            if (p == 0) CUDA_TRY(c, cudaMemcpyAsync(tmp, src, cnt * 4, cudaMemcpyDeviceToDevice, st));
            else moe_loopback_add_kernel<<<c->num_sms, 256, 0, st>>>(tmp, src, (int64_t)cnt);
        }
        if ((s = lb_sync(c, st))) return s;
        g->barrier();
        CUDA_TRY(c, cudaMemcpyAsync(buf, tmp, cnt * 4, cudaMemcpyDeviceToDevice, st));
        if ((s = lb_sync(c, st))) return s;
        g->barrier();
        return MOE_OK;
    }
    NCCL_TRY(c, g_nccl.AllReduce(buf, buf, cnt, ncclFloat32, ncclSum, cm.comm, st));
    return MOE_OK;
}

// all-to-all with per-peer row counts (EP exact mode): rows of peer-bucket p live at
// slot p*cap (row = row_elems elements); scount[p] rows go to p, rcount[p] come from p.
moe_status comm_alltoallv(moe_ctx* c, CommRef cm, const void* send, void* recv, const int32_t* scount,
                          const int32_t* rcount, int64_t cap, size_t row_elems, int nccl_type, size_t esize,
                          cudaStream_t st) {
    const size_t row_b = row_elems * esize;
    if (LoopbackRank* lr = as_loopback(cm.comm)) {
        moe_status s;
        if ((s = lb_sync(c, st))) return s;
        LoopbackGroup* g = lr->g;
        g->ptr[lr->rank] = send;
        g->barrier();
        for (int p = 0; p < g->world; ++p)
            if (rcount[p] > 0)
                CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(recv) + p * cap * row_b,
                                            static_cast<const char*>(g->ptr[p]) + lr->rank * cap * row_b,
                                            rcount[p] * row_b, cudaMemcpyDeviceToDevice, st));
        if ((s = lb_sync(c, st))) return s;
        g->barrier();
        return MOE_OK;
    }
    NcclGroup grp;
    NCCL_TRY(c, grp.start(true));
    for (int p = 0; p < cm.world; ++p) {
        if (scount[p] > 0)
            NCCL_TRY(c, g_nccl.Send(static_cast<const char*>(send) + p * cap * row_b, scount[p] * row_elems, nccl_type,
                                    p, cm.comm, st));
        if (rcount[p] > 0)
            NCCL_TRY(c, g_nccl.Recv(static_cast<char*>(recv) + p * cap * row_b, rcount[p] * row_elems, nccl_type, p,
                                    cm.comm, st));
    }
    NCCL_TRY(c, grp.end());
    return MOE_OK;
}

// in-place all-gather: my block lives at recv + rank*cnt
moe_status comm_allgather_inplace(moe_ctx* c, CommRef cm, void* recv, size_t cnt, int nccl_type, size_t esize,
                                  cudaStream_t st) {
    const size_t b = cnt * esize;
    if (LoopbackRank* lr = as_loopback(cm.comm)) {
        moe_status s;
        if ((s = lb_sync(c, st))) return s;
        LoopbackGroup* g = lr->g;
        g->ptr[lr->rank] = recv;
        g->barrier();
        for (int p = 0; p < g->world; ++p)
            if (p != lr->rank)
                CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(recv) + p * b,
                                            static_cast<const char*>(g->ptr[p]) + p * b, b, cudaMemcpyDeviceToDevice,
                                            st));
        if ((s = lb_sync(c, st))) return s;
        g->barrier();
        return MOE_OK;
    }
    NCCL_TRY(c, g_nccl.AllGather(static_cast<char*>(recv) + cm.rank * b, recv, cnt, nccl_type, cm.comm, st));
    return MOE_OK;
}

CommRef ep_comm(const moe_ctx* c) { return {c->cfg.nccl_comm, c->ep_world, c->ep_rank}; }
CommRef tp_comm(const moe_ctx* c) {
    return {c->cfg.par == MOE_PAR_HYBRID ? c->cfg.tp_comm : c->cfg.nccl_comm, c->tp_world, c->tp_rank};
}

moe_status check_ready(moe_ctx* c) {
    if (!c) return MOE_ERR_INVALID;
    if (c->poisoned) return fail(c, MOE_ERR_STATE, "context poisoned by an earlier CUDA error: %s", c->err.c_str());
    CUDA_TRY(c, cudaSetDevice(c->device));
    return MOE_OK;
}

// The counter of exchange idx collects exactly G arrivals per forward (one from the last
// block of every rank's producing kernel, p2p.cuh p2p_signal_last_block); after the wait
// this rank resets it to 0 (a stream memory op), so every forward waits for the SAME
// value and the P2P forward can be captured into a CUDA graph. The reset cannot race
// with the next forward's arrivals: a peer signals exchange idx of forward n+1 only
// after it has received data this rank produces after the reset (the EP return / the
// TP finished rows of forward n, or this rank's next dispatch), i.e. causally later.
moe_status p2p_wait(moe_ctx* c, int idx, cudaStream_t st) {
    const int64_t sig_off = c->so.sig + 8 * idx;
    const CUdeviceptr ctr = reinterpret_cast<CUdeviceptr>(c->sym + sig_off);
    CUresult r = get_wait64_fn()(reinterpret_cast<CUstream>(st), ctr, (uint64_t)c->p2p_world, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(c, MOE_ERR_CUDA, "cuStreamWaitValue64 failed (%d)", (int)r);
    r = get_write64_fn()(reinterpret_cast<CUstream>(st), ctr, 0, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(c, MOE_ERR_CUDA, "cuStreamWriteValue64 failed (%d)", (int)r);
    return MOE_OK;
}

moe_status forward_impl(moe_ctx* c, const void* tokens, int32_t T, const void* router_w, const int32_t* in_idx,
                        const float* in_w, const moe_expert_weights* w, void* out, const moe_aux* aux,
                        cudaStream_t st);
moe_status forward_ep(moe_ctx* c, const void* tokens, int32_t T, const void* router_w, void* out,
                      const moe_aux* aux, cudaStream_t st);

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* moe_status_string(moe_status s) {
    switch (s) {
        case MOE_OK: return "MOE_OK";
        case MOE_ERR_INVALID: return "MOE_ERR_INVALID";
        case MOE_ERR_UNSUPPORTED: return "MOE_ERR_UNSUPPORTED";
        case MOE_ERR_OOM: return "MOE_ERR_OOM";
        case MOE_ERR_CUDA: return "MOE_ERR_CUDA";
        case MOE_ERR_NCCL: return "MOE_ERR_NCCL";
        case MOE_ERR_STATE: return "MOE_ERR_STATE";
    }
    return "MOE_ERR_UNKNOWN";
}

const char* moe_last_error(const moe_ctx* ctx) { return ctx ? ctx->err.c_str() : g_init_error.c_str(); }

moe_status moe_packed_sizes(const moe_config* cfg, size_t* w13_bytes, size_t* w2_bytes) {
    moe_status s = validate_cfg(cfg, nullptr);
    if (s) return s;
    if (!w13_bytes || !w2_bytes) return fail(nullptr, MOE_ERR_INVALID, "NULL output pointer");
    const ParShape ps = par_shape(cfg);
    *w13_bytes = (size_t)ps.E_local * 2 * ps.f_local * cfg->hidden * 2;
    *w2_bytes = (size_t)ps.E_local * ((cfg->hidden + 255) / 256 * 256) * ps.f_local * 2;  // rows padded (tiled layout)
    return MOE_OK;
}

moe_status moe_packed_sizes_fp8(const moe_config* cfg, size_t* w13_bytes, size_t* w2_bytes, size_t* w13_scale_bytes,
                                size_t* w2_scale_bytes) {
    moe_status s = validate_cfg(cfg, nullptr);
    if (s) return s;
    if (!w13_bytes || !w2_bytes || !w13_scale_bytes || !w2_scale_bytes)
        return fail(nullptr, MOE_ERR_INVALID, "NULL output pointer");
    const ParShape ps = par_shape(cfg);
    *w13_bytes = (size_t)ps.E_local * 2 * ps.f_local * cfg->hidden;
    *w2_bytes = (size_t)ps.E_local * cfg->hidden * ps.f_local;
    *w13_scale_bytes = (size_t)ps.E_local * 2 * ps.f_local * 4;
    *w2_scale_bytes = (size_t)ps.E_local * cfg->hidden * 4;
    return MOE_OK;
}

moe_status moe_init(const moe_config* cfg, moe_ctx** out) {
    if (!out) return fail(nullptr, MOE_ERR_INVALID, "out is NULL");
    *out = nullptr;
    moe_status s = validate_cfg(cfg, nullptr);
    if (s) return s;
    int dev = cfg->device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return fail(nullptr, MOE_ERR_UNSUPPORTED, "no CUDA device");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || dev >= ndev)
        return fail(nullptr, MOE_ERR_UNSUPPORTED, "CUDA device %d not available", dev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
        return fail(nullptr, MOE_ERR_UNSUPPORTED, "cudaGetDeviceProperties failed");
    if (prop.major != 10 || prop.minor != 0)
        return fail(nullptr, MOE_ERR_UNSUPPORTED, "libmoe is built for sm_100a (B200); device %d is sm_%d%d", dev,
                    prop.major, prop.minor);
    if (!get_encode_fn()) return fail(nullptr, MOE_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");

    moe_ctx* c = new (std::nothrow) moe_ctx();
    if (!c) return fail(nullptr, MOE_ERR_OOM, "host allocation failed");
    c->cfg = *cfg;
    c->device = dev;
    c->num_sms = prop.multiProcessorCount;
    c->d = cfg->hidden; c->f = cfg->ffn; c->E = cfg->num_experts; c->k = cfg->top_k;
    {
        const ParShape ps = par_shape(cfg);
        c->G = ps.G; c->E_local = ps.E_local; c->e_lo = ps.e_lo; c->f_local = ps.f_local; c->f_off = ps.f_off;
        c->ep_world = ps.ep_world; c->ep_rank = ps.ep_rank; c->tp_world = ps.tp_world; c->tp_rank = ps.tp_rank;
    }
    c->rank = cfg->rank;
    c->max_T = cfg->max_tokens;
    c->w13_nt = 2 * c->f_local / 256;
    c->w2_nt = (c->d + 255) / 256 * 2;
    c->fp8 = (cfg->flags & MOE_FLAG_FP8_WEIGHTS) != 0;
    if (const moe_tuning* tu = cfg->tuning) {
        c->pair_tune = tu->pair_order;
        if (tu->pair_nblk) c->pair_nblk = tu->pair_nblk == 1 ? 1 : 2;
        c->swap_nb_cap = tu->swap_nb_cap;
        c->tune_g1_nb = tu->g1_nb;
        c->pair_hints = tu->pair_hints;
        c->tune_g2_nb = tu->g2_nb;
        c->router_cc_max_T = tu->router_cc_max_T;
        if (tu->g1_swap_rows) c->swap_rows_per_expert = tu->g1_swap_rows;
        if (tu->g2_swap_rows) c->swap2_rows_per_expert = tu->g2_swap_rows;
        if (tu->spec_l2) c->spec_l2 = std::max(0, tu->spec_l2);
        c->g1_grid = tu->g1_grid;
        c->g2_grid = tu->g2_grid;
        c->host_zero_copy = tu->host_stage == 0;
        c->swap_hint_mode = tu->weight_hint;
        c->swap_pair_mode = tu->swap_pair;
        c->fused_mode = tu->fused;
        c->fused_splits = tu->fused_splits;
        c->fused_stages = tu->fused_stages;
        c->fused_uniform = tu->fused_uniform;
        c->fused_combine_mode = tu->fused_combine;
        c->fused_chain_mode = tu->fused_chain;
        c->fused_half_mode = tu->fused_half;
        c->combine_vec = tu->combine_vec;
        c->ep_fold_mode = tu->ep_fold;
    }
    if (cfg->flags & MOE_FLAG_GATHER) c->gather = true;
    // EP: a rank may receive up to every token of every peer (dropless, reading R6).
    const bool ep_like = cfg->par == MOE_PAR_EP || cfg->par == MOE_PAR_HYBRID;
    // router blocks of >= 2 rows; EP-like contexts (also at ep_world 1) route the
    // ep_world*max_T*k receive slots too
    c->nblk_max = (int)(((int64_t)c->max_T * (ep_like ? c->ep_world * c->k : 1) + 1) / 2 + 1);
    const int64_t rows_in = ep_like ? (int64_t)c->max_T * c->ep_world : c->max_T;
    c->cap = round_up(rows_in * c->k + (int64_t)c->E_local * (kSegAlign - 1), kSegAlign);
    const int64_t swap_T = std::min<int64_t>(rows_in, (int64_t)c->swap2_rows_per_expert * c->E_local / c->k);
    c->cap_swap = round_up(swap_T * c->k + (int64_t)c->E_local * (kSegAlign - 1), kSegAlign);
    c->y_elems = std::max<int64_t>(c->cap, c->cap_swap * c->max_splits) * c->d;

    auto fail_init = [&](const char* what, cudaError_t e) {
        std::string m = std::string("workspace allocation failed (") + what + "): " + cudaGetErrorString(e);
        moe_destroy(c);
        g_init_error = m;
        return e == cudaErrorMemoryAllocation ? MOE_ERR_OOM : MOE_ERR_CUDA;
    };
    cudaError_t e;
    if ((e = cudaSetDevice(dev)) != cudaSuccess) return fail_init("cudaSetDevice", e);
    {
        const int want_world[2] = {cfg->par == MOE_PAR_TP ? c->tp_world : c->ep_world, c->tp_world};
        const int want_rank[2] = {cfg->par == MOE_PAR_TP ? c->tp_rank : c->ep_rank, c->tp_rank};
        void* comms[2] = {cfg->nccl_comm, cfg->par == MOE_PAR_HYBRID ? cfg->tp_comm : nullptr};
        for (int i = 0; i < 2; ++i)
            if (LoopbackRank* lr = as_loopback(comms[i]))
                if (lr->rank != want_rank[i] || lr->g->world != want_world[i]) {
                    moe_destroy(c);
                    return fail(nullptr, MOE_ERR_INVALID, "loopback comm rank/world does not match cfg");
                }
    }
    if (!(cfg->flags & MOE_FLAG_P2P) && !as_loopback(cfg->nccl_comm) && cfg->par != MOE_PAR_NONE && c->G > 1) {
        std::string lerr;
        if (!load_nccl(lerr)) {
            moe_destroy(c);
            return fail(nullptr, MOE_ERR_UNSUPPORTED, "%s", lerr.c_str());
        }
    }
#define ALLOC(ptr, bytes)                                                               \
    if ((e = cudaMalloc(reinterpret_cast<void**>(&(ptr)), (bytes))) != cudaSuccess)     \
        return fail_init(#ptr, e);
    const int64_t nblk_rows = c->nblk_max;
    ALLOC(c->topk_idx, sizeof(int32_t) * c->max_T * c->k);
    ALLOC(c->topk_w, sizeof(float) * c->max_T * c->k);
    ALLOC(c->pos, sizeof(int32_t) * c->max_T * c->k);
    ALLOC(c->blockcount, sizeof(int32_t) * nblk_rows * 32);
    ALLOC(c->blockoff, sizeof(int32_t) * nblk_rows * 32);
    ALLOC(c->counts, sizeof(int32_t) * 64);
    ALLOC(c->offsets, sizeof(int32_t) * 64);
    ALLOC(c->done, sizeof(unsigned int) * 4);
    ALLOC(c->fold_epoch, sizeof(unsigned int) * 4);
    ALLOC(c->fused_sched, sizeof(int32_t) * 4);
    ALLOC(c->fused_ready, sizeof(int32_t) * ((int64_t)c->E_local * (c->f_local / 64) + 4));
    ALLOC(c->fused_arrive, sizeof(int32_t) * (c->d / 256 + 4));
    // output tiles of one split: sum_e ceil(rows_e / NB) * d/256 <= (rows / 16 + E_local) * d/256
    c->fused_chain_n = ((int64_t)c->cap_swap / 16 + c->E_local + 1) * std::max(1, c->d / 256);
    ALLOC(c->fused_chain, sizeof(int32_t) * c->fused_chain_n);
    ALLOC(c->x_perm, sizeof(__nv_bfloat16) * c->cap * c->d);
    ALLOC(c->tok_scale, sizeof(float) * c->cap);
    if (c->fp8) {
        ALLOC(c->h8, (size_t)2 * c->cap * c->f_local);
        ALLOC(c->h_sf, (size_t)(c->cap / 32) * (c->f_local / 128) * 512);  // max over NB: 512 B per 32 rows
    }
    ALLOC(c->src_row, sizeof(int32_t) * (c->cap + 512));
    ALLOC(c->h, sizeof(__nv_bfloat16) * c->cap * c->f_local);
    ALLOC(c->y, sizeof(float) * c->y_elems);
    ALLOC(c->stage_in, 2 * sizeof(__nv_bfloat16) * c->max_T * c->d);
    if ((e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail_init("copy stream", e);
    for (int i = 0; i < 2; ++i)
        if ((e = cudaEventCreateWithFlags(&c->slot_free[i], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&c->slot_loaded[i], cudaEventDisableTiming)) != cudaSuccess)
            return fail_init("staging events", e);
    ALLOC(c->stage_out, sizeof(__nv_bfloat16) * c->max_T * c->d);
    if (cfg->par == MOE_PAR_TP) {
        ALLOC(c->tp_partial, sizeof(float) * c->max_T * c->d);
        ALLOC(c->tp_scatter, sizeof(float) * ((int64_t)c->max_T * c->d / c->G + 64));
    }
    if (ep_like) {
        // fixed per-peer capacity of max_T*k rows (dropless)
        const int64_t slots = (int64_t)c->ep_world * c->max_T * c->k;
        ALLOC(c->ep_send, sizeof(__nv_bfloat16) * slots * c->d);
        ALLOC(c->ep_recv, sizeof(__nv_bfloat16) * slots * c->d);
        ALLOC(c->ep_ysend, sizeof(float) * slots * c->d);
        ALLOC(c->ep_yrecv, sizeof(float) * slots * c->d);
        ALLOC(c->ep_meta_send, sizeof(int32_t) * slots + 64);
        ALLOC(c->ep_meta_recv, sizeof(int32_t) * slots + 64);
        ALLOC(c->ep_ridx, sizeof(int32_t) * slots + 64);
        ALLOC(c->ep_rpos, sizeof(int32_t) * slots + 64);
        ALLOC(c->ep_rw, sizeof(float) * slots + 64);
        ALLOC(c->ep_rcounts, sizeof(int32_t) * 64);
        if ((e = cudaMallocHost(reinterpret_cast<void**>(&c->h_counts), sizeof(int32_t) * 128)) != cudaSuccess)
            return fail_init("h_counts", e);
    }
    if (cfg->flags & MOE_FLAG_P2P) {
        // symmetric region: identical layout on every rank of the group
        c->p2p = true;
        c->p2p_world = cfg->par == MOE_PAR_TP ? c->tp_world : c->ep_world;
        c->p2p_rank = cfg->par == MOE_PAR_TP ? c->tp_rank : c->ep_rank;
        int64_t off = 0;
        auto take = [&](int64_t bytes) { const int64_t o = off; off = round_up(off + bytes, 4096); return o; };
        if (cfg->par == MOE_PAR_EP) {
            const int64_t slots = (int64_t)c->ep_world * c->max_T * c->k;
            c->so.ep_rows = take(slots * c->d * 2);
            c->so.ep_meta = take(slots * 4);
            c->so.ep_yret = take(slots * c->d * 4);
        } else {
            c->tp_shard_max = (c->max_T + c->tp_world - 1) / c->tp_world;
            c->so.tp_slots = take((int64_t)c->tp_world * c->tp_shard_max * c->d * 4);
            c->so.tp_keep16 = take((int64_t)c->max_T * c->d * 2);
            c->so.tp_keep32 = take((int64_t)c->max_T * c->d * 4);
        }
        c->so.sig = take(64);
        c->sym_bytes = (size_t)off;
        ALLOC(c->sym, c->sym_bytes);
        if ((e = cudaMemset(c->sym, 0, c->sym_bytes)) != cudaSuccess) return fail_init("memset", e);
        ALLOC(c->d_peers, sizeof(uint8_t*) * c->p2p_world);
        ALLOC(c->p2p_tickets, sizeof(unsigned int) * 4);
        if ((e = cudaMemset(c->p2p_tickets, 0, sizeof(unsigned int) * 4)) != cudaSuccess) return fail_init("memset", e);
    }
#undef ALLOC
    if (cfg->flags & MOE_FLAG_NVLS) {
        if (as_loopback(cfg->nccl_comm)) {
            moe_destroy(c);
            return fail(nullptr, MOE_ERR_INVALID, "MOE_FLAG_NVLS needs a real NCCL communicator");
        }
        char nerr[256] = {0};
        c->nvls_blocks = 2 * c->num_sms;
        if (moe_nvls::setup(cfg->nccl_comm, c->max_T, c->d, c->nvls_blocks, &c->nvls, nerr, sizeof(nerr))) {
            moe_destroy(c);
            return fail(nullptr, MOE_ERR_UNSUPPORTED, "%s", nerr);
        }
    }
    if ((e = cudaMemset(c->done, 0, sizeof(unsigned int) * 4)) != cudaSuccess ||
        (e = cudaMemset(c->fold_epoch, 0, sizeof(unsigned int) * 4)) != cudaSuccess)
        return fail_init("memset", e);
    if ((e = cudaMemset(c->fused_sched, 0, sizeof(int32_t) * 4)) != cudaSuccess ||
        (e = cudaMemset(c->fused_ready, 0, sizeof(int32_t) * ((int64_t)c->E_local * (c->f_local / 64) + 4))) != cudaSuccess ||
        (e = cudaMemset(c->fused_arrive, 0, sizeof(int32_t) * (c->d / 256 + 4))) != cudaSuccess ||
        (e = cudaMemset(c->fused_chain, 0, sizeof(int32_t) * c->fused_chain_n)) != cudaSuccess)
        return fail_init("memset", e);
    if ((e = cudaMemset(c->x_perm, 0, sizeof(__nv_bfloat16) * c->cap * c->d)) != cudaSuccess) return fail_init("memset", e);
    if ((e = cudaMemset(c->src_row, 0, sizeof(int32_t) * (c->cap + 512))) != cudaSuccess) return fail_init("memset", e);
    if ((e = cudaMemset(c->h, 0, sizeof(__nv_bfloat16) * c->cap * c->f_local)) != cudaSuccess) return fail_init("memset", e);
    if (c->fp8 && ((e = cudaMemset(c->h8, 0, (size_t)2 * c->cap * c->f_local)) != cudaSuccess ||
                   (e = cudaMemset(c->h_sf, 0x7F, (size_t)(c->cap / 32) * (c->f_local / 128) * 512)) != cudaSuccess))
        return fail_init("memset", e);

    // workspace TMA descriptors
    bool ok = encode_map(&c->tm_x_tiled, c->x_perm, 2, c->d, c->cap, 1, 128) &&
              encode_map(&c->tm_h_tiled, c->h, 2, c->f_local, c->cap, 1, 128) &&
              encode_store_map(&c->tm_h_store, c->h, false, c->f_local, c->cap) &&
              encode_store_map(&c->tm_y_store, c->y, true, c->d, c->y_elems / c->d);
    const uint32_t nbs[6] = {32, 64, 128, 256, 192, 96};
    for (int i = 0; i < 6 && ok; ++i)
        ok = encode_map(&c->tm_x_swap[i], c->x_perm, 2, c->d, c->cap, 1, nbs[i]) &&
             encode_map(&c->tm_h_swap[i], c->h, 2, c->f_local, c->cap, 1, nbs[i]);
    for (int i = 0; i < 3 && ok && c->fp8; ++i)
        ok = encode_map_fp8(&c->tm_x8[i], c->x_perm, c->d, c->cap, 2, nbs[i], 128) &&
             encode_map_fp8(&c->tm_h8[i], c->h8, c->f_local, c->cap, 2, nbs[i], 128);
    if (!ok) {
        moe_destroy(c);
        return fail(nullptr, MOE_ERR_CUDA, "cuTensorMapEncodeTiled(workspace) failed");
    }
    moe_status as;
    if ((as = set_gemm_attr<kG1Tiled, 256>(c)) || (as = set_gemm_attr<kG2Tiled, 256>(c)) ||
        (as = set_gemm_attr<kG1Swap, 32>(c)) || (as = set_gemm_attr<kG2Swap, 32>(c)) ||
        (as = set_gemm_attr<kG1Swap, 64>(c)) || (as = set_gemm_attr<kG2Swap, 64>(c)) ||
        (as = set_gemm_attr<kG1Swap, 128>(c)) || (as = set_gemm_attr<kG2Swap, 128>(c)) ||
        (as = set_gemm_attr<kG2Swap, 256>(c)) || (as = set_gemm_attr<kG1Swap, 192>(c)) ||
        (as = set_gemm_attr<kG2Swap, 192>(c)) ||
        (as = set_spair_attr<128>(c)) || (as = set_spair_attr<192>(c)) || (as = set_spair_attr<256>(c)) ||
        (as = set_pair_attr<kG1Pair, 1>(c)) || (as = set_pair_attr<kG2Pair, 1>(c)) ||
        (as = set_pair_attr<kG1Pair, 2>(c)) || (as = set_pair_attr<kG2Pair, 2>(c)) ||
        (as = set_fp8x_attr<32>(c)) || (as = set_fp8x_attr<64>(c)) || (as = set_fp8x_attr<128>(c)) ||
        (as = set_fused_attr<32>(c)) || (as = set_fused_attr<64>(c)) || (as = set_fused_attr<128>(c))) {
        std::string m = c->err;
        moe_destroy(c);
        g_init_error = m;
        return as;
    }
    // Load every kernel now. Under CUDA lazy loading a kernel's first launch loads its
    // code, which can wait on work already queued on the device -- including a P2P
    // rank's stream blocked until a peer signals (and the peer's signal may sit behind
    // that load): load up front so no launch inside a forward ever loads code.
    {
        cudaFuncAttributes fa;
        const void* fns[] = {
            reinterpret_cast<const void*>(moe_router_mma_kernel<1>), reinterpret_cast<const void*>(moe_router_mma_kernel<8>),
            reinterpret_cast<const void*>(moe_router_kernel<8, 2>), reinterpret_cast<const void*>(moe_router_kernel<16, 2>),
            reinterpret_cast<const void*>(moe_router_kernel<32, 2>), reinterpret_cast<const void*>(moe_permute_kernel),
            reinterpret_cast<const void*>(moe_combine_kernel<4>), reinterpret_cast<const void*>(moe_combine_kernel<1>),
            reinterpret_cast<const void*>(moe_ep_gather_kernel),
            reinterpret_cast<const void*>(moe_tp_finish_kernel), reinterpret_cast<const void*>(moe_loopback_add_kernel),
reinterpret_cast<const void*>(moe_ep_p2p_fill_kernel),
            reinterpret_cast<const void*>(moe_tp_p2p_finish_kernel), reinterpret_cast<const void*>(moe_tp_p2p_pull_kernel),
            reinterpret_cast<const void*>(moe_gemm_kernel<kG1Tiled, 256>), reinterpret_cast<const void*>(moe_gemm_kernel<kG2Tiled, 256>),
            reinterpret_cast<const void*>(moe_gemm_kernel<kG1Swap, 32>), reinterpret_cast<const void*>(moe_gemm_kernel<kG2Swap, 32>),
            reinterpret_cast<const void*>(moe_gemm_kernel<kG1Swap, 64>), reinterpret_cast<const void*>(moe_gemm_kernel<kG2Swap, 64>),
            reinterpret_cast<const void*>(moe_gemm_kernel<kG1Swap, 128>), reinterpret_cast<const void*>(moe_gemm_kernel<kG2Swap, 128>),
            reinterpret_cast<const void*>(moe_gemm_kernel<kG2Swap, 256>), reinterpret_cast<const void*>(moe_gemm_pair_kernel<kG1Pair, 1>),
            reinterpret_cast<const void*>(moe_gemm_kernel<kG1Swap, 192>), reinterpret_cast<const void*>(moe_gemm_kernel<kG2Swap, 192>),
            reinterpret_cast<const void*>(moe_gemm_pair_kernel<kG2Pair, 1>), reinterpret_cast<const void*>(moe_gemm_pair_kernel<kG1Pair, 2>),
            reinterpret_cast<const void*>(moe_gemm_pair_kernel<kG2Pair, 2>),
            reinterpret_cast<const void*>(moe_gemm_swap_pair_kernel<kG1Swap, 128>),
            reinterpret_cast<const void*>(moe_gemm_swap_pair_kernel<kG1Swap, 192>),
            reinterpret_cast<const void*>(moe_gemm_swap_pair_kernel<kG1Swap, 256>),
            reinterpret_cast<const void*>(moe_gemm_swap_pair_kernel<kG2Swap, 128>),
            reinterpret_cast<const void*>(moe_gemm_swap_pair_kernel<kG2Swap, 192>),
            reinterpret_cast<const void*>(moe_gemm_swap_pair_kernel<kG2Swap, 256>),
            reinterpret_cast<const void*>(moe_gemm_fp8x_kernel<kG1Swap, 32>),
            reinterpret_cast<const void*>(moe_gemm_fp8x_kernel<kG1Swap, 64>),
            reinterpret_cast<const void*>(moe_gemm_fp8x_kernel<kG1Swap, 128>),
            reinterpret_cast<const void*>(moe_gemm_fp8x_kernel<kG2Swap, 32>),
            reinterpret_cast<const void*>(moe_gemm_fp8x_kernel<kG2Swap, 64>),
            reinterpret_cast<const void*>(moe_gemm_fp8x_kernel<kG2Swap, 128>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<32, false>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<64, false>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<128, false>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<32, true>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<64, true>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<128, true>),
            reinterpret_cast<const void*>(moe_ffn_fused_kernel<32, false, true>)};
        for (const void* fn : fns)
            if ((e = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess) return fail_init("cudaFuncGetAttributes", e);
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail_init("sync", e);
    *out = c;
    return MOE_OK;
}

moe_status moe_destroy(moe_ctx* c) {
    if (!c) return MOE_OK;
    cudaSetDevice(c->device);
    void* bufs[] = {c->topk_idx, c->topk_w, c->pos, c->blockcount, c->blockoff, c->counts, c->offsets, c->done,
                    c->x_perm, c->h, c->y, c->stage_in, c->stage_out, c->tp_partial, c->tp_scatter, c->ep_send,
                    c->ep_recv, c->ep_ysend, c->ep_yrecv, c->ep_meta_send, c->ep_meta_recv,
                    c->ep_ridx, c->ep_rpos, c->ep_rw, c->ep_rcounts, c->lb_scratch, c->d_peers, c->p2p_tickets, c->src_row,
                    c->tok_scale, c->h8, c->h_sf, c->fused_sched, c->fused_ready, c->fused_arrive, c->fused_chain, c->fold_epoch};
    for (void* p : c->p2p_opened) cudaIpcCloseMemHandle(p);
    if (c->nvls) {
        cudaDeviceSynchronize();  // no fused combine still reads / writes the window
        moe_nvls::destroy(c->nvls);
    }
    if (c->sym) {
        cudaDeviceSynchronize();  // peers' stores into this region have drained (same-process group)
        cudaFree(c->sym);
    }
    for (void* b : bufs)
        if (b) cudaFree(b);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    for (int i = 0; i < 2; ++i) {
        if (c->slot_free[i]) cudaEventDestroy(c->slot_free[i]);
        if (c->slot_loaded[i]) cudaEventDestroy(c->slot_loaded[i]);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (auto& ev : c->pending) { cudaEventDestroy(ev.a); cudaEventDestroy(ev.b); }
    for (auto ev : c->ev_pool) cudaEventDestroy(ev);
    delete c;
    return MOE_OK;
}

moe_status moe_pack_weights(moe_ctx* c, const void* w1, const void* w3, const void* w2, void* w13_out, void* w2_out,
                            void* stream) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (!w1 || !w3 || !w2 || !w13_out || !w2_out) return fail(c, MOE_ERR_INVALID, "NULL weight pointer");
    if (!aligned16(w1) || !aligned16(w3) || !aligned16(w2) || !aligned16(w13_out) || !aligned16(w2_out))
        return fail(c, MOE_ERR_INVALID, "weight pointers must be 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int e_off = c->e_lo;  // 0 unless experts are sharded (EP, hybrid)
    if ((s = launch(c, kSlotPack, moe_pack_w13_kernel, dim3(4 * c->num_sms), dim3(256), 0, st,
                    static_cast<const __nv_bfloat16*>(w1), static_cast<const __nv_bfloat16*>(w3),
                    static_cast<__nv_bfloat16*>(w13_out), c->E_local, e_off, c->d, c->f, c->f_local, c->f_off, 1)))
        return s;
    if ((s = launch(c, kSlotPack, moe_pack_w2_kernel, dim3(4 * c->num_sms), dim3(256), 0, st,
                    static_cast<const __nv_bfloat16*>(w2), static_cast<__nv_bfloat16*>(w2_out), c->E_local, e_off,
                    c->d, c->f, c->f_local, c->f_off, 1, 1)))
        return s;
    // descriptors keyed by these pointers must be re-encoded if memory was reused
    (void)w13_out;  // descriptors hold addresses only; repacking in place keeps them valid
    return MOE_OK;
}

moe_status moe_pack_weights_fp8(moe_ctx* c, const void* q1, const void* q3, const void* q2, const float* s1,
                                const float* s3, const float* s2, void* w13_out, void* w2_out, float* w13_scale_out,
                                float* w2_scale_out, void* stream) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (!c->fp8) return fail(c, MOE_ERR_INVALID, "context was not created with MOE_FLAG_FP8_WEIGHTS");
    if (!q1 || !q3 || !q2 || !s1 || !s3 || !s2 || !w13_out || !w2_out || !w13_scale_out || !w2_scale_out)
        return fail(c, MOE_ERR_INVALID, "NULL pointer");
    if (!aligned16(q1) || !aligned16(q3) || !aligned16(q2) || !aligned16(w13_out) || !aligned16(w2_out))
        return fail(c, MOE_ERR_INVALID, "fp8 weight pointers must be 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int e_off = c->e_lo;
    // one byte per weight, tiled like the bf16 weights: pairs of E4M3 move as 2-byte units
    // through the bf16 packers, so a [rows][64 units] chunk is a [rows][128 B] chunk of
    // 128 E4M3 weights (w13: 256-row tiles, w2: 128-row tiles, include/moe.h)
    if ((s = launch(c, kSlotPack, moe_pack_w13_kernel, dim3(4 * c->num_sms), dim3(256), 0, st,
                    static_cast<const __nv_bfloat16*>(q1), static_cast<const __nv_bfloat16*>(q3),
                    static_cast<__nv_bfloat16*>(w13_out), c->E_local, e_off, c->d / 2, c->f, c->f_local, c->f_off, 1)))
        return s;
    if ((s = launch(c, kSlotPack, moe_pack_w2_kernel, dim3(4 * c->num_sms), dim3(256), 0, st,
                    static_cast<const __nv_bfloat16*>(q2), static_cast<__nv_bfloat16*>(w2_out), c->E_local, e_off,
                    c->d, c->f / 2, c->f_local / 2, c->f_off / 2, 1, 0)))
        return s;
    if ((s = launch(c, kSlotPack, moe_pack_scales_kernel, dim3(c->num_sms), dim3(256), 0, st, s1, s3, s2,
                    w13_scale_out, w2_scale_out, c->E_local, e_off, c->d, c->f, c->f_local, c->f_off)))
        return s;
    return MOE_OK;
}

moe_status moe_forward(moe_ctx* c, const void* tokens, int32_t T, const void* router_w,
                       const moe_expert_weights* w, void* out, const moe_aux* aux, void* stream) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (!router_w || !aligned16(router_w)) return fail(c, MOE_ERR_INVALID, "router_w must be a 16-byte aligned device pointer");
    return forward_impl(c, tokens, T, router_w, nullptr, nullptr, w, out, aux, static_cast<cudaStream_t>(stream));
}

moe_status moe_forward_routed(moe_ctx* c, const void* tokens, int32_t T, const int32_t* topk_idx,
                              const float* topk_w, const moe_expert_weights* w, void* out, const moe_aux* aux,
                              void* stream) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (c->cfg.par == MOE_PAR_EP || c->cfg.par == MOE_PAR_HYBRID)
        return fail(c, MOE_ERR_UNSUPPORTED, "moe_forward_routed: single-GPU / TP only");
    if (T > 0 && (!topk_idx || !topk_w)) return fail(c, MOE_ERR_INVALID, "NULL routing");
    return forward_impl(c, tokens, T, nullptr, topk_idx, topk_w, w, out, aux, static_cast<cudaStream_t>(stream));
}

moe_status moe_forward_host(moe_ctx* c, const void* tokens_host, int32_t T, const void* router_w,
                            const moe_expert_weights* w, void* out_host, void* stream) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (T < 0 || T > c->max_T) return fail(c, MOE_ERR_INVALID, "T out of range");
    if (T > 0 && (!tokens_host || !out_host)) return fail(c, MOE_ERR_INVALID, "NULL host buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)T * c->d * sizeof(__nv_bfloat16);
    // Double-buffered token staging: the host->device copy runs on the context's copy
    // stream as soon as its slot's previous forward has finished, so consecutive calls
    // overlap this call's upload with the previous call's forward; the forward waits
    // for the upload, the result is copied back on `stream` (ready once the caller
    // synchronises `stream`).
    const int slot = c->host_slot;
    c->host_slot ^= 1;
    __nv_bfloat16* in = c->stage_in + (size_t)slot * c->max_T * c->d;
    if (T > 0) {
        CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->slot_free[slot], 0));
        CUDA_TRY(c, cudaMemcpyAsync(in, tokens_host, bytes, cudaMemcpyHostToDevice, c->copy_stream));
        CUDA_TRY(c, cudaEventRecord(c->slot_loaded[slot], c->copy_stream));
        CUDA_TRY(c, cudaStreamWaitEvent(st, c->slot_loaded[slot], 0));
    }
    // Pinned (page-locked, device-mapped) output: the combine kernel stores the bf16 rows
    // straight into host memory over the host link -- no staging buffer, no separate
    // device->host copy on the stream. Pageable output: staging buffer + copy.
    void* out_dev = nullptr;
    if (T > 0 && c->host_zero_copy) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, out_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer && aligned16(pa.devicePointer))
            out_dev = pa.devicePointer;
        cudaGetLastError();  // pageable memory: not an error
    }
    c->host_out_now = out_dev != nullptr;
    s = moe_forward(c, in, T, router_w, w, out_dev ? out_dev : c->stage_out, nullptr, stream);
    c->host_out_now = false;
    if (s) return s;
    if (T > 0) {
        CUDA_TRY(c, cudaEventRecord(c->slot_free[slot], st));
        if (!out_dev) CUDA_TRY(c, cudaMemcpyAsync(out_host, c->stage_out, bytes, cudaMemcpyDeviceToHost, st));
    }
    return MOE_OK;
}

moe_status moe_set_profiling(moe_ctx* c, int enable) {
    if (!c) return MOE_ERR_INVALID;
    c->profiling = enable != 0;
    return MOE_OK;
}

moe_status moe_reset_profile(moe_ctx* c) {
    if (!c) return MOE_ERR_INVALID;
    for (auto& ev : c->pending) {
        cudaEventSynchronize(ev.b);
        c->ev_pool.push_back(ev.a);
        c->ev_pool.push_back(ev.b);
    }
    c->pending.clear();
    for (int i = 0; i < MOE_NUM_KERNEL_SLOTS; ++i) { c->ms[i] = 0; c->launches[i] = 0; }
    return MOE_OK;
}

moe_status moe_kernel_times(moe_ctx* c, double* ms, int64_t* launches) {
    if (!c || !ms || !launches) return MOE_ERR_INVALID;
    for (auto& ev : c->pending) {
        cudaError_t e = cudaEventSynchronize(ev.b);
        if (e != cudaSuccess) return fail(c, MOE_ERR_CUDA, "event sync: %s", cudaGetErrorString(e));
        float t = 0.f;
        cudaEventElapsedTime(&t, ev.a, ev.b);
        c->ms[ev.slot] += t;
        c->launches[ev.slot] += 1;
        c->ev_pool.push_back(ev.a);
        c->ev_pool.push_back(ev.b);
    }
    c->pending.clear();
    for (int i = 0; i < MOE_NUM_KERNEL_SLOTS; ++i) { ms[i] = c->ms[i]; launches[i] = c->launches[i]; }
    return MOE_OK;
}

int64_t moe_launch_count(const moe_ctx* c) { return c ? c->launch_count : -1; }

moe_status moe_nccl_unique_id(void* id128) {
    if (!id128) return fail(nullptr, MOE_ERR_INVALID, "NULL id");
    std::string err;
    if (!load_nccl(err)) return fail(nullptr, MOE_ERR_UNSUPPORTED, "%s", err.c_str());
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r) return fail(nullptr, MOE_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
    std::memcpy(id128, &id, 128);
    return MOE_OK;
}

moe_status moe_nccl_comm_init(const void* id128, int32_t world, int32_t rank, int32_t device, void** comm) {
    if (!id128 || !comm || world < 1 || rank < 0 || rank >= world) return fail(nullptr, MOE_ERR_INVALID, "bad args");
    std::string err;
    if (!load_nccl(err)) return fail(nullptr, MOE_ERR_UNSUPPORTED, "%s", err.c_str());
    if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return fail(nullptr, MOE_ERR_CUDA, "cudaSetDevice");
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t cm = nullptr;
    ncclResult_t r = g_nccl.CommInitRank(&cm, world, id, rank);
    if (r) return fail(nullptr, MOE_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
    *comm = cm;
    return MOE_OK;
}

moe_status moe_loopback_comm_create(int32_t world, void** group) {
    if (world < 1 || world > 64 || !group) return fail(nullptr, MOE_ERR_INVALID, "bad loopback world/group");
    LoopbackGroup* g = new (std::nothrow) LoopbackGroup();
    if (!g) return fail(nullptr, MOE_ERR_OOM, "host allocation failed");
    g->world = world;
    g->ptr.assign(world, nullptr);
    *group = g;
    return MOE_OK;
}

moe_status moe_loopback_comm_rank(void* group, int32_t rank, void** comm) {
    LoopbackGroup* g = static_cast<LoopbackGroup*>(group);
    if (!g || !comm || rank < 0 || rank >= g->world) return fail(nullptr, MOE_ERR_INVALID, "bad loopback rank");
    LoopbackRank* r = new (std::nothrow) LoopbackRank();
    if (!r) return fail(nullptr, MOE_ERR_OOM, "host allocation failed");
    r->g = g;
    r->rank = rank;
    *comm = r;
    return MOE_OK;
}

namespace {
struct P2PHandle {
    uint32_t magic;     // "MP2P"
    int32_t pid, device, rank;
    uint64_t ptr, bytes;
    cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(P2PHandle) <= MOE_P2P_HANDLE_BYTES, "handle too large");
constexpr uint32_t kP2PMagic = 0x5032504Du;
}  // namespace

moe_status moe_p2p_handle(moe_ctx* c, void* handle_out) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (!handle_out) return fail(c, MOE_ERR_INVALID, "handle_out is NULL");
    if (!c->p2p) return fail(c, MOE_ERR_STATE, "context was not created with MOE_FLAG_P2P");
    P2PHandle h{};
    h.magic = kP2PMagic;
    h.pid = (int32_t)getpid();
    h.device = c->device;
    h.rank = c->p2p_rank;
    h.ptr = reinterpret_cast<uint64_t>(c->sym);
    h.bytes = c->sym_bytes;
    CUDA_TRY(c, cudaIpcGetMemHandle(&h.ipc, c->sym));
    memset(handle_out, 0, MOE_P2P_HANDLE_BYTES);
    memcpy(handle_out, &h, sizeof(h));
    return MOE_OK;
}

moe_status moe_p2p_connect(moe_ctx* c, const void* handles, int32_t world) {
    moe_status s = check_ready(c);
    if (s) return s;
    if (!handles) return fail(c, MOE_ERR_INVALID, "handles is NULL");
    if (!c->p2p) return fail(c, MOE_ERR_STATE, "context was not created with MOE_FLAG_P2P");
    if (c->p2p_ready) return fail(c, MOE_ERR_STATE, "already connected");
    if (world != c->p2p_world) return fail(c, MOE_ERR_INVALID, "world %d != group size %d", world, c->p2p_world);
    if (!get_wait64_fn() || !get_write64_fn())
        return fail(c, MOE_ERR_UNSUPPORTED, "cuStreamWaitValue64 / cuStreamWriteValue64 unavailable");
    std::vector<uint8_t*> bases(world, nullptr);
    const int me = (int)getpid();
    for (int r = 0; r < world; ++r) {
        P2PHandle h;
        memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * MOE_P2P_HANDLE_BYTES, sizeof(h));
        if (h.magic != kP2PMagic || h.rank != r) return fail(c, MOE_ERR_INVALID, "handle %d is not rank %d's", r, r);
        if (h.bytes != c->sym_bytes)
            return fail(c, MOE_ERR_INVALID, "rank %d region is %llu bytes, mine %zu (configs differ)", r,
                        (unsigned long long)h.bytes, c->sym_bytes);
        if (r == c->p2p_rank) {
            if (h.pid != me || h.ptr != reinterpret_cast<uint64_t>(c->sym))
                return fail(c, MOE_ERR_INVALID, "handle %d is not this context's", r);
            bases[r] = c->sym;
        } else if (h.pid == me) {
            if (h.device != c->device) {  // same process, another GPU: direct peer access
                cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else CUDA_TRY(c, e);
            }
            bases[r] = reinterpret_cast<uint8_t*>(h.ptr);
        } else {
            void* p = nullptr;
            CUDA_TRY(c, cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
            c->p2p_opened.push_back(p);
            bases[r] = static_cast<uint8_t*>(p);
        }
    }
    CUDA_TRY(c, cudaMemcpy(c->d_peers, bases.data(), sizeof(uint8_t*) * world, cudaMemcpyHostToDevice));
    c->p2p_ready = true;
    return MOE_OK;
}

moe_status moe_loopback_comm_destroy(void* group_or_rank) {
    if (!group_or_rank) return MOE_OK;
    if (LoopbackRank* r = as_loopback(group_or_rank)) {
        r->magic = 0;
        delete r;
    } else {
        delete static_cast<LoopbackGroup*>(group_or_rank);
    }
    return MOE_OK;
}

moe_status moe_nccl_comm_destroy(void* comm) {
    if (!comm) return MOE_OK;
    std::string err;
    if (!load_nccl(err)) return fail(nullptr, MOE_ERR_UNSUPPORTED, "%s", err.c_str());
    ncclResult_t r = g_nccl.CommDestroy(comm);
    if (r) return fail(nullptr, MOE_ERR_NCCL, "ncclCommDestroy: %s", g_nccl.GetErrorString(r));
    return MOE_OK;
}

#if MOE_TIMELINE
// Probe builds only (not declared in include/moe.h): copies the per-block timestamps of
// the last forward ([5 slots][3 stamps][kTlBlocks] u64 ns) to `out` and clears them.
MOE_API int moe_debug_timeline(unsigned long long* out) {
    using moe::ptx::g_moe_tl;
    if (cudaMemcpyFromSymbol(out, g_moe_tl, sizeof(g_moe_tl)) != cudaSuccess) return -1;
    static unsigned long long zero[5 * 3 * moe::ptx::kTlBlocks];
    return cudaMemcpyToSymbol(g_moe_tl, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif

}  // extern "C"

namespace {

moe_status forward_impl(moe_ctx* c, const void* tokens, int32_t T, const void* router_w, const int32_t* in_idx,
                        const float* in_w, const moe_expert_weights* w, void* out, const moe_aux* aux,
                        cudaStream_t st) {
    if (T < 0 || T > c->max_T) return fail(c, MOE_ERR_INVALID, "T=%d out of range [0, %d]", T, c->max_T);
    if (!w || !w->w13 || !w->w2 || !aligned16(w->w13) || !aligned16(w->w2))
        return fail(c, MOE_ERR_INVALID, "expert weights must be 16-byte aligned device pointers");
    if (T > 0 && (!tokens || !out || !aligned16(tokens) || !aligned16(out)))
        return fail(c, MOE_ERR_INVALID, "tokens / out must be 16-byte aligned device pointers");
    if (aux && aux->out_f32 && !aligned16(aux->out_f32)) return fail(c, MOE_ERR_INVALID, "aux.out_f32 misaligned");
    if (c->fp8 && (!w->w13_scale || !w->w2_scale))
        return fail(c, MOE_ERR_INVALID, "MOE_FLAG_FP8_WEIGHTS needs w13_scale and w2_scale");
    if (c->p2p && !c->p2p_ready) return fail(c, MOE_ERR_STATE, "MOE_FLAG_P2P context: call moe_p2p_connect first");
    c->cur_w = *w;
    moe_status s = ensure_weight_maps(c, w);
    if (s) return s;
    if (c->cfg.par == MOE_PAR_EP || c->cfg.par == MOE_PAR_HYBRID) return forward_ep(c, tokens, T, router_w, out, aux, st);
    if (T == 0) return MOE_OK;  // TP: every rank passes the same T, so all skip together

    const bool tp = (c->cfg.par == MOE_PAR_TP && c->G > 1) || c->nvls;  // NVLS: the fused path at any G
    RouteSpec r;
    r.x = tokens; r.T = T; r.k = c->k;
    r.router_w = router_w; r.in_idx = in_idx; r.in_w = in_w;
    r.key_lo = c->e_lo; r.key_div = 1; r.nkeys = c->E_local; r.seg_align = kSegAlign;
    r.logits = aux ? aux->logits : nullptr;
    r.topk_idx = c->topk_idx; r.topk_w = c->topk_w;
    r.pos = c->pos; r.pos_aux = aux ? aux->pos : nullptr;
    // Gather mode (MOE_FLAG_GATHER, bf16 weights): the w1/w3 GEMM fetches token rows
    // from `tokens` through a {64, 1}-box map with tile::gather4; the permute step only
    // records which token each permuted row is. Off by default: one gather4 moves 512 B
    // and measured ~70 SM cycles each, so the GEMM's producer becomes the bottleneck
    // (r01: decode 0.533 vs 0.451 ms, prefill 37.5 vs 19.1 ms with the copy).
    c->gather_now = c->gather && !c->fp8;
    if (c->gather_now && !encode_map(&c->tm_src, tokens, 2, c->d, (uint64_t)T, 1, 1))
        return fail(c, MOE_ERR_CUDA, "cuTensorMapEncodeTiled(tokens) failed");
    r.dst_rows = c->gather_now ? nullptr : c->x_perm;
    r.src_row = c->gather_now ? c->src_row : nullptr;
    const GemmPaths gpaths = gemm_paths(c, (int64_t)T * c->k);
    c->spec_now = c->spec_l2 > 0 && gpaths.swap1 && !c->gather_now && T >= 16 && T <= 128 && !c->profiling;
    r.early = c->spec_now;
    moe_status s2 = route_and_permute(c, r, st);
    c->spec_now = c->spec_now && s2 == MOE_OK;
    if ((s = s2)) return s;
    int splits = 1;
    const bool residual = (c->cfg.flags & MOE_FLAG_RESIDUAL) != 0;
    // in-kernel combine by the fused FFN (tuning.fused_combine; single GPU, one combine task
    // per CTA). Into device memory the combine kernel after the fused FFN is faster: graph-
    // replayed 64-token decode 0.4066-0.4073 ms in-kernel vs 0.4029-0.4036 ms (3 of 3
    // interleaved rounds, profiles/r03/fused_ab.md). Into mapped host memory (moe_forward_host,
    // the default auto mode) the in-kernel combine wins: each 256-column slice crosses the
    // host link as soon as its w2 tiles are done instead of the whole output after the last
    // tile -- e2e 0.4155-0.4156 vs 0.4183-0.4184 ms (3 of 3)
    c->fcomb = moe_ctx::FusedCombine{};
    c->fcomb_done = false;
    const bool fcomb_want = c->fused_combine_mode == 1 || (c->fused_combine_mode == 0 && c->host_out_now);
    if (!tp && fcomb_want && T <= 256) {
        c->fcomb.on = true;
        c->fcomb.T = T;
        c->fcomb.x = residual ? tokens : nullptr;
        c->fcomb.out = out;
        c->fcomb.out_f32 = aux ? aux->out_f32 : nullptr;
    }
    s = run_gemms(c, gpaths, T, (int64_t)T * c->k, (int64_t)T * c->k, &splits, st);
    c->spec_now = false;
    c->fcomb.on = false;
    if (s) return s;
    if ((s = copy_aux(c, aux, T, st)) || (s = copy_aux_segments(c, aux, st))) return s;
    if (c->fcomb_done) return MOE_OK;  // the fused FFN wrote out / out_f32

    CombineParams cp{};
    cp.y = c->y;
    cp.split_stride = c->split_stride;
    cp.splits = splits;
    cp.pos = c->pos;
    cp.topk_w = c->topk_w;
    cp.T = T; cp.d = c->d; cp.k = c->k;
    if (!tp) {
        cp.x = residual ? static_cast<const __nv_bfloat16*>(tokens) : nullptr;
        cp.out = static_cast<__nv_bfloat16*>(out);
        cp.out_f32 = aux ? aux->out_f32 : nullptr;
        return launch_combine(c, cp, T, st);
    }
    if (c->nvls) {
        // ---- TP over NVLink SHARP (MOE_FLAG_NVLS, nvls.cu): combine, switch-side fp32 sum,
        // one rounding and the all-gather in ONE kernel (multimem on a symmetric window)
        moe_nvls::CombineArgs na{c->y, c->split_stride, splits, c->pos, c->topk_w,
                                 residual ? static_cast<const __nv_bfloat16*>(tokens) : nullptr, T, c->d, c->k,
                                 static_cast<__nv_bfloat16*>(out), aux ? aux->out_f32 : nullptr};
        StepTimer tn(c, kSlotCombine, st);
        cudaError_t ce = moe_nvls::launch_tp_combine(c->nvls, na, std::min(T, c->nvls_blocks),
                                                     !(c->cfg.flags & MOE_FLAG_NO_PDL), st);
        if (ce != cudaSuccess) return fail(c, MOE_ERR_CUDA, "NVLS combine launch failed: %s", cudaGetErrorString(ce));
        c->launch_count++;
        tn.done();
        return MOE_OK;
    }
    // ---- TP: fp32 partial of this rank's ffn slice -> fp32 reduce-scatter ->
    // one bf16 rounding (+ residual) -> bf16 all-gather (R7: single rounding)
    cp.x = nullptr;
    cp.out = nullptr;
    cp.out_f32 = c->tp_partial;
    if (c->p2p) {
        // reduce-scatter by stores: each token's fp32 partial goes to its owner's slot
        cp.out_f32 = nullptr;
        cp.peers = c->d_peers; cp.peer_off = c->so.tp_slots;
        cp.G = c->tp_world; cp.my_rank = c->tp_rank; cp.shard_max = c->tp_shard_max;
        cp.p2p_ticket = c->p2p_tickets + 2; cp.p2p_sig_off = c->so.sig + 8 * 2;
    }
    if ((s = launch_combine(c, cp, T, st)))
        return s;
    if (c->p2p) {
        const int G = c->tp_world, r = c->tp_rank;
        const int t0 = (int)((int64_t)r * T / G), n = (int)((int64_t)(r + 1) * T / G) - t0;
        float* of32 = aux ? aux->out_f32 : nullptr;
        StepTimer t1(c, kSlotExchange, st);
        if ((s = p2p_wait(c, 2, st))) return s;
        t1.done();
        const int fb = (int)std::max<int64_t>(1, std::min<int64_t>(4 * c->num_sms, ((int64_t)n * c->d / 4 + 255) / 256));
        if ((s = launch(c, kSlotCombine, moe_tp_p2p_finish_kernel, dim3(fb), dim3(256), 0, st,
                        reinterpret_cast<const float*>(c->sym + c->so.tp_slots), G, c->tp_shard_max, t0, n, c->d,
                        residual ? static_cast<const __nv_bfloat16*>(tokens) : nullptr,
                        static_cast<__nv_bfloat16*>(out), of32, reinterpret_cast<__nv_bfloat16*>(c->sym + c->so.tp_keep16),
                        reinterpret_cast<float*>(c->sym + c->so.tp_keep32), static_cast<uint8_t* const*>(c->d_peers),
                        c->p2p_tickets + 3, c->so.sig + 8 * 3)))
            return s;
        StepTimer t2(c, kSlotExchange, st);
        if ((s = p2p_wait(c, 3, st))) return s;
        const int pb = (int)std::max<int64_t>(1, std::min<int64_t>(4 * c->num_sms, ((int64_t)T * c->d / 8 + 255) / 256));
        if ((s = launch(c, kSlotExchange, moe_tp_p2p_pull_kernel, dim3(pb), dim3(256), 0, st,
                        static_cast<uint8_t* const*>(c->d_peers), c->so.tp_keep16, c->so.tp_keep32, G, r, T, c->d,
                        static_cast<__nv_bfloat16*>(out), of32)))
            return s;
        t2.done();
        return MOE_OK;
    }
    const int64_t n = (int64_t)T * c->d, cnt = n / c->G, base = cnt * c->rank;
    const CommRef tpc = tp_comm(c);
    ncclComm_t comm = c->cfg.nccl_comm;
    StepTimer t1(c, kSlotExchange, st);
    if ((s = comm_reduce_scatter_f32(c, tpc, c->tp_partial, c->tp_scatter, (size_t)cnt, st))) return s;
    t1.done();
    float* of32 = aux ? aux->out_f32 : nullptr;
    const int blocks = (int)std::min<int64_t>(4 * c->num_sms, (cnt / 4 + 255) / 256 + 1);
    if ((s = launch(c, kSlotCombine, moe_tp_finish_kernel, dim3(blocks), dim3(256), 0, st,
                    static_cast<const float*>(c->tp_scatter), cnt, base,
                    residual ? static_cast<const __nv_bfloat16*>(tokens) : nullptr, static_cast<__nv_bfloat16*>(out),
                    of32)))
        return s;
    StepTimer t2(c, kSlotExchange, st);
    NcclGroup grp;
    NCCL_TRY(c, grp.start(as_loopback(comm) == nullptr));
    if ((s = comm_allgather_inplace(c, tpc, out, (size_t)cnt, ncclBfloat16, 2, st))) return s;
    if (of32 && (s = comm_allgather_inplace(c, tpc, of32, (size_t)cnt, ncclFloat32, 4, st))) return s;
    NCCL_TRY(c, grp.end());
    t2.done();
    return MOE_OK;
}

// ---- EP ("distributes experts of an MoE across GPUs"):
// route local tokens over all E experts -> bucket rows by destination rank into
// fixed-capacity send slots (dropless: cap = max_tokens*k per peer) -> NCCL
// all-to-all (bf16 rows + local-expert ids, -1 = empty slot) -> group the received
// rows by local expert (same K1/K2 machinery, k = 1) -> K3/K4 -> fp32 rows back to
// their slots -> NCCL all-to-all -> K5 combine at the source rank.
// EP over peer memory (MOE_FLAG_P2P): the dispatch permute stores each routed row
// into its slot of the destination's receive buffer, the gather kernel stores each
// expert-output row into the source's return buffer; one arrival counter per
// exchange. Same slots, same arithmetic as the NCCL capacity path.
moe_status forward_ep_p2p(moe_ctx* c, const void* tokens, int32_t T, const void* router_w, void* out,
                          const moe_aux* aux, cudaStream_t st) {
    moe_status s;
    const int G = c->ep_world, me = c->ep_rank;
    const int cap = c->max_T * c->k;
    const int64_t R = (int64_t)cap * G;
    uint8_t* const* peers = c->d_peers;
    StepTimer t1(c, kSlotDispatch, st);
    // folded dispatch: T <= 64 (the router's blocks -- 16 tokens each on the tensor-core router,
    // 2 on the CUDA-core one -- are all resident while they wait for the scan)
    // Opt-in (tuning.ep_fold = 2): on one GPU shared by two P2P ranks the folded dispatch measured
    // 0.768-0.774 vs 0.748 ms per EP step (the router's 1-4 blocks copy the rows where the
    // permute spreads them over T/2 blocks; profiles/r03/experiments/ab_ep_fold_one_gpu.txt)
    const bool fold = T > 0 && T <= 64 && c->ep_fold_mode == 2;
    if (T > 0) {
        RouteSpec r;
        r.x = tokens; r.T = T; r.k = c->k; r.router_w = router_w;
        r.key_lo = 0; r.key_div = c->E_local; r.nkeys = G; r.seg_align = 1;
        r.logits = aux ? aux->logits : nullptr;
        r.topk_idx = c->topk_idx; r.topk_w = c->topk_w;
        r.pos = c->pos; r.pos_aux = aux ? aux->pos : nullptr;
        r.dst_rows = nullptr; r.cap = cap; r.meta = nullptr;
        r.peers = peers; r.peer_rows_off = c->so.ep_rows; r.peer_meta_off = c->so.ep_meta; r.my_rank = me;
        // small batches: the router's blocks (<= 32, all resident) dispatch their own rows after
        // the scan (EP dispatch issued by the router; no permute / fill launch)
        r.fold = fold;
        r.fold_ticket = c->p2p_tickets + 0;
        r.fold_sig_off = c->so.sig + 8 * 0;
        if ((s = route_and_permute(c, r, st))) return s;
        if ((s = copy_aux(c, aux, T, st))) return s;
    }
    if (!fold) {
        // this rank's unused slots in every destination's receive buffer -> -1
        const int fbx = std::max(1, std::min(64, (cap + 255) / 256));
        if ((s = launch(c, kSlotDispatch, moe_ep_p2p_fill_kernel, dim3(fbx, G), dim3(256), 0, st, peers, c->so.ep_meta,
                        T > 0 ? static_cast<const int32_t*>(c->counts) : nullptr, G, cap, me, c->p2p_tickets + 0,
                        c->so.sig + 8 * 0)))
            return s;
    }
    if ((s = p2p_wait(c, 0, st))) return s;
    t1.done();
    // receive side: as the NCCL path, over this rank's region
    RouteSpec r2;
    r2.x = c->sym + c->so.ep_rows; r2.T = (int)R; r2.k = 1;
    r2.in_idx = reinterpret_cast<const int32_t*>(c->sym + c->so.ep_meta); r2.in_w = nullptr; r2.allow_neg = 1;
    r2.key_lo = 0; r2.key_div = 1; r2.nkeys = c->E_local; r2.seg_align = kSegAlign;
    r2.topk_idx = c->ep_ridx; r2.topk_w = c->ep_rw; r2.pos = c->ep_rpos;
    r2.dst_rows = c->x_perm;
    if ((s = route_and_permute(c, r2, st))) return s;
    if ((s = copy_aux_segments(c, aux, st))) return s;
    const int64_t rows_expected = (int64_t)T * c->k;
    int splits = 1;
    if ((s = run_gemms(c, gemm_paths(c, rows_expected), std::min<int64_t>(R, (int64_t)G * c->max_T), R, rows_expected,
                       &splits, st)))
        return s;
    StepTimer t2(c, kSlotExchange, st);
    if ((s = launch(c, kSlotExchange, moe_ep_gather_kernel, dim3((unsigned)((c->d + 1023) / 1024 * R)), dim3(256), 0,
                    st, static_cast<const float*>(c->y), c->split_stride, splits,
                    static_cast<const int32_t*>(c->ep_rpos), (int)R, c->d, static_cast<float*>(nullptr), peers,
                    c->so.ep_yret, cap, me, G, c->p2p_tickets + 1, c->so.sig + 8 * 1)))
        return s;
    if ((s = p2p_wait(c, 1, st))) return s;
    t2.done();
    if (T == 0) return MOE_OK;
    CombineParams cp{};
    cp.y = reinterpret_cast<const float*>(c->sym + c->so.ep_yret);
    cp.split_stride = 0;
    cp.splits = 1;
    cp.pos = c->pos;
    cp.topk_w = c->topk_w;
    cp.x = (c->cfg.flags & MOE_FLAG_RESIDUAL) ? static_cast<const __nv_bfloat16*>(tokens) : nullptr;
    cp.T = T; cp.d = c->d; cp.k = c->k;
    cp.out = static_cast<__nv_bfloat16*>(out);
    cp.out_f32 = aux ? aux->out_f32 : nullptr;
    return launch_combine(c, cp, T, st);
}

moe_status forward_ep(moe_ctx* c, const void* tokens, int32_t T, const void* router_w, void* out,
                      const moe_aux* aux, cudaStream_t st) {
    moe_status s;
    c->gather_now = false;  // received rows are compacted into x_perm by the receive-side permute
    const int G = c->ep_world;
    const CommRef epc = ep_comm(c);
    const int64_t cap = (int64_t)c->max_T * c->k;
    const int64_t R = cap * G;
    ncclComm_t comm = c->cfg.nccl_comm;
    if (c->p2p) return forward_ep_p2p(c, tokens, T, router_w, out, aux, st);
    CUDA_TRY(c, cudaMemsetAsync(c->ep_meta_send, 0xFF, sizeof(int32_t) * R, st));  // all slots empty (-1)
    if (T > 0) {
        RouteSpec r;
        r.x = tokens; r.T = T; r.k = c->k; r.router_w = router_w;
        r.key_lo = 0; r.key_div = c->E_local; r.nkeys = G; r.seg_align = 1;
        r.logits = aux ? aux->logits : nullptr;
        r.topk_idx = c->topk_idx; r.topk_w = c->topk_w;
        r.pos = c->pos; r.pos_aux = aux ? aux->pos : nullptr;
        r.dst_rows = c->ep_send; r.cap = (int)cap; r.meta = c->ep_meta_send;
        if ((s = route_and_permute(c, r, st))) return s;
        if ((s = copy_aux(c, aux, T, st))) return s;
    }
    // Exchange. Capacity mode (decode): every peer gets its whole fixed-size bucket,
    // no host synchronisation (graph-capturable). Exact mode (large batches, or
    // MOE_FLAG_EP_EXACT): the per-destination counts are exchanged first and read
    // on the host (one stream sync), then only the occupied rows travel.
    const bool exact = (c->cfg.flags & MOE_FLAG_EP_EXACT) || cap * c->d * 2 * G > c->ep_exact_bytes;
    StepTimer t1(c, kSlotDispatch, st);
    const bool nccl = as_loopback(comm) == nullptr;
    if (exact) {
        if (T == 0) CUDA_TRY(c, cudaMemsetAsync(c->counts, 0, sizeof(int32_t) * G, st));
        if ((s = comm_alltoall(c, epc, c->counts, c->ep_rcounts, 1, ncclInt32, 4, st))) return s;
        CUDA_TRY(c, cudaMemcpyAsync(c->h_counts, c->counts, sizeof(int32_t) * G, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(c, cudaMemcpyAsync(c->h_counts + 64, c->ep_rcounts, sizeof(int32_t) * G, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(c, cudaStreamSynchronize(st));
        CUDA_TRY(c, cudaMemsetAsync(c->ep_meta_recv, 0xFF, sizeof(int32_t) * R, st));
        if ((s = comm_alltoallv(c, epc, c->ep_meta_send, c->ep_meta_recv, c->h_counts, c->h_counts + 64, cap, 1, ncclInt32,
                                4, st)))
            return s;
        if ((s = comm_alltoallv(c, epc, c->ep_send, c->ep_recv, c->h_counts, c->h_counts + 64, cap, c->d, ncclBfloat16, 2,
                                st)))
            return s;
    } else {
        NcclGroup grp;
        NCCL_TRY(c, grp.start(nccl));
        if ((s = comm_alltoall(c, epc, c->ep_meta_send, c->ep_meta_recv, (size_t)cap, ncclInt32, 4, st))) return s;
        if ((s = comm_alltoall(c, epc, c->ep_send, c->ep_recv, (size_t)(cap * c->d), ncclBfloat16, 2, st))) return s;
        NCCL_TRY(c, grp.end());
    }
    t1.done();
    // receive side: R slots (peer-major), k = 1, expert = meta (local index, -1 empty)
    RouteSpec r2;
    r2.x = c->ep_recv; r2.T = (int)R; r2.k = 1;
    r2.in_idx = c->ep_meta_recv; r2.in_w = nullptr; r2.allow_neg = 1;
    r2.key_lo = 0; r2.key_div = 1; r2.nkeys = c->E_local; r2.seg_align = kSegAlign;
    r2.topk_idx = c->ep_ridx; r2.topk_w = c->ep_rw; r2.pos = c->ep_rpos;
    r2.dst_rows = c->x_perm;
    if ((s = route_and_permute(c, r2, st))) return s;
    if ((s = copy_aux_segments(c, aux, st))) return s;
    // expected rows per rank ~ T*k (balanced routing); an expert gets at most G*max_T rows
    int64_t rows_expected = (int64_t)T * c->k;  // balanced routing: a rank receives about what it sends
    if (exact) {
        rows_expected = 0;
        for (int p = 0; p < G; ++p) rows_expected += c->h_counts[64 + p];
    }
    int splits = 1;
    if ((s = run_gemms(c, gemm_paths(c, rows_expected), std::min<int64_t>(R, (int64_t)G * c->max_T), R, rows_expected,
                       &splits, st)))
        return s;
    if ((s = launch(c, kSlotExchange, moe_ep_gather_kernel, dim3((unsigned)((c->d + 1023) / 1024 * R)), dim3(256), 0,
                    st, static_cast<const float*>(c->y), c->split_stride, splits,
                    static_cast<const int32_t*>(c->ep_rpos), (int)R, c->d, c->ep_ysend,
                    static_cast<uint8_t* const*>(nullptr), (int64_t)0, 0, 0, 0, static_cast<unsigned int*>(nullptr),
                    (int64_t)0)))
        return s;
    StepTimer t2(c, kSlotExchange, st);
    if (c->tp_world > 1) {
        // hybrid EP x TP: the rows' expert outputs are partial sums over this rank's
        // ffn slice; the TP group (same experts, same received rows) sums them in fp32
        const CommRef tpc = tp_comm(c);
        if (exact) {
            for (int p = 0; p < G; ++p)
                if (c->h_counts[64 + p] > 0 &&
                    (s = comm_allreduce_f32(c, tpc, c->ep_ysend + p * cap * c->d, (size_t)c->h_counts[64 + p] * c->d,
                                            st)))
                    return s;
        } else if ((s = comm_allreduce_f32(c, tpc, c->ep_ysend, (size_t)(R * c->d), st))) {
            return s;
        }
    }
    if (exact) {  // rows go back to where they came from: counts swap roles
        if ((s = comm_alltoallv(c, epc, c->ep_ysend, c->ep_yrecv, c->h_counts + 64, c->h_counts, cap, c->d, ncclFloat32, 4,
                                st)))
            return s;
    } else if ((s = comm_alltoall(c, epc, c->ep_ysend, c->ep_yrecv, (size_t)(cap * c->d), ncclFloat32, 4, st))) {
        return s;
    }
    t2.done();
    if (T == 0) return MOE_OK;
    CombineParams cp{};
    cp.y = c->ep_yrecv;
    cp.split_stride = 0;
    cp.splits = 1;
    cp.pos = c->pos;
    cp.topk_w = c->topk_w;
    cp.x = (c->cfg.flags & MOE_FLAG_RESIDUAL) ? static_cast<const __nv_bfloat16*>(tokens) : nullptr;
    cp.T = T; cp.d = c->d; cp.k = c->k;
    cp.out = static_cast<__nv_bfloat16*>(out);
    cp.out_f32 = aux ? aux->out_f32 : nullptr;
    return launch_combine(c, cp, T, st);
}

}  // namespace
