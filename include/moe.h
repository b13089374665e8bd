/* include/moe.h -- C ABI of libmoe: the batched Mixtral-8x7B sparse-MoE FFN block
 * on B200 (sm_100a).
 *
 * What the calls compute.  BASELINE.json north_star: "router GEMM, softmax,
 * top-2 expert selection with renormalised gate weights, token permutation by
 * expert, grouped SwiGLU expert GEMMs (w1/w3 then w2) and a weighted
 * scatter-combine back to token order", behind "moe_init / moe_forward(tokens
 * [T,4096], router_w, expert_w, out) / moe_destroy". PAPER.md names the model
 * (Sec. 2, Sec. 4.1, Sec. 5: Mixtral 8x7B) and the parallel
 * variants (Sec. 4.1: tensor parallel = "splitting tensors into
 * non-overlapping pieces", expert parallel = "distributes experts of an MoE
 * across GPUs") but prints no formula; the block is (reading R1):
 *     l = x W_g^T ; S = top-k(l) ; w_j = softmax(l)_{S_j} / sum_j' softmax(l)_{S_j'}
 *     y = sum_j w_j * W2_{S_j} ( silu(W1_{S_j} x) * (W3_{S_j} x) )
 * Precision contract (reading R7): bf16 inputs/weights; router logits, gates,
 * expert outputs and the combine in fp32; exactly two roundings to bf16 (the
 * SwiGLU activation h, and the final output, both round-to-nearest-even).
 *
 * Conventions.
 *   - All tensors are row-major, contiguous, 16-byte aligned device memory
 *     unless a parameter says "host". bf16 = IEEE bfloat16 bit patterns.
 *   - "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - The caller owns every buffer it passes (tokens, weights, out, aux) and
 *     the NCCL communicator; the library owns the context, its workspace and a
 *     TMA-descriptor cache. The library never frees or retains caller memory
 *     beyond the call that received it, except the descriptor cache, which
 *     stores weight *addresses* (not contents) and is keyed by them.
 *   - Calls validate their arguments BEFORE enqueuing anything; an invalid
 *     argument returns MOE_ERR_INVALID and nothing runs. Kernel launches are
 *     asynchronous; an asynchronous device fault surfaces as MOE_ERR_CUDA on a
 *     later call and is sticky (MOE_ERR_STATE thereafter for that context).
 *   - No exception crosses the ABI; the library never calls exit().
 *   - One host thread per context at a time, and the forwards of one context must be
 *     ordered on the device (one stream, or streams ordered by events): they share the
 *     context's workspace (permuted rows, h, fp32 partials) and, for the fused decode FFN,
 *     its device-side tile-claim / readiness counters, which each launch's last CTA resets.
 *   - There is no CPU fallback: every step of the forward runs in libmoe's own
 *     CUDA kernels on the device (sm_100a). A machine without an sm_100 GPU
 *     gets MOE_ERR_UNSUPPORTED from moe_init.
 */
#ifndef PAPER_2408_00008_B200_MOE_H
#define PAPER_2408_00008_B200_MOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_ABI_VERSION 2

#if defined(__GNUC__)
#define MOE_API __attribute__((visibility("default")))
#else
#define MOE_API
#endif

typedef struct moe_ctx moe_ctx; /* opaque, library-owned */

typedef enum {
    MOE_OK = 0,
    MOE_ERR_INVALID = 1,     /* bad argument; nothing was enqueued            */
    MOE_ERR_UNSUPPORTED = 2, /* shape / feature / device not supported        */
    MOE_ERR_OOM = 3,         /* workspace allocation failed in moe_init        */
    MOE_ERR_CUDA = 4,        /* CUDA launch or runtime failure (see last_error)*/
    MOE_ERR_NCCL = 5,        /* NCCL failure (EP / TP variants)                */
    MOE_ERR_STATE = 6        /* context poisoned by an earlier device fault    */
} moe_status;

/* Parallel variant (Sec. 4.1). */
typedef enum {
    MOE_PAR_NONE = 0, /* single GPU: all experts, all ffn columns                  */
    MOE_PAR_EP = 1,   /* expert parallel: rank r owns experts [r*E/G, (r+1)*E/G);
                         tokens are sharded by the caller (T may differ per rank);
                         rows are exchanged with NCCL all-to-all (bf16 out, fp32 back) */
    MOE_PAR_TP = 2,   /* tensor parallel: rank r owns ffn columns [r*f/G, (r+1)*f/G)
                         of every expert; every rank passes the same tokens; the
                         fp32 partial outputs are summed across ranks (all-reduce) */
    MOE_PAR_HYBRID = 3 /* EP x TP ("a hybrid of the two", P:337-349 EP2TP4 / EP4TP2):
                         G = ep * tp ranks, rank = ep_rank * tp + tp_rank (tp = tp_size).
                         EP group ep_rank owns experts [ep_rank*E/ep, ...) and each of
                         its tp ranks an ffn slice [tp_rank*f/tp, ...); the tp ranks of
                         an EP group pass the same tokens (the group's shard). Rows
                         travel over nccl_comm (the ep ranks with my tp_rank); expert
                         outputs are summed over tp_comm (the tp ranks of my group) */
} moe_par;

/* Flags (moe_config.flags). */
#define MOE_FLAG_RESIDUAL    0x1u /* out = x + MoE(x): C5 stack composition (reading R12) */
#define MOE_FLAG_FORCE_SWAP  0x2u /* always use the decode (weights-as-M, swap-AB) GEMMs */
#define MOE_FLAG_FORCE_TILED 0x4u /* always use the prefill (tokens-as-M) GEMMs          */
#define MOE_FLAG_NO_PDL      0x8u /* disable programmatic dependent launch               */
#define MOE_FLAG_NO_PAIR     0x10u /* prefill GEMMs on single CTAs (M=128) instead of CTA pairs (M=256) */
#define MOE_FLAG_FP8_WEIGHTS 0x40u /* expert weights are FP8 E4M3 with per-row power-of-two scales
                                      (moe_pack_weights_fp8); decode (swap-AB) GEMMs at any T
                                      (SURVEY 8(f) NEXT #2); hidden % 128 == 0. Both GEMMs run
                                      8-bit tensor-core MMAs: the w1/w3 GEMM on tokens split into
                                      two E4M3 terms (hi + lo == the bf16 token exactly above
                                      ~1e-3 of its row max), the w2 GEMM block-scaled
                                      (kind::mxf8f6f4) on h stored as two E4M3 terms with one
                                      UE8M0 scale per 32 ffn columns (R15)             */
#define MOE_FLAG_EP_EXACT    0x20u /* EP: always exchange exact row counts (one host sync per forward);
                                      default: exact only when a fixed-capacity exchange would move
                                      more than 32 MB, i.e. prefill-sized batches                  */
#define MOE_FLAG_GATHER      0x80u /* bf16, non-EP: the w1/w3 GEMM fetches token rows itself with TMA
                                      tile::gather4 instead of step 7 copying them into a permuted
                                      buffer. Bit-identical results; measured
                                      SLOWER on B200, so off by default            */

/* Tuning overrides (moe_config.tuning; NULL = the measured defaults). These change
 * only which kernel variant / grid / tile order runs, never the arithmetic of the
 * block: every setting is covered by the parity tests (tests/test_gpu_parity.py).
 * A zero field keeps the default; the library reads nothing from the environment
 * (except MOE_NCCL_LIB, the path of libnccl.so.2 to dlopen).                     */
typedef struct moe_tuning {
    int32_t g1_swap_rows;   /* w1/w3 GEMM on the decode (swap-AB) kernels while the mean rows
                               per local expert is <= this (0: 256); tiles beyond           */
    int32_t g2_swap_rows;   /* w2 GEMM, same rule (0: 256)                                   */
    int32_t g1_grid;        /* decode w1/w3 GEMM CTAs (0: auto)                */
    int32_t g2_grid;        /* decode w2 GEMM CTAs (0: auto)                                 */
    int32_t spec_l2;        /* decode speculative L2 weight prefetch, K blocks per CTA
                               (0: 48; < 0: off)                                              */
    int32_t swap_nb_cap;    /* cap the swap-AB token tile at 32/64/128 rows (0: no cap): an
                               expert with more rows runs several token tiles               */
    int32_t pair_nblk;      /* prefill CTA-pair tile width in 256-column blocks, 1 or 2 (0: 2) */
    int32_t pair_order;     /* prefill tile-order override (0: default): bits 0-1 w1/w3 order,
                               2-3 w2 order, 4-9 w1/w3 band, 10-15 w2 band (tiles)          */
    int32_t router_cc_max_T;/* CUDA-core router for T <= this (0: tensor-core router, E <= 8) */
    int32_t weight_hint;    /* L2 policy of the decode weight stream: 0 auto, 1 evict-first,
                               2 evict-normal, 3 evict-last                                  */
    int32_t host_stage;     /* moe_forward_host: 1 = always stage the output on the device and
                               copy it back (0: pinned output written directly)             */
    int32_t g1_nb;          /* force the swap-AB token tile of the w1/w3 GEMM: 32/64/128/192 (0: auto) */
    int32_t g2_nb;          /* same for the w2 GEMM, also 256 (0: auto)                        */
    int32_t pair_hints;     /* prefill CTA-pair L2 policies, 2 bits each (0 evict-normal, 1 evict-first,
                               2 evict-last): bits 0-1 w1/w3 tokens, 2-3 w1/w3 weights, 4-5 w2 h,
                               6-7 w2 weights (0: all evict-normal)                          */
    int32_t swap_pair;      /* swap-AB GEMMs on CTA pairs (cta_group::2, token tile split over
                               the pair): 0 auto (token tiles >= 128 rows), 1 off, 2 always
                               where the shape allows (w1/w3 needs ffn/tp_world % 256 == 0) */
    int32_t fused;          /* decode FFN as ONE persistent kernel (w1/w3 + SwiGLU and w2 tiles
                               claimed from one device work counter, w2 tiles waiting per
                               128-column h tile): 0 auto, 1 off, 2 on where the
                               shape allows (bf16, token tile <= 128 rows, hidden % 256 == 0) */
    int32_t fused_splits;   /* K splits of the fused kernel's w2 tiles, 1..8 (0: auto)        */
    int32_t fused_stages;   /* pipeline stages of the fused kernel, 2..8 (0: all that fit)     */
    int32_t fused_uniform;  /* 1: equal w2 K splits in whole ffn tiles (the two-kernel path's split,
                               bit-identical results); 0: tapered splits, the last ones shortest
                               (split i weighted 2^(S-1-i) where one split's w2 tiles cover half
                               the grid, else and for FP8 weights S-i); 2: weighted S-i;
                               3: weighted (S-i)^2; 4: weighted 2^(S-1-i)                       */
    int32_t fused_combine;  /* 1: single-GPU forwards of <= 256 tokens run step a9 inside the fused
                               FFN (combine tasks after the last w2 tiles; bit-identical); 2: the
                               combine kernel runs after it (faster into device memory); 0 (auto):
                               in-kernel where moe_forward_host writes mapped host memory, else 2 */
    int32_t fused_chain;    /* 1: the fused FFN's w2 tile of split s adds into buffer 0 after split
                               s-1 of the same output tile stored (same sums, same order; the
                               combine reads one partial); 0: S partial buffers the combine adds */
    int32_t fused_half;     /* fused FFN w1/w3 tiles of 128 rows (64 w1 + 64 w3 rows, a/b paired
                               through shared memory): 0 auto (where the 256-row tiles do not
                               fill the SMs), 1 off, 2 on                                      */
    int32_t combine_vec;    /* combine kernel: 4-column groups per thread, 1 or 4 (0: 1 up to 256
                               tokens -- more blocks for the latency-bound decode combine -- else 4) */
    int32_t ep_fold;        /* EP over peer memory, T <= 64: 2 = the router's blocks dispatch the rows
                               themselves after the scan (no permute / fill launch; bit-identical);
                               0 / 1 = the permute kernel dispatches (default: faster measured)  */
    int32_t reserved[8];    /* must be zero                                                  */
} moe_tuning;

typedef struct {
    int32_t hidden;      /* d: 4096 for Mixtral (C1: 64). Must be a multiple of 64.   */
    int32_t ffn;         /* f: 14336 for Mixtral (C1: 128). f/G must be a multiple of 128. */
    int32_t num_experts; /* E: 8 for Mixtral. 1 <= E <= 32; E % G == 0 for EP.       */
    int32_t top_k;       /* k: 2 for Mixtral; 1 is also supported. k <= E.           */
    int32_t max_tokens;  /* per-rank T capacity; sizes the workspace. >= 1.           */
    int32_t par;         /* moe_par                                                    */
    int32_t world_size;  /* G (1 for MOE_PAR_NONE)                                     */
    int32_t rank;        /* 0 <= rank < G                                              */
    void* nccl_comm;     /* ncclComm_t from moe_nccl_comm_init (caller-owned); EP/TP  */
    uint32_t flags;      /* MOE_FLAG_*                                                 */
    int32_t split_k;     /* decode w2 GEMM split-K factor; 0 = automatic               */
    int32_t device;      /* CUDA device ordinal the context binds to; -1 = current    */
    int32_t tp_size;     /* MOE_PAR_HYBRID: TP degree (world_size = ep * tp_size); else 0 */
    void* tp_comm;       /* MOE_PAR_HYBRID: communicator of my TP group; else NULL      */
    const moe_tuning* tuning; /* optional overrides (copied at moe_init); NULL = defaults */
    int32_t reserved[2]; /* must be zero                                               */
} moe_config;

/* Packed expert weights of THIS rank (device, produced by moe_pack_weights).
 *   w13 rows: 2*f_local per expert, w1 and w3 rows interleaved in blocks of 128:
 *        packed row 256*b + i     = w1 row 128*b + i  (i < 128)
 *        packed row 256*b + 128+i = w3 row 128*b + i
 *   w2 rows: d per expert (HF layout rows, ffn slice of this rank), zero rows
 *        appended up to a multiple of 256.
 *   bf16 (moe_pack_weights) -- TILED: the rows of each expert are cut into tiles
 *        (w13: 256 rows, w2: 128 rows) and each tile is stored as K/64 consecutive
 *        [tile_rows][64] blocks (K = d for w13, f_local for w2), so one 64-wide K
 *        step of one tile is one contiguous 32 / 16 KB range:
 *        element (e, row, k) of w13 at ((((e*T13 + row/256)*(d/64) + k/64)*256
 *        + row%256)*64 + k%64, T13 = 2*f_local/256 (w2 alike with 128, f_local, T2).
 *   FP8 (moe_pack_weights_fp8) -- TILED the same way with 128-byte K chunks: w13 tiles of
 *        256 rows, w2 tiles of 128 rows, each stored as K/128 consecutive [rows][128 B]
 *        blocks (one E4M3 byte per weight).
 * (E_local = E/ep, f_local = f/tp: EP ep = G, TP tp = G, hybrid ep * tp = G.)   */
typedef struct {
    const void* w13;
    const void* w2;
    const float* w13_scale; /* MOE_FLAG_FP8_WEIGHTS: [E_local, 2*f_local] fp32, packed row order */
    const float* w2_scale;  /* MOE_FLAG_FP8_WEIGHTS: [E_local, d] fp32; both NULL for bf16     */
} moe_expert_weights;

/* Optional debug / parity outputs (any pointer may be NULL). Device memory,
 * T = this call's token count on this rank.
 *   logits  [T, E] fp32  router logits, fp32 accumulation, never rounded to bf16
 *   topk_idx[T, k] int32 selected experts, slot 0 = larger logit, ties -> lower index
 *   topk_w  [T, k] fp32  renormalised gates
 *   expert_counts [E_local] int32 rows routed to each local expert
 *   expert_offsets [E_local+1] int32 first row of each expert's segment in the
 *                  permuted buffer (segments padded to multiples of 128 rows)
 *   pos     [T, k] int32 permuted row of each assignment (single-GPU / TP only)
 *   out_f32 [T, d] fp32  the combined output before the final bf16 rounding      */
typedef struct {
    float* logits;
    int32_t* topk_idx;
    float* topk_w;
    int32_t* expert_counts;
    int32_t* expert_offsets;
    int32_t* pos;
    float* out_f32;
} moe_aux;

/* Create a context bound to cfg->device: validates cfg, allocates the
 * workspace for max_tokens (permuted tokens, activations, fp32 expert outputs,
 * routing metadata; about 3.5 GB at max_tokens = 32768 for Mixtral), and
 * encodes the workspace TMA descriptors. Returns MOE_ERR_UNSUPPORTED if the
 * device is not sm_100. *out is set only on MOE_OK. */
MOE_API moe_status moe_init(const moe_config* cfg, moe_ctx** out);

/* Bytes of this rank's packed w13 / w2 buffers for cfg (no device work). */
MOE_API moe_status moe_packed_sizes(const moe_config* cfg, size_t* w13_bytes, size_t* w2_bytes);

/* Pack HF-layout weights (device, bf16) into this rank's layout (see
 * moe_expert_weights): w1, w3 [E, f, d], w2 [E, d, f] are the FULL model
 * tensors; the kernel extracts this rank's expert range (EP) or ffn slice (TP).
 * w13_out / w2_out must hold moe_packed_sizes bytes. Enqueued on stream. */
MOE_API moe_status moe_pack_weights(moe_ctx* ctx, const void* w1, const void* w3, const void* w2,
                            void* w13_out, void* w2_out, void* stream);

/* FP8 weights ("applying quantization techniques using ... 8-bit (fp8)").
 * q1, q3 [E, f, d] and q2 [E, d, f] are FP8 E4M3 bytes (HF layout, FULL model);
 * s1, s3 [E, f] and s2 [E, d] are fp32 per-output-row scales, each a power of two,
 * so that w = q * s exactly (the caller quantises; the library never rounds a
 * weight). Packs this rank's share like moe_pack_weights, plus the scales. The
 * context must have MOE_FLAG_FP8_WEIGHTS. Sizes from moe_packed_sizes_fp8.     */
MOE_API moe_status moe_packed_sizes_fp8(const moe_config* cfg, size_t* w13_bytes, size_t* w2_bytes,
                                        size_t* w13_scale_bytes, size_t* w2_scale_bytes);
MOE_API moe_status moe_pack_weights_fp8(moe_ctx* ctx, const void* q1, const void* q3, const void* q2,
                                        const float* s1, const float* s3, const float* s2, void* w13_out,
                                        void* w2_out, float* w13_scale_out, float* w2_scale_out, void* stream);

/* The block forward. tokens [T, d] bf16, router_w [E, d] bf16 (full, replicated
 * on every rank), out [T, d] bf16. 0 <= T <= max_tokens. T == 0 enqueues nothing
 * (except the EP collectives, in which every rank takes part). No host
 * synchronisation on the single-GPU and TP paths, so they are CUDA-graph
 * capturable; no allocation. aux may be NULL. */
MOE_API moe_status moe_forward(moe_ctx* ctx, const void* tokens, int32_t T, const void* router_w,
                       const moe_expert_weights* weights, void* out, const moe_aux* aux,
                       void* stream);

/* Same as moe_forward with the routing supplied by the caller (the oracle's
 * "forced routing" mode): topk_idx [T, k] int32
 * (distinct experts per token, each in [0, E)), topk_w [T, k] fp32 gates used
 * as given. Single-GPU and TP only. Indices are validated on the device: an
 * out-of-range index makes the routing kernel trap (MOE_ERR_CUDA later). */
MOE_API moe_status moe_forward_routed(moe_ctx* ctx, const void* tokens, int32_t T, const int32_t* topk_idx,
                              const float* topk_w, const moe_expert_weights* weights, void* out,
                              const moe_aux* aux, void* stream);

/* End-to-end call with HOST token/output buffers (ideally pinned): copies
 * tokens_host [T, d] bf16 to a library-owned device buffer, runs moe_forward,
 * copies the result to out_host [T, d] bf16, all enqueued on stream. The caller
 * synchronises the stream before reading out_host. */
MOE_API moe_status moe_forward_host(moe_ctx* ctx, const void* tokens_host, int32_t T, const void* router_w,
                            const moe_expert_weights* weights, void* out_host, void* stream);

/* Release the context and its workspace. NULL is a no-op. */
MOE_API moe_status moe_destroy(moe_ctx* ctx);

/* Last error text of ctx (or of the last failed moe_init when ctx == NULL). */
MOE_API const char* moe_last_error(const moe_ctx* ctx);
MOE_API const char* moe_status_string(moe_status s);

/* Instrumentation (bench.py).
 * moe_set_profiling(ctx, 1): every subsequent forward records a CUDA event pair
 *   around each kernel on the launch stream; moe_kernel_times returns, per
 *   kernel slot, the summed milliseconds and launch count since the last
 *   moe_reset_profile (it synchronises on the recorded events). Slots:
 *   0 router, 1 permute, 2 gemm1(w1/w3+SwiGLU), 3 gemm2(w2), 4 combine,
 *   5 dispatch (EP), 6 exchange-back / all-reduce (EP/TP), 7 pack.
 * moe_launch_count: kernels libmoe launched since context creation.  */
#define MOE_NUM_KERNEL_SLOTS 8
MOE_API moe_status moe_set_profiling(moe_ctx* ctx, int enable);
MOE_API moe_status moe_reset_profile(moe_ctx* ctx);
MOE_API moe_status moe_kernel_times(moe_ctx* ctx, double* ms /*[8]*/, int64_t* launches /*[8]*/);
MOE_API int64_t moe_launch_count(const moe_ctx* ctx);

/* NCCL plumbing for the EP / TP variants (libnccl.so.2 is loaded at run time;
 * the single-GPU path never touches NCCL). id128: 128-byte ncclUniqueId buffer,
 * broadcast by the caller (e.g. over the host process group). */
MOE_API moe_status moe_nccl_unique_id(void* id128);
MOE_API moe_status moe_nccl_comm_init(const void* id128, int32_t world, int32_t rank, int32_t device,
                              void** comm);
MOE_API moe_status moe_nccl_comm_destroy(void* comm);

/* TEST TRANSPORT. A loopback "communicator" that emulates a G-rank group inside
 * ONE process on ONE device: G contexts (par EP/TP, world G, rank r, nccl_comm =
 * the rank handle) are driven by G host threads; each collective synchronises
 * the caller's stream, meets the other ranks at a host barrier and moves data
 * with device copies (fp32 sums in ascending rank order). It runs the exact EP /
 * TP device path so parity can be tested at G = 2..8 without G GPUs; it is not
 * a production transport (no overlap, host-synchronous, not graph-capturable).
 *   moe_loopback_comm_create(world, &group); moe_loopback_comm_rank(group, r, &comm_r);
 *   moe_loopback_comm_destroy(comm_r) for every rank handle, then (group).      */
MOE_API moe_status moe_loopback_comm_create(int32_t world, void** group);
MOE_API moe_status moe_loopback_comm_rank(void* group, int32_t rank, void** comm);
MOE_API moe_status moe_loopback_comm_destroy(void* group_or_rank);

/* ---- Peer-memory transport (MOE_FLAG_P2P, "NVLink").
 * The EP / TP exchange steps become stores and loads into the other ranks' device
 * memory issued by the kernels that produce / consume the rows (dispatch permute,
 * expert-output gather, TP combine / finish), completed by a device-side release
 * counter per exchange and a stream wait -- no NCCL call and no staging copy on
 * the data path. Each context owns one symmetric device region; the ranks of the
 * EP group (MOE_PAR_EP) or TP group (MOE_PAR_TP) exchange its handle once:
 *   1. every rank: moe_p2p_handle(ctx, buf)  -> MOE_P2P_HANDLE_BYTES opaque bytes
 *   2. all-gather the buffers over any host channel (a process-group all-gather, files ...)
 *   3. every rank: moe_p2p_connect(ctx, all, world)  (rank-ordered concatenation)
 * Handles of ranks in the same process are used directly (loopback tests: G ranks
 * on one GPU); others are opened with CUDA IPC (one process per GPU, or several
 * processes on one GPU). nccl_comm may be NULL with this flag. MOE_PAR_HYBRID is
 * not supported (MOE_ERR_UNSUPPORTED). moe_forward before moe_p2p_connect fails
 * with MOE_ERR_STATE. Every rank must call moe_forward the same number of times
 * (TP: with the same T), as with the NCCL transport. Forwards can be captured
 * into a CUDA graph: each exchange waits for its counter to reach G and resets it
 * (stream memory ops, the same values every forward; EP capacity mode).
 * Teardown: every rank's last forward must have completed on every rank (e.g.
 * stream sync + process-group barrier) before any rank calls moe_destroy, since
 * peers load from / store into this rank's region until then.                */
#define MOE_FLAG_P2P 0x100u

/* ---- NVLink SHARP all-reduce (MOE_FLAG_NVLS).
 * MOE_PAR_TP with an NCCL communicator from NCCL >= 2.28: moe_init (collective: every
 * rank of the TP group calls it) allocates a symmetric window with ncclMemAlloc,
 * registers it (NCCL_WIN_COLL_SYMMETRIC) and creates an NCCL device communicator with
 * multimem; every forward then ends in ONE kernel that forms this rank's fp32 partial
 * output, has the NVSwitch sum the ranks' partials (multimem.ld_reduce) for this rank's
 * column slice, rounds once to bf16 (+ residual) and multicasts the finished slice to
 * every rank (multimem.st), with device-side LSA barriers in between -- no separate
 * reduce-scatter / all-gather calls, and the forward stays graph-capturable. The switch
 * sums in its own order (fp32): results equal the collective path's up to fp32 rounding.
 * moe_init returns MOE_ERR_UNSUPPORTED when the process's NCCL has no device API or the
 * group has no multicast object (NVLS needs >= 2 GPUs on one NVSwitch domain).    */
#define MOE_FLAG_NVLS 0x200u
#define MOE_P2P_HANDLE_BYTES 128
MOE_API moe_status moe_p2p_handle(moe_ctx* ctx, void* handle_out);
MOE_API moe_status moe_p2p_connect(moe_ctx* ctx, const void* handles, int32_t world);

#ifdef __cplusplus
}
#endif
#endif /* PAPER_2408_00008_B200_MOE_H */
