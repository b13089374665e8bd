// ffn_fused.cuh -- the decode expert FFN (steps a7 + a8 of SURVEY.md Sec. 8(a)) as ONE
// persistent kernel: the w1/w3 GEMM + SwiGLU tiles and the w2 GEMM tiles of every local
// expert are claimed from a single device-side work counter, and a w2 tile streams its
// weights as soon as it is claimed, waiting only for the h columns it multiplies.
//
//   GEMM1 (+SwiGLU): h[r, i] = bf16_rne( silu(x_r . W1_e[i,:]) * (x_r . W3_e[i,:]) )
//   GEMM2          : y_s[r, c] = sum_{i in split s} h[r, i] * W2_e[c, i]   (fp32 partial s)
// Same arithmetic, K order and partial-sum layout as the two-kernel swap-AB path
// (moe_gemm_kernel<kG1Swap> / <kG2Swap>, gemm_sm100.cuh): the combine adds the split
// partials in a fixed order, so results do not depend on which path ran
// (R1, R7; PAPER.md prints no formula for the block).
//
// Why: at decode the block is a weight stream (2.82 GB per Mixtral layer). Two kernels
// each pay a ramp and a tail (the w1/w3 GEMM's CTAs exit over ~10 us and the w2 GEMM
// only starts streaming after the last one; profiles/r02/experiments/timeline_r02.log),
// and at the per-rank shapes of EP/TP (E/G experts or f/G columns: 112-256 short units)
// those edges are a third of the step. Here the stream never stops: a CTA that runs out
// of w1/w3 tiles claims w2 tiles, whose dependency is the finished h tiles of that
// expert, tracked per (expert, 128-column ffn tile) by counters in global memory.
//
// Tiles (swap-AB: weights are the M operand, the expert's tokens the N operand):
//   G1 tile (e, m, n): W13 rows of ffn tile m (128 w1 rows + 128 w3 rows) x token tile n
//       -> h[:, 128m .. 128m+128) of the tile's tokens; K = d.
//   G2 tile (s, e, m2, n): W2 rows [256 m2, 256 m2 + 256) (two M=128 MMAs sharing the token
//       operand, so h is read from L2 once per 256 weight rows) x token tile n, K = the
//       ffn tiles [split_j[s], split_j[s+1]) of split s -> y partial s.
// Both tile kinds stage 256 weight rows x 64 K (32 KB, one TMA box) + NB token rows x 64 K
// per pipeline stage and accumulate into two TMEM column blocks ([0, NB) and [128, 128+NB))
// of one of two accumulator slots, so one stage ring and one MMA loop serve both.
//
// Work order: G1 tiles (expert-major, ffn tile, token tile fastest), then G2 tiles
// (split-major, expert, weight tile, token tile fastest; splits tapered so the last are short). Every tile is claimed with an
// atomicAdd on sched[0] by the producer lane of a RUNNING CTA, so a claimed G2 tile only
// ever waits for G1 tiles claimed earlier by running CTAs: no dependency on a CTA that is
// not resident, deadlock-free at any grid size. The claimed index is handed to the MMA
// and epilogue warps through a small shared-memory ring (tile_full / tile_empty).
//
// h hand-off between CTAs: each G1 epilogue thread stores its h values (generic proxy),
// fences them towards the async proxy, the four epilogue warps meet on a named barrier,
// and one thread publishes with __threadfence + atomicAdd(ready[e][m]). A G2 producer
// reads the counters relaxed (batched), and when every ffn tile its next stages need is
// complete: fence.acq_rel.gpu (acquire pattern) + fence.proxy.async.global, then the TMA
// loads of h. Weight loads of a G2 tile never wait: they run up to the ring depth ahead
// of the h loads.
//
// sched[0] (claims), sched[1] (CTA exits) and ready[] are zero between launches: the last
// CTA to exit resets them (graph-replay safe, no host work).
#pragma once

#include "gemm_sm100.cuh"

#ifndef MOE_FUSED_BF16_G2_128
#define MOE_FUSED_BF16_G2_128 0  // bf16 w2 tiles of 128 rows x two K blocks per stage (A/B knob)
#endif

namespace moe {

struct FusedParams {
    GemmParams g;            // counts / offsets / E / d / f / h (g.out) / w_nt (W13 tiles per expert)
    float* y;                // fp32 partials [splits][rows, d]
    int64_t y_split_stride;  // elements between split buffers
    int32_t splits;          // S: K splits of the w2 tiles (over whole ffn tiles)
    int32_t w2_nt;           // W2 tiles (128 rows) per expert in the tiled layout
    int32_t* sched;          // [4] claims, CTA exits, finished G1 tiles (zero between launches)
    int32_t* ready;          // [E * (f/64)] finished G1 token tiles per (expert, 64 h columns)
    int32_t stages;          // pipeline stages used (1..kStages; 0 = all that fit)
    int32_t split_j[9];      // ffn-tile boundaries of the w2 K splits: 0 = j_0 < .. < j_S = f/128
    // In-kernel combine (single GPU, step a9; combine_T = 0: off, moe_combine_kernel runs
    // after): once every w2 tile of a 256-column slice m has stored its partial (arrive[m]),
    // "combine tasks" (slice m, comb_chunk tokens), one per CTA after the GEMM tiles, compute
    // out[t, slice] = bf16_rne(sum_j w_j * sum_s y_s[pos_j] (+ x[t])) in moe_combine_kernel's
    // exact order, so the results are bit-identical to the separate combine.
    int32_t combine_T;
    int32_t k;
    const int32_t* pos;          // [T, k] permuted row of each (token, choice), < 0: none
    const float* topk_w;         // [T, k]
    const __nv_bfloat16* x_res;  // residual rows (nullable)
    __nv_bfloat16* out;          // [T, d]
    float* out_f32;              // [T, d] (nullable)
    int32_t* arrive;             // [d / 256] finished w2 tiles per slice (zero between launches)
    int32_t comb_chunk;          // tokens per combine task; the host keeps the task count <= the grid
    // Split chaining (chain != nullptr): the w2 tile of split s > 0 waits until split s-1 of the
    // same output tile (e, m, n) has stored, then stores y = y + acc into the split-0 buffer, so
    // ((acc_0 + acc_1) + acc_2) + .. lands in one buffer -- the same sums in the same order as
    // the combine kernel adding S partial buffers, and the combine then reads one partial.
    // chain[i] = splits stored so far for output tile i (the tile's index within its split).
    int32_t* chain;
    // FP8 weights (FP8 instantiation; GemmParams h_sf / plane_rows / sf_nb as the two-kernel
    // FP8 path): per-row weight scales and per-token scales of the two-term E4M3 tokens
    const float* w13_scale;  // [E][2 f] (w1 rows then w3 rows of each 128-row block pair)
    const float* w2_scale;   // [E][d]
    const float* tok_scale;  // [rows] 2^-s of each permuted row
};

constexpr int kFusedTileRing = 8;  // claimed-tile hand-off ring depth
constexpr int kFusedEpiBar = 1;    // named barrier of the 4 epilogue warps

// HALF (small per-rank shapes, round 3): w1/w3 tiles of 128 rows -- 64 w1 + 64 w3 rows of
// one 64-column h tile, two 64-row TMA boxes per K block -- so the first wave of w1/w3 work
// spreads over twice as many CTAs; a stage then carries two K blocks of such a tile (32 KB
// of weights + 2 x NB token rows), and the epilogue pairs a (TMEM lanes 0-63) with b (lanes
// 64-127) through a shared-memory exchange buffer. w2 tiles are the same in both variants.
// FP8 (E4M3 weights, round 3): the two-kernel FP8 path's tiles (moe_gemm_fp8x_kernel) in the
// fused schedule, 32 KB of weights per stage in both phases. A w1/w3 stage = one 128-byte K
// chunk of a 256-row W13 tile + the hi and lo E4M3 terms of the NB token rows (stacked, N = 2 NB;
// kind::f8f6f4 MMAs, w1 and w3 halves into two accumulators). A w2 stage = TWO K chunks of a
// 128-row W2 tile, each with its hi / lo h rows and UE8M0 B-scale block (block-scaled
// kind::mxf8f6f4 MMAs, B scales copied into TMEM per chunk, A scales a constant 2^0 atom) --
// 256-row w2 tiles (two MMAs sharing the scales) measured slower. NB = 32 only.
template <int NB, bool HALF = false, bool FP8 = false>
struct FusedCfg {
    static constexpr int kABytes = 256 * 128;       // 256 weight rows x 64 bf16 (HALF G1: 2 x 128 rows x 64; FP8: x 128 E4M3)
    // FP8: a w2 stage carries TWO K chunks of a 128-row W2 tile (2 x 16 KB weights, 2 x the hi/lo
    // h rows, 2 scale blocks) -- the same weight bytes per stage as a w1/w3 stage, whose single
    // 128-byte K chunk of 256 rows uses half of the B region
    static constexpr bool kG2Pair = FP8 || (MOE_FUSED_BF16_G2_128 && !HALF);  // w2: 128-row tiles, 2 K units / stage
    static constexpr int kBBytes = FP8 ? 2 * 2 * NB * 128 : (HALF || kG2Pair ? 2 : 1) * NB * 128;  // token rows x 128 B (x 2 K blocks / terms)
    static constexpr int kSFBytes = FP8 ? 2 * 512 : 0;  // FP8 G2: the tile's B scale blocks of the stage's two K chunks
    static constexpr int kStageBytes = kABytes + kBBytes + kSFBytes;
    static constexpr int kXPitch = NB + 1;          // exchange row pitch in floats (bank-conflict free)
    static constexpr int kXBytes = HALF ? 64 * kXPitch * 4 : 0;
    static constexpr int kSfaBytes = FP8 ? 512 : 0;  // FP8: the constant A scale atom (UE8M0 127)
    static constexpr int kStagesRaw = (kSmemBudget - 2048 - kXBytes - kSfaBytes) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static constexpr int kSmemBytes = kStages * kStageBytes + kXBytes + kSfaBytes + 2048;
    static constexpr int kAccStride = FP8 ? 4 * NB : 256;  // TMEM columns per accumulator stage
    static constexpr int kG2Rows = kG2Pair ? 128 : 256;    // w2 tile rows (128: one MMA per K step)
    static constexpr uint32_t kSfaCol = 480, kSfbCol = 488;  // FP8 scale columns in TMEM
    static_assert(NB >= 16 && NB <= 128 && NB % 16 == 0, "fused tile: a/b accumulators of <= 128 columns");
    static_assert(!FP8 || (!HALF && NB == 32), "FP8 fused tiles: 32-row token tiles, 256-row w1/w3 tiles");
    static_assert(kStages >= 3, "pipeline too shallow");
};

struct FusedTile {
    bool g1;
    int32_t e, rows, b_row;  // expert, its rows, first token row of the tile (permuted buffer)
    int32_t m;               // G1: ffn tile; G2: 256-row weight tile
    int32_t hf;              // HALF G1: which 64 columns of ffn tile m
    int32_t s;               // G2: split
    int32_t kb0, nkb;        // K blocks (64 columns) of the tile
    int32_t n_valid;         // valid token columns
    int32_t pidx;            // G2: index of the output tile (e, m, n) within its split
    int32_t nt;              // token tiles of the expert
};

__device__ __forceinline__ int fused_nt(int rows, int NB) { return rows > 0 ? (rows + NB - 1) / NB : 0; }

// Tile lists (every role decodes the same claimed index t):
//   [0, total1)      G1 tiles, expert-major: (e, m, n), token tile fastest
//   [total1, total)  G2 tiles, split-major: (s, e, m256, n). Split s covers the ffn tiles
//                    [split_j[s], split_j[s+1]) -- by default tapered (the host gives the
//                    first splits the most K and the last the least), so the stream ends on
//                    the shortest tiles and the CTAs' exits bunch up.
template <int NB, bool HALF, bool FP8>
__device__ __forceinline__ void fused_decode(int t, const FusedParams& p, const int32_t* s_counts,
                                             const int32_t* s_offsets, int total1, int per_split, FusedTile& ti) {
    const int wt = p.g.f / 128 * (HALF ? 2 : 1);  // w1/w3 tiles per expert and token tile
    const int mt2 = p.g.d / FusedCfg<NB, HALF, FP8>::kG2Rows;
    ti.g1 = t < total1;
    ti.s = 0;
    if (!ti.g1) {
        t -= total1;
        ti.s = t / per_split;
        t -= ti.s * per_split;
    }
    ti.pidx = t;
    int e = 0;
    for (; e < p.g.E; ++e) {
        const int nt = fused_nt(s_counts[e], NB);
        const int n = nt * (ti.g1 ? wt : mt2);
        if (t < n) break;
        t -= n;
    }
    ti.e = e;
    ti.rows = s_counts[e];
    ti.nt = fused_nt(ti.rows, NB);
    const int n_idx = t % ti.nt;
    ti.m = t / ti.nt;
    ti.hf = 0;
    if (ti.g1 && HALF) {
        ti.hf = ti.m & 1;
        ti.m >>= 1;
    }
    // K units: 64 bf16 (K block) or 128 E4M3 (FP8 K chunk = one ffn tile of h)
    if (ti.g1) {
        ti.kb0 = 0;
        ti.nkb = p.g.d / (FP8 ? 128 : 64);
    } else {
        ti.kb0 = (FP8 ? 1 : 2) * p.split_j[ti.s];
        ti.nkb = (FP8 ? 1 : 2) * (p.split_j[ti.s + 1] - p.split_j[ti.s]);
    }
    ti.b_row = s_offsets[e] + n_idx * NB;
    const int rem = ti.rows - n_idx * NB;
    ti.n_valid = rem < NB ? rem : NB;
}

__device__ __forceinline__ int ld_relaxed_gpu(const int32_t* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// tmW13: W13 tiled map (box 64 x 256 rows; HALF: 64 x 64 rows); tmX: permuted tokens (box
// 64 x NB); tmW2: W2 tiled map with 2-tile boxes (64 x 128 rows x 1 x 2 = 256 rows); tmH: h
// (box 64 x NB)
template <int NB, bool HALF, bool FP8 = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    moe_ffn_fused_kernel(const FusedParams p, const __grid_constant__ CUtensorMap tmW13,
                         const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW2,
                         const __grid_constant__ CUtensorMap tmH) {
    using C = FusedCfg<NB, HALF, FP8>;
    constexpr int S = C::kStages;
    constexpr int R = kFusedTileRing;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + S * C::kABytes;
    uint8_t* smem_sf = smem_b + S * C::kBBytes;                            // FP8: per-stage B scale blocks
    float* smem_x = reinterpret_cast<float*>(smem + S * C::kStageBytes);  // HALF: [64][kXPitch] b values
    uint8_t* smem_sfa = smem + S * C::kStageBytes + C::kXBytes;             // FP8: A scale atom
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes + C::kXBytes + C::kSfaBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tmem_full = bars + 2 * S;
    uint64_t* tmem_empty = bars + 2 * S + 2;
    uint64_t* tile_full = bars + 2 * S + 4;
    uint64_t* tile_empty = tile_full + R;
    int32_t* s_tile = reinterpret_cast<int32_t*>(tile_empty + R);       // [R]
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(s_tile + R);  // [1]
    int32_t* s_last = reinterpret_cast<int32_t*>(tmem_base_slot + 1);   // [1]
    int32_t* s_counts = s_last + 2;                                      // [32]
    int32_t* s_offsets = s_counts + 32;                                  // [33]

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    // ring depth in use: fewer bytes in flight per SM can stream faster when every SM
    // streams (scripts/exp/read_bw.cu: 3-4 stages of 32 KB peak)
    const int SR = p.stages > 0 && p.stages < S ? p.stages : S;
    MOE_TL(2, 0);
#if MOE_TIMELINE
    // probe build: slot 3 = [first w2-tile claim, last (failing) claim, entry + ns spent
    // waiting for h tiles] of this CTA's producer
    const unsigned long long tl_entry = ptx::tl_now();
    unsigned long long tl_stall = 0;
    bool tl_g2 = false;
#endif

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmW13);
        ptx::prefetch_tmap(&tmX);
        ptx::prefetch_tmap(&tmW2);
        ptx::prefetch_tmap(&tmH);
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tmem_full[i], 1);
            ptx::mbar_init(&tmem_empty[i], 4);
        }
        for (int i = 0; i < R; ++i) {
            ptx::mbar_init(&tile_full[i], 1);
            ptx::mbar_init(&tile_empty[i], 5);  // MMA lane + 4 epilogue warps
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc(tmem_base_slot, 512);
        ptx::tmem_relinquish();
        if (FP8) {  // A scales of the block-scaled w2 MMAs: UE8M0 127 = 2^0 for every row and K block
            reinterpret_cast<uint4*>(smem_sfa)[lane] = make_uint4(0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu);
            ptx::fence_proxy_async();  // generic-proxy stores visible to tcgen05.cp
        }
    }
    // Before the routing is known (PDL: the router / permute may still run): prefetch into
    // L2 the first K blocks of the w1/w3 tile this CTA most likely claims first, assuming
    // every expert holds one token tile (tile b = expert b / wt, ffn tile b % wt). A wrong
    // guess only costs the prefetch; whoever claims the tile reads it from L2. Issued by an
    // epilogue lane (idle until the first accumulator is ready): a CTA that starts late can
    // stall several us issuing prefetches into a busy memory system, and the producer must
    // not wait for that (timeline r03: post-wait stamps up to 9 us late when lane 0 issued).
    if (!FP8 && p.g.spec_l2 > 0 && threadIdx.x == 160) {
        const int wt = p.g.f / 128 * (HALF ? 2 : 1);
        if ((int)blockIdx.x < p.g.E * wt) {
            const int e = blockIdx.x / wt, m = (blockIdx.x % wt) / (HALF ? 2 : 1), hf = HALF ? blockIdx.x % 2 : 0;
            const int nk = min(p.g.spec_l2, p.g.d / kBK);
            for (int kb = 0; kb < nk; ++kb) {
                const WCoord w = wcoord(p.g, kb * kBK, m * 256 + 64 * hf, e);
                ptx::tma_prefetch_l2_4d(&tmW13, 0, w.c1, w.c2, w.c3);
                if (HALF) {  // the w3 rows of the same 64 columns
                    const WCoord w3 = wcoord(p.g, kb * kBK, m * 256 + 128 + 64 * hf, e);
                    ptx::tma_prefetch_l2_4d(&tmW13, 0, w3.c1, w3.c2, w3.c3);
                }
            }
        }
    }
    if (FP8 && p.g.spec_l2 > 0 && threadIdx.x == 160) {
        // the same guess for the E4M3 W13 tiles: 128-byte K chunks of 32 KB (half the K chunks
        // of the bf16 depth: a 256-row FP8 tile is 32 chunks)
        const int wt = p.g.f / 128;
        if ((int)blockIdx.x < p.g.E * wt) {
            const int e = blockIdx.x / wt, m = blockIdx.x % wt;
            const int nk = min(p.g.spec_l2 / 2, p.g.d / 128);
            for (int kq = 0; kq < nk; ++kq) ptx::tma_prefetch_l2_4d(&tmW13, 0, 0, kq, m + e * wt);
        }
    }
    ptx::pdl_wait();
    MOE_TL(2, 1);
    if (threadIdx.x < 32) {
        for (int e = threadIdx.x; e < p.g.E; e += 32) {
            s_counts[e] = p.g.counts[e];
            s_offsets[e] = p.g.offsets[e];
        }
    }
    // setup hand-off: producer + MMA warps sync with each other (barrier 2) and release the
    // epilogue warps (barrier 3) without waiting for them
    ptx::tc_fence_before();
    if (warp < 2) {
        ptx::named_bar_sync(2, 64);
        ptx::named_bar_arrive(3, 192);
    } else {
        ptx::named_bar_sync(3, 192);
    }
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_base_slot;

    const int wt = p.g.f / 128;
    const int wq = p.g.f / 64;  // 64-column h tiles per expert (readiness granularity)
    int total1 = 0, per_split = 0;
    for (int e = 0; e < p.g.E; ++e) {
        const int nt = fused_nt(s_counts[e], NB);
        total1 += nt * wt * (HALF ? 2 : 1);
        per_split += nt * (p.g.d / C::kG2Rows);
    }
    const int total = total1 + per_split * p.splits;
    // combine tasks after the GEMM tiles; a slice is complete after S * sum_e nt_e w2 tiles
    // Each CTA takes at most ONE combine task (sched[3]), after its producer found no GEMM tile
    // left: tasks queued behind each other in one CTA's epilogue would run back to back after
    // the last w2 tile (measured: +46 us at the 64-token decode with 8-token tasks claimed
    // like tiles). The host sizes the chunks so that ncomb <= gridDim.x.
    const int nchunk = p.combine_T > 0 ? (p.combine_T + p.comb_chunk - 1) / p.comb_chunk : 0;
    const int ncomb = (p.g.d / 256) * nchunk;
    const int total_all = total + ncomb;
    // (each w2 tile row range of kG2Rows columns counts towards its 256-column slice)
    const int slice_need = p.splits * (per_split / (p.g.d / C::kG2Rows)) * (256 / C::kG2Rows);
    const uint64_t w_hint = p.g.hint_a ? p.g.hint_a : ptx::kEvictFirst;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer (lane 0)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int ts = 0;
            uint32_t tph = 0;
            bool all_ready = false;  // every G1 tile of this launch finished (sched[2] == total1), acquired
            // A tile is claimed only when the previous one's loads are all issued (the ring still
            // holds SR stages of it, which hides the atomic's round trip). Claiming ahead was
            // measured slower: a CTA then holds two tiles at the end of the stream (tail) and,
            // at EP ranks, two waiting w2 tiles while G1 tiles run (profiles/r03).
            bool comb_taken = false;
            while (true) {
                int t = atomicAdd(&p.sched[0], 1);
                if (t >= total) {
                    const int cidx = (ncomb > 0 && !comb_taken) ? atomicAdd(&p.sched[3], 1) : ncomb;
                    comb_taken = true;
                    t = cidx < ncomb ? total + cidx : total_all;
                }
                ptx::mbar_wait(&tile_empty[ts], tph ^ 1);
                s_tile[ts] = t;
                ptx::mbar_arrive(&tile_full[ts]);
                if (++ts == R) { ts = 0; tph ^= 1; }
#if MOE_TIMELINE && !MOE_TL_TEARDOWN
                if (blockIdx.x < ptx::kTlBlocks) {
                    if (t >= total_all) {
                        ptx::g_moe_tl[3][1][blockIdx.x] = ptx::tl_now();
                        ptx::g_moe_tl[3][2][blockIdx.x] = tl_entry + tl_stall;
                    } else if (t >= total1 && !tl_g2) {
                        tl_g2 = true;
                        ptx::g_moe_tl[3][0][blockIdx.x] = ptx::tl_now();
                    }
                }
#endif
                if (t >= total_all) break;
                if (t >= total) continue;  // combine task: the epilogue warps only
                FusedTile ti;
                fused_decode<NB, HALF, FP8>(t, p, s_counts, s_offsets, total1, per_split, ti);
                if (!ti.g1 && !all_ready && ld_relaxed_gpu(&p.sched[2]) >= total1) {
                    fence_acq_rel_gpu();
                    fence_proxy_async_global();
                    all_ready = true;
                }
                if (FP8 && (ti.g1 || all_ready)) {
                    // w1/w3: one 128-byte K chunk per stage (256 weight rows, hi / lo token rows);
                    // w2: two K chunks per stage (128 weight rows + hi / lo h rows + scales each)
                    const int d128 = p.g.d / 128;
                    const int step = ti.g1 ? 1 : 2;
                    for (int kb = 0; kb < ti.nkb; kb += step) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = smem_a + stage * C::kABytes;
                        uint8_t* sb = smem_b + stage * C::kBBytes;
                        if (ti.g1) {
                            const int kq = ti.kb0 + kb;
                            ptx::mbar_arrive_expect_tx(&full[stage], C::kABytes + 2 * NB * 128);
                            ptx::tma_load_4d(&tmW13, &full[stage], sa, 0, 0, kq, ti.m + ti.e * wt, w_hint);
                            ptx::tma_load_3d(&tmX, &full[stage], sb, kq * 128, ti.b_row, 0, ptx::kEvictLast);
                            ptx::tma_load_3d(&tmX, &full[stage], sb + NB * 128, kq * 128, ti.b_row, 1, ptx::kEvictLast);
                        } else {
                            const int nc = min(2, ti.nkb - kb);
                            ptx::mbar_arrive_expect_tx(&full[stage], nc * (16384 + 2 * NB * 128 + 512));
                            for (int u = 0; u < nc; ++u) {
                                const int kq = ti.kb0 + kb + u;
                                ptx::tma_load_4d(&tmW2, &full[stage], sa + u * 16384, 0, 0, kq, ti.m + ti.e * d128, w_hint);
                                uint8_t* sbu = sb + u * 2 * NB * 128;
                                ptx::tma_load_3d(&tmH, &full[stage], sbu, kq * 128, ti.b_row, 0, ptx::kEvictLast);
                                ptx::tma_load_3d(&tmH, &full[stage], sbu + NB * 128, kq * 128, ti.b_row, 1, ptx::kEvictLast);
                                ptx::bulk_load(smem_sf + stage * C::kSFBytes + u * 512,
                                               p.g.h_sf + ((int64_t)(ti.b_row / NB) * wt + kq) * 512, 512, &full[stage]);
                            }
                        }
                        if (++stage == SR) { stage = 0; phase ^= 1; }
                    }
                } else if (HALF && ti.g1) {
                    // two K blocks per stage: [kb: 64 w1 rows | 64 w3 rows][kb+1: ...] + 2 x NB tokens
                    for (int kb = 0; kb < ti.nkb; kb += 2) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        uint8_t* sa = smem_a + stage * C::kABytes;
                        uint8_t* sb = smem_b + stage * C::kBBytes;
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const WCoord w1c = wcoord(p.g, (kb + u) * kBK, ti.m * 256 + 64 * ti.hf, ti.e);
                            const WCoord w3c = wcoord(p.g, (kb + u) * kBK, ti.m * 256 + 128 + 64 * ti.hf, ti.e);
                            ptx::tma_load_4d(&tmW13, &full[stage], sa + u * 16384, 0, w1c.c1, w1c.c2, w1c.c3, w_hint);
                            ptx::tma_load_4d(&tmW13, &full[stage], sa + u * 16384 + 8192, 0, w3c.c1, w3c.c2, w3c.c3,
                                             w_hint);
                            ptx::tma_load_2d(&tmX, &full[stage], sb + u * NB * 128, (kb + u) * kBK, ti.b_row,
                                             ptx::kEvictLast);
                        }
                        if (++stage == SR) { stage = 0; phase ^= 1; }
                    }
                } else if (C::kG2Pair && !ti.g1 && all_ready) {
                    // bf16 w2: two K blocks of a 128-row W2 tile per stage (2 x 16 KB + 2 x NB h rows)
                    for (int kb = 0; kb < ti.nkb; kb += 2) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        ptx::mbar_arrive_expect_tx(&full[stage], 2 * (16384 + NB * 128));
                        uint8_t* sa = smem_a + stage * C::kABytes;
                        uint8_t* sb = smem_b + stage * C::kBBytes;
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int kq = ti.kb0 + kb + u;
                            ptx::tma_load_4d(&tmW2, &full[stage], sa + u * 16384, 0, 0, kq, ti.m + ti.e * p.w2_nt, w_hint);
                            ptx::tma_load_2d(&tmH, &full[stage], sb + u * NB * 128, kq * kBK, ti.b_row, ptx::kEvictLast);
                        }
                        if (++stage == SR) { stage = 0; phase ^= 1; }
                    }
                } else if (ti.g1 || all_ready) {
                    for (int kb = 0; kb < ti.nkb; ++kb) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        ptx::mbar_arrive_expect_tx(&full[stage], C::kABytes + NB * 128);
                        uint8_t* sa = smem_a + stage * C::kABytes;
                        uint8_t* sb = smem_b + stage * C::kBBytes;
                        if (ti.g1) {
                            const WCoord w = wcoord(p.g, kb * kBK, ti.m * 256, ti.e);
                            ptx::tma_load_4d(&tmW13, &full[stage], sa, 0, w.c1, w.c2, w.c3, w_hint);
                            ptx::tma_load_2d(&tmX, &full[stage], sb, kb * kBK, ti.b_row, ptx::kEvictLast);
                        } else {
                            const int kq = ti.kb0 + kb;
                            ptx::tma_load_4d(&tmW2, &full[stage], sa, 0, 0, kq, 2 * ti.m + ti.e * p.w2_nt, w_hint);
                            ptx::tma_load_2d(&tmH, &full[stage], sb, kq * kBK, ti.b_row, ptx::kEvictLast);
                        }
                        if (++stage == SR) { stage = 0; phase ^= 1; }
                    }
                } else {
                    // Some G1 tiles still run: h loads of K block q need the 64 h columns of K block
                    // kb0 + q of expert e finished by all of its token tiles; weight loads run up to
                    // the ring depth ahead. ok = consecutive finished K blocks from kb0 (relaxed
                    // reads, then fence.acq_rel = acquire, then the proxy fence for the TMA reads).
                    constexpr int fpq = FP8 ? 2 : 1;  // 64-column readiness flags per K unit
                    const int32_t* rdy = p.ready + ti.e * wq + ti.kb0 * fpq;
                    const int nj = ti.nkb * fpq;
                    int ok = 0;
                    auto refresh = [&]() {
                        const int ok0 = ok;
                        while (ok < nj) {
                            int v[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) v[i] = ok + i < nj ? ld_relaxed_gpu(rdy + ok + i) : 0;
                            int c = 0;
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                if (c == i && ok + i < nj && v[i] >= ti.nt) ++c;
                            ok += c;
                            if (c < 8) break;
                        }
                        if (ok > ok0) {
                            fence_acq_rel_gpu();
                            fence_proxy_async_global();
                        }
                    };
                    const int st0 = stage;
                    int bq = 0;  // K blocks whose h load is issued
                    // K units of the stages: FP8 = pairs of K chunks (the last one may be single)
                    const int nunits = C::kG2Pair ? (ti.nkb + 1) / 2 : ti.nkb;
                    auto issue_b = [&](int q) {
                        const int sq = (st0 + q) % SR;
                        if (FP8) {
                            const int nc = min(2, ti.nkb - 2 * q);
                            for (int u = 0; u < nc; ++u) {
                                const int kq = ti.kb0 + 2 * q + u;
                                uint8_t* sb = smem_b + sq * C::kBBytes + u * 2 * NB * 128;
                                ptx::tma_load_3d(&tmH, &full[sq], sb, kq * 128, ti.b_row, 0, ptx::kEvictLast);
                                ptx::tma_load_3d(&tmH, &full[sq], sb + NB * 128, kq * 128, ti.b_row, 1, ptx::kEvictLast);
                                ptx::bulk_load(smem_sf + sq * C::kSFBytes + u * 512,
                                               p.g.h_sf + ((int64_t)(ti.b_row / NB) * wt + kq) * 512, 512, &full[sq]);
                            }
                        } else if (C::kG2Pair) {
                            const int nc = min(2, ti.nkb - 2 * q);
                            for (int u = 0; u < nc; ++u)
                                ptx::tma_load_2d(&tmH, &full[sq], smem_b + sq * C::kBBytes + u * NB * 128,
                                                 (ti.kb0 + 2 * q + u) * kBK, ti.b_row, ptx::kEvictLast);
                        } else {
                            ptx::tma_load_2d(&tmH, &full[sq], smem_b + sq * C::kBBytes, (ti.kb0 + q) * kBK, ti.b_row,
                                             ptx::kEvictLast);
                        }
                    };
                    auto unit_ok = [&](int q) {  // K unit q's h is ready
                        return (C::kG2Pair ? min(2 * q + 2, ti.nkb) : q + 1) * fpq <= ok;
                    };
                    auto wait_ready = [&](int q) {
#if MOE_TIMELINE
                        const unsigned long long w0 = !unit_ok(q) ? ptx::tl_now() : 0;
#endif
                        while (!unit_ok(q)) {
                            refresh();
                            if (!unit_ok(q)) __nanosleep(64);
                        }
#if MOE_TIMELINE
                        if (w0) tl_stall += ptx::tl_now() - w0;
#endif
                    };
                    for (int q = 0; q < nunits; ++q) {
                        // the stage about to be reused must have its h load in flight (its MMA
                        // frees it only after both operands arrived)
                        while (bq <= q - SR) {
                            wait_ready(bq);
                            issue_b(bq++);
                        }
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        const int ncq = C::kG2Pair ? min(2, ti.nkb - 2 * q) : 1;
                        ptx::mbar_arrive_expect_tx(&full[stage], FP8 ? ncq * (16384 + 2 * NB * 128 + 512)
                                                                 : C::kG2Pair ? ncq * (16384 + NB * 128)
                                                                              : C::kABytes + NB * 128);
                        uint8_t* sa = smem_a + stage * C::kABytes;
                        const int kq = ti.kb0 + q;
                        if (FP8) {
                            const int d128 = p.g.d / 128;
                            for (int u = 0; u < ncq; ++u)
                                ptx::tma_load_4d(&tmW2, &full[stage], sa + u * 16384, 0, 0, ti.kb0 + 2 * q + u,
                                                 ti.m + ti.e * d128, w_hint);
                        } else if (C::kG2Pair) {
                            for (int u = 0; u < ncq; ++u)
                                ptx::tma_load_4d(&tmW2, &full[stage], sa + u * 16384, 0, 0, ti.kb0 + 2 * q + u,
                                                 ti.m + ti.e * p.w2_nt, w_hint);
                        } else {
                            ptx::tma_load_4d(&tmW2, &full[stage], sa, 0, 0, kq, 2 * ti.m + ti.e * p.w2_nt, w_hint);
                        }
                        // weights of the first stages go out before the first readiness check
                        if (q == SR - 1 || q == nunits - 1 || (q >= SR && (q & 3) == 3)) {
                            if (!unit_ok(bq)) refresh();
                        }
                        while (bq <= q && unit_ok(bq)) issue_b(bq++);
                        if (++stage == SR) { stage = 0; phase ^= 1; }
                    }
                    while (bq < nunits) {
                        wait_ready(bq);
                        issue_b(bq++);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer (lane 0)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int ts = 0;
            uint32_t tph = 0;
            const uint32_t sfa = tmem_base + C::kSfaCol, sfb = tmem_base + C::kSfbCol;
            if (FP8) ptx::tmem_cp_32x128b_x4(sfa, ptx::make_smem_desc_rows16(ptx::smem_u32(smem_sfa)));
            while (true) {
                ptx::mbar_wait(&tile_full[ts], tph);
                const int t = s_tile[ts];
                ptx::mbar_arrive(&tile_empty[ts]);
                if (++ts == R) { ts = 0; tph ^= 1; }
                if (t >= total_all) break;
                if (t >= total) continue;
                FusedTile ti;
                fused_decode<NB, HALF, FP8>(t, p, s_counts, s_offsets, total1, per_split, ti);
                const uint32_t n_mma = (uint32_t)((ti.n_valid + 15) / 16 * 16);
                const uint32_t idesc = ptx::make_idesc_bf16(128, n_mma);
                const uint32_t d_tmem = tmem_base + acc * C::kAccStride;
                ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const bool half_g1 = HALF && ti.g1;
                const bool pair_g2 = C::kG2Pair && !ti.g1;  // two K units per stage
                for (int kb = 0; kb < ti.nkb; kb += (half_g1 || pair_g2) ? 2 : 1) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t sa = ptx::smem_u32(smem_a + stage * C::kABytes);
                    const uint32_t sb = ptx::smem_u32(smem_b + stage * C::kBBytes);
                    if (FP8) {
                        // hi and lo terms stacked: N = 2 NB; 32 bytes of K per MMA (+2 in the descriptor)
                        constexpr uint32_t N2 = 2 * NB;
                        const uint64_t a1 = ptx::make_smem_desc_sw128(sa);
                        const uint64_t b0 = ptx::make_smem_desc_sw128(sb);
                        if (ti.g1) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint32_t acc_in = (kb | kk) ? 1u : 0u;
                                const uint32_t id8 = (1u << 4) | ((N2 >> 3) << 17) | ((128u >> 4) << 24);  // D f32, E4M3
                                ptx::mma_e4m3(d_tmem, a1 + 2 * kk, b0 + 2 * kk, id8, acc_in);
                                ptx::mma_e4m3(d_tmem + N2, a1 + (16384 >> 4) + 2 * kk, b0 + 2 * kk, id8, acc_in);
                            }
                        } else {
                            const int nc = min(2, ti.nkb - kb);
                            for (int u = 0; u < nc; ++u) {
                                // this chunk's B scales -> TMEM (in order before its MMAs)
                                ptx::tmem_cp_32x128b_x4(sfb, ptx::make_smem_desc_rows16(
                                                                 ptx::smem_u32(smem_sf + stage * C::kSFBytes + u * 512)));
                                const uint64_t au = a1 + (u * 16384 >> 4);
                                const uint64_t bu = b0 + (u * 2 * NB * 128 >> 4);
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk) {
                                    const uint32_t acc_in = (kb | u | kk) ? 1u : 0u;
                                    const uint32_t sel = static_cast<uint32_t>(kk) << 30;  // K block kk of the chunk
                                    const uint32_t idmx = ptx::make_idesc_mx_e4m3(128, N2, kk, kk);
                                    ptx::mma_mx_e4m3(d_tmem, au + 2 * kk, bu + 2 * kk, idmx, acc_in, sfa | sel, sfb | sel);
                                }
                            }
                        }
                    } else if (pair_g2) {
                        const int nc = min(2, ti.nkb - kb);
                        for (int u = 0; u < nc; ++u) {
                            const uint64_t adesc = ptx::make_smem_desc_sw128(sa + u * 16384);
                            const uint64_t bdesc = ptx::make_smem_desc_sw128(sb + u * NB * 128);
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk) {
                                const uint32_t accum = (kb | u | kk) ? 1u : 0u;
                                ptx::mma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, accum);
                            }
                        }
                    } else if (half_g1) {
                        // A = [K block kb: 64 w1 + 64 w3 rows][K block kb+1], one M = 128 MMA per k16:
                        // a lands in TMEM lanes 0-63, b in lanes 64-127
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const uint64_t adesc = ptx::make_smem_desc_sw128(sa + u * 16384);
                            const uint64_t bdesc = ptx::make_smem_desc_sw128(sb + u * NB * 128);
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk) {
                                const uint32_t accum = (kb | u | kk) ? 1u : 0u;
                                ptx::mma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, accum);
                            }
                        }
                    } else {
                        const uint64_t adesc = ptx::make_smem_desc_sw128(sa);
                        const uint64_t adesc2 = ptx::make_smem_desc_sw128(sa + 128 * 128);
                        const uint64_t bdesc = ptx::make_smem_desc_sw128(sb);
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk) {
                            const uint32_t accum = (kb | kk) ? 1u : 0u;
                            ptx::mma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, accum);
                            ptx::mma_bf16(d_tmem + 128, adesc2 + 2 * kk, bdesc + 2 * kk, idesc, accum);
                        }
                    }
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == SR) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit(&tmem_full[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue (warps 2..5)
        const int q = warp & 3;
        const int r = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        int ts = 0;
        uint32_t tph = 0;
        while (true) {
            ptx::mbar_wait(&tile_full[ts], tph);
            const int t = s_tile[ts];
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tile_empty[ts]);
            if (++ts == R) { ts = 0; tph ^= 1; }
            if (t >= total_all) break;
            if (t >= total) {
                // ---- combine task: slice m = 256 columns, tokens [t0, t0 + comb_chunk)
                const int m = (t - total) / nchunk;
                const int t0 = ((t - total) % nchunk) * p.comb_chunk;
                if (lane == 0) {
                    while (ld_relaxed_gpu(p.arrive + m) < slice_need) __nanosleep(64);
                    fence_acq_rel_gpu();
                }
                __syncwarp();
                const int tid = (warp - 2) * 32 + lane;  // 0..127
                const int c = m * 256 + (tid & 63) * 4;
                for (int tt = t0 + (tid >> 6); tt < min(t0 + p.comb_chunk, p.combine_T); tt += 2) {
                    int32_t pr[2];
                    float w[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        pr[j] = j < p.k ? p.pos[(int64_t)tt * p.k + j] : -1;
                        w[j] = j < p.k ? p.topk_w[(int64_t)tt * p.k + j] : 0.f;
                    }
                    float4 sj[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        sj[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (pr[j] >= 0) sj[j] = __ldcg(reinterpret_cast<const float4*>(p.y + (int64_t)pr[j] * p.g.d + c));
                    }
                    for (int sp = 1; sp < (p.chain ? 1 : p.splits); ++sp)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            if (pr[j] >= 0) {
                                const float4 u = __ldcg(reinterpret_cast<const float4*>(
                                    p.y + sp * p.y_split_stride + (int64_t)pr[j] * p.g.d + c));
                                sj[j].x += u.x; sj[j].y += u.y; sj[j].z += u.z; sj[j].w += u.w;
                            }
                    float4 rr = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (pr[0] >= 0) rr = make_float4(w[0] * sj[0].x, w[0] * sj[0].y, w[0] * sj[0].z, w[0] * sj[0].w);
                    if (pr[1] >= 0) {
                        rr.x = fmaf(w[1], sj[1].x, rr.x); rr.y = fmaf(w[1], sj[1].y, rr.y);
                        rr.z = fmaf(w[1], sj[1].z, rr.z); rr.w = fmaf(w[1], sj[1].w, rr.w);
                    }
                    if (p.x_res) {
                        const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(p.x_res + (int64_t)tt * p.g.d + c);
                        const float2 a = __bfloat1622float2(xs[0]), b = __bfloat1622float2(xs[1]);
                        rr.x += a.x; rr.y += a.y; rr.z += b.x; rr.w += b.y;
                    }
                    if (p.out_f32) __stcs(reinterpret_cast<float4*>(p.out_f32 + (int64_t)tt * p.g.d + c), rr);
                    __nv_bfloat162 o0 = __floats2bfloat162_rn(rr.x, rr.y), o1 = __floats2bfloat162_rn(rr.z, rr.w);
                    uint2 ov;
                    ov.x = *reinterpret_cast<uint32_t*>(&o0);
                    ov.y = *reinterpret_cast<uint32_t*>(&o1);
                    *reinterpret_cast<uint2*>(p.out + (int64_t)tt * p.g.d + c) = ov;
                }
                continue;
            }
            FusedTile ti;
            fused_decode<NB, HALF, FP8>(t, p, s_counts, s_offsets, total1, per_split, ti);
            ptx::mbar_wait(&tmem_full[acc], acc_phase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + acc * C::kAccStride + (static_cast<uint32_t>(q * 32) << 16);
            const int nchunks = (ti.n_valid + 15) / 16;
            if (FP8 && ti.g1) {
                // columns [0, NB): w1 hi term, [NB, 2 NB): w1 lo, then the w3 accumulator (moe_gemm_fp8x_kernel's
                // epilogue): dequantise, SwiGLU, h -> two E4M3 planes + UE8M0 scales per 32 ffn columns
                // token scales of the tile's NB = 32 rows: one per lane, broadcast with shuffles (no
                // dependent global load per token inside the warp-synchronous loop below)
                const float ts_lane = lane < ti.n_valid ? p.tok_scale[ti.b_row + lane] : 0.f;
                const float* sc = p.w13_scale + (int64_t)ti.e * 2 * p.g.f + ti.m * 256;
                const float s1v = sc[r], s3v = sc[128 + r];
                const int64_t plane = p.g.plane_rows * p.g.f;
                uint8_t* hp = static_cast<uint8_t*>(p.g.out) + static_cast<int64_t>(ti.b_row) * p.g.f + ti.m * 128 + r;
                constexpr int snb = NB;
                constexpr int sfbytes = 512;
#pragma unroll 1
                for (int cc = 0; cc < nchunks; ++cc) {
                    uint32_t a0[16], a1[16], b0[16], b1[16];
                    ptx::tmem_ld16(tbase + cc * 16, a0);
                    ptx::tmem_ld16(tbase + NB + cc * 16, a1);
                    ptx::tmem_ld16(tbase + 2 * NB + cc * 16, b0);
                    ptx::tmem_ld16(tbase + 3 * NB + cc * 16, b1);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = cc * 16 + i;
                        const float tsn = __shfl_sync(0xffffffffu, ts_lane, n & 31);
                        if (n < ti.n_valid) {  // warp-uniform
                            const float av = __uint_as_float(a0[i]) + __uint_as_float(a1[i]);
                            const float bv = __uint_as_float(b0[i]) + __uint_as_float(b1[i]);
                            const float hv = silu_f32(av * (s1v * tsn)) * (bv * (s3v * tsn));
                            const uint32_t mbits = __reduce_max_sync(0xffffffffu, __float_as_uint(hv) & 0x7FFFFFFFu);
                            const float mx = __uint_as_float(mbits);
                            int u = 0;
                            if (mx > 0.f) {
                                const float ratio = 448.f / mx;
                                u = isinf(ratio) ? 120 : ((__float_as_int(ratio) >> 23) & 0xFF) - 127;
                                u = max(-120, min(120, u));
                            }
                            const float v = hv * __int_as_float((u + 127) << 23);
                            const uint8_t hi = f32_to_e4m3(v);
                            const uint8_t lo = f32_to_e4m3((v - e4m3_to_f32(hi)) * 16.f);
                            hp[static_cast<int64_t>(n) * p.g.f] = hi;
                            hp[static_cast<int64_t>(n) * p.g.f + plane] = lo;
                            if (lane < 2) {
                                const int64_t row = ti.b_row + n;
                                const int v_row = static_cast<int>(row % snb) + lane * snb;
                                const int64_t o = ((row / snb) * (p.g.f / 128) + ti.m) * sfbytes + 512 * (v_row / 128) +
                                                  16 * (v_row % 32) + 4 * ((v_row % 128) / 32) + q;
                                p.g.h_sf[o] = static_cast<uint8_t>((lane ? 123 : 127) - u);
                            }
                        }
                    }
                }
                fence_proxy_async_global();  // h planes + scales -> visible to the w2 tiles' TMA / bulk loads
            } else if (FP8) {
                // row 128 m + r (columns [0, NB): hi term, [NB, 2 NB): lo term)
                const int drow = ti.m * 128 + r;
                const float s2a = p.w2_scale[(int64_t)ti.e * p.g.d + drow];
                float* y = p.y + p.y_split_stride * ti.s + static_cast<int64_t>(ti.b_row) * p.g.d + drow;
#pragma unroll 1
                for (int cc = 0; cc < nchunks; ++cc) {
                    uint32_t v0[16], v1[16];
                    ptx::tmem_ld16(tbase + cc * 16, v0);
                    ptx::tmem_ld16(tbase + NB + cc * 16, v1);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = cc * 16 + i;
                        if (n < ti.n_valid)
                            y[static_cast<int64_t>(n) * p.g.d] = (__uint_as_float(v0[i]) + __uint_as_float(v1[i])) * s2a;
                    }
                }
            } else if (HALF && ti.g1) {
                // a of h column j (64 per tile) in TMEM lane j (warps q = 0, 1), b in lane 64 + j
                // (warps q = 2, 3): b goes through shared memory, warps 0 / 1 finish h
                if (q >= 2) {
                    float* xr = smem_x + (r - 64) * C::kXPitch;
#pragma unroll 1
                    for (int c = 0; c < nchunks; ++c) {
                        uint32_t b[16];
                        ptx::tmem_ld16(tbase + c * 16, b);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) xr[c * 16 + i] = __uint_as_float(b[i]);
                    }
                }
                ptx::named_bar_sync(kFusedEpiBar, 128);
                if (q < 2) {
                    const float* xr = smem_x + r * C::kXPitch;
                    __nv_bfloat16* h = static_cast<__nv_bfloat16*>(p.g.out) +
                                       static_cast<int64_t>(ti.b_row) * p.g.f + ti.m * 128 + 64 * ti.hf + r;
#pragma unroll 1
                    for (int c = 0; c < nchunks; ++c) {
                        uint32_t a[16];
                        ptx::tmem_ld16(tbase + c * 16, a);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int n = c * 16 + i;
                            if (n < ti.n_valid) {
                                const float hv = silu_f32(__uint_as_float(a[i])) * xr[n];
                                h[static_cast<int64_t>(n) * p.g.f] = __float2bfloat16_rn(hv);
                            }
                        }
                    }
                    fence_proxy_async_global();
                }
            } else if (ti.g1) {
                __nv_bfloat16* h = static_cast<__nv_bfloat16*>(p.g.out) + static_cast<int64_t>(ti.b_row) * p.g.f +
                                   ti.m * 128 + r;
#pragma unroll 1
                for (int c = 0; c < nchunks; ++c) {
                    uint32_t a[16], b[16];
                    ptx::tmem_ld16(tbase + c * 16, a);
                    ptx::tmem_ld16(tbase + 128 + c * 16, b);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = c * 16 + i;
                        if (n < ti.n_valid) {
                            const float hv = silu_f32(__uint_as_float(a[i])) * __uint_as_float(b[i]);
                            h[static_cast<int64_t>(n) * p.g.f] = __float2bfloat16_rn(hv);
                        }
                    }
                }
                fence_proxy_async_global();  // this thread's h stores -> visible to TMA readers
            } else {
                // rows 256 m + r (first MMA) and 256 m + 128 + r (second); 128-row tiles: 128 m + r
                const bool chained = p.chain != nullptr;
                float* y = p.y + (chained ? 0 : p.y_split_stride * ti.s) + static_cast<int64_t>(ti.b_row) * p.g.d +
                           ti.m * C::kG2Rows + r;
                const bool add = chained && ti.s > 0;
                if (add) {  // split s-1 of this output tile stored (acquire), then y += acc
                    if (lane == 0) {
                        while (ld_relaxed_gpu(p.chain + ti.pidx) < ti.s) __nanosleep(32);
                        fence_acq_rel_gpu();
                    }
                    __syncwarp();
                }
#pragma unroll 1
                for (int c = 0; c < nchunks; ++c) {
                    uint32_t v0[16], v1[16];
                    ptx::tmem_ld16(tbase + c * 16, v0);
                    if (C::kG2Rows == 256) ptx::tmem_ld16(tbase + 128 + c * 16, v1);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = c * 16 + i;
                        if (n < ti.n_valid) {
                            float* yn = y + static_cast<int64_t>(n) * p.g.d;
                            if (add) {
                                yn[0] = __ldcg(yn) + __uint_as_float(v0[i]);
                                if (C::kG2Rows == 256) yn[128] = __ldcg(yn + 128) + __uint_as_float(v1[i]);
                            } else {
                                yn[0] = __uint_as_float(v0[i]);
                                if (C::kG2Rows == 256) yn[128] = __uint_as_float(v1[i]);
                            }
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tmem_empty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            if (!ti.g1 && (p.combine_T > 0 || p.chain)) {
                // publish this tile's partial: the next split of the output tile (chain) and the
                // combine tasks of slice m
                ptx::named_bar_sync(kFusedEpiBar, 128);
                if (warp == 2 && lane == 0) {
                    __threadfence();
                    if (p.chain) atomicExch(p.chain + ti.pidx, ti.s + 1);
                    if (p.combine_T > 0) atomicAdd(p.arrive + ti.m * C::kG2Rows / 256, 1);
                }
            }
            if (ti.g1) {
                // publish: all four warps' h stores of this tile -> one release of ready[e][m]
                ptx::named_bar_sync(kFusedEpiBar, 128);
                if (warp == 2 && lane == 0) {
                    __threadfence();
                    if (HALF) {
                        atomicAdd(p.ready + ti.e * wq + 2 * ti.m + ti.hf, 1);
                    } else {
                        atomicAdd(p.ready + ti.e * wq + 2 * ti.m, 1);
                        atomicAdd(p.ready + ti.e * wq + 2 * ti.m + 1, 1);
                    }
                    atomicAdd(&p.sched[2], 1);
                }
            }
        }
    }
    ptx::pdl_launch_dependents();
    ptx::tc_fence_before();
    __syncthreads();
#if !MOE_TL_LATE_EXIT
    MOE_TL(2, 2);
#endif
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 512);
    }
    // last CTA out resets the claim / exit counters and the ready counters
    if (threadIdx.x == 0) {
        __threadfence();
#if MOE_TL_TEARDOWN
        ptx::g_moe_tl[3][0][blockIdx.x] = ptx::tl_now();
#endif
        *s_last = atomicAdd(&p.sched[1], 1) == (int)gridDim.x - 1;
#if MOE_TL_TEARDOWN
        ptx::g_moe_tl[3][1][blockIdx.x] = ptx::tl_now();
#endif
    }
    __syncthreads();
#if MOE_TL_TEARDOWN
    if (threadIdx.x == 0) ptx::g_moe_tl[3][2][blockIdx.x] = ptx::tl_now();
#endif
    if (*s_last) {
        __threadfence();
        const int nready = p.g.E * wq;  // 16-byte stores (cudaMalloc'd, 16-B aligned) + a tail
        for (int i = threadIdx.x; i < nready / 4; i += blockDim.x)
            reinterpret_cast<int4*>(p.ready)[i] = make_int4(0, 0, 0, 0);
        if (threadIdx.x < (nready & 3)) p.ready[(nready & ~3) + threadIdx.x] = 0;
        if (p.combine_T > 0)
            for (int i = threadIdx.x; i < p.g.d / 256; i += blockDim.x) p.arrive[i] = 0;
        if (p.chain)
            for (int i = threadIdx.x; i < per_split; i += blockDim.x) p.chain[i] = 0;
        if (threadIdx.x == 0) {
            p.sched[0] = 0;
            p.sched[1] = 0;
            p.sched[2] = 0;
            p.sched[3] = 0;
        }
    }
#if MOE_TL_LATE_EXIT
    MOE_TL(2, 2);  // probe: exit stamp after the counter hand-off (every CTA)
#endif
}

}  // namespace moe
