// kernels.cuh -- the non-GEMM steps of the MoE block (CUDA cores, warp shuffles):
//   K1  router     : logits = x W_g^T (fp32), top-k, renormalised gates, per-block
//                    expert histogram, and (last block) the exclusive scan.   [a2-a5]
//   K2  permute    : stable rank of every assignment inside its expert segment,
//                    16-byte-vector scatter of token rows into the segments.  [a6]
//   K5  combine    : gate-weighted un-permute back to token order, fp32 sum,
//                    one bf16 RNE rounding.                                    [a9]
//   pack           : HF weights -> this rank's packed layout (init-time).
// Step labels refer to SURVEY.md Sec. 8(a); the math is BASELINE.json
// north_star's ("router GEMM, softmax, top-2 expert selection with renormalised
// gate weights, token permutation by expert ... weighted scatter-combine back to
// token order"), the paper being silent (R1-R7).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include "sm100.cuh"
#include "p2p.cuh"

namespace moe {

constexpr int kRouteThreads = 128;      // router block: 4 warps split the hidden dim
constexpr int kPermuteThreads = 256;    // permute block: 8 warps
constexpr int kSegAlign = 128;          // expert segments padded to the GEMM M tile

struct RouteParams {
    const __nv_bfloat16* x;   // [T, d]
    const __nv_bfloat16* wg;  // [E, d]
    const int32_t* in_idx;    // routed mode: caller's [T, k] (else nullptr)
    const float* in_w;        // routed mode: caller's gates [T, k]
    int32_t T, d, E, k;
    // histogram key of an assignment to expert e: (e - key_lo) / key_div, counted
    // when 0 <= key < nkeys. Local experts: key_lo = e_lo, key_div = 1, nkeys = E_local.
    // EP dispatch: key = destination rank (key_lo = 0, key_div = E/G, nkeys = G).
    int32_t key_lo, key_div, nkeys;
    int32_t seg_align;        // segment padding of the scan (128: GEMM M tile; 1: none)
    int32_t allow_neg;        // routed mode: negative expert index = empty slot (EP receive)
    float* logits;            // [T, E] optional debug output
    int32_t* topk_idx;        // [T, k] workspace
    float* topk_w;            // [T, k] workspace
    int32_t* rank;            // [T, k] stable rank of each assignment among same-key ones of its block
    int32_t* blockcount;      // [nblk, nkeys]
    int32_t* blockoff;        // [nblk, nkeys]
    int32_t* counts;          // [nkeys]
    int32_t* offsets;         // [nkeys + 1]
    unsigned int* done;       // block-completion counter (zero between launches)
    // decode speculative weight prefetch (moe.cu spec_l2): let the permute kernel (and
    // through it the w1/w3 GEMM) launch while this grid still runs
    int32_t early_trigger;
    // EP dispatch folded into the router (peer-memory transport, small batches; nullable
    // scan_epoch = off): the last block bumps scan_epoch after the scan; every block waits for
    // it and then does the permute kernel's dispatch for its own tokens -- positions, the rows
    // into the destination ranks' receive buffers, the meta entries -- fills its share of the
    // unused slots and takes part in the exchange's completion signal (p2p_signal_last_block).
    unsigned int* scan_epoch;
    uint8_t* const* peers;
    int64_t peer_rows_off, peer_meta_off, sig_off;
    int32_t cap, my_rank;
    int32_t* pos_aux;           // [T, k] optional copy of the positions
    unsigned int* p2p_ticket;
};

__device__ __forceinline__ int hist_key(int e, int key_lo, int key_div, int nkeys) {
    if (e < key_lo) return -1;
    const int q = (e - key_lo) / key_div;
    return q < nkeys ? q : -1;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// a4 + a5 for one router block whose routing sits in s_idx[ntok][2] (shared):
//   rank[t][j]      = #{(t', j') < (t, j) in this block with the same key} (stable order)
//   blockcount[b][] = assignments of this block per key
// then the last block to finish runs the exclusive scan over blocks (one block,
// fixed order: deterministic; classic threadfence-reduction handshake):
//   blockoff[b][key], counts[key], offsets[key] (segments padded to seg_align).
// Kept small on purpose: every loop over keys / warps / blocks runs with a runtime
// trip count and is not unrolled. The earlier form held 32-entry per-key register
// arrays with fully unrolled key loops (~6.7k SASS instructions per router kernel)
// and cost ~15 us per launch at decode even for T = 1 -- fixed cost of cold
// instruction fetch, since the 2.8 GB weight stream evicts the kernel's code from
// L2 every step (scripts/exp/router_lat.py).
template <int NTHREADS>
__device__ __forceinline__ void route_block_finish(const RouteParams& p, const int32_t (*s_idx)[2], int ntok,
                                                   int tok0) {
    constexpr int NW = NTHREADS / 32;
    __shared__ int s_last;
    __shared__ int32_t s_wk[NW][32];    // per-warp assignment count of every key
    __shared__ int32_t s_tot[32];
    const int NK = p.nkeys;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // thread i <-> assignment i = (token i / k, slot i % k); NTHREADS >= TB * k
    const int i = threadIdx.x;
    const bool valid = i < ntok * p.k;
    int key = -1;
    if (valid) {
        const int e = s_idx[i / p.k][i % p.k];
        if (p.k > 1 && (i % p.k) == 1 && e >= 0 && e == s_idx[i / p.k][0]) __trap();  // duplicate expert
        key = e >= 0 ? hist_key(e, p.key_lo, p.key_div, NK) : -1;
    }
    for (int j = threadIdx.x; j < NW * 32; j += NTHREADS) (&s_wk[0][0])[j] = 0;
    __syncthreads();
    // lanes with the same key: stable in-warp rank and the warp's count of that key
    const uint32_t same = __match_any_sync(0xffffffffu, key);
    const int32_t lrank = __popc(same & ((1u << lane) - 1u));
    if (key >= 0 && lrank == 0) s_wk[warp][key] = __popc(same);
    __syncthreads();
    if (key >= 0) {
        int32_t r = lrank;
#pragma unroll 1
        for (int w = 0; w < warp; ++w) r += s_wk[w][key];
        p.rank[(int64_t)tok0 * p.k + i] = r;
    } else if (valid) {
        p.rank[(int64_t)tok0 * p.k + i] = 0;
    }
    if (threadIdx.x < NK) {
        int32_t cnt = 0;
#pragma unroll 1
        for (int w = 0; w < NW; ++w) cnt += s_wk[w][threadIdx.x];
        p.blockcount[(int64_t)blockIdx.x * NK + threadIdx.x] = cnt;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // Exclusive scan over blocks, all keys at once: a group of R lanes (R = 32 / KP,
    // KP = keys per warp, a power of two) owns one key; lane g of the group owns the
    // contiguous run of blocks [g*per, (g+1)*per). Pass 1 sums the run (independent
    // loads), a shuffle scan inside the group gives each run's base, pass 2 writes the
    // per-block offsets. Fixed order: deterministic.
    int KP = 1;  // keys per warp: the smallest power of two with KP * NW >= NK
    while (KP * NW < NK && KP < 32) KP <<= 1;
    const int R = 32 / KP;                                   // lanes per key
    const int my_key = warp * KP + lane / R, g = lane % R;
    const int nblk = gridDim.x;
    const int per = (nblk + R - 1) / R;
    const int b0 = min(nblk, g * per), b1 = min(nblk, b0 + per);
    const bool own = my_key < NK;
    int32_t sum = 0;
    if (own) {
#pragma unroll 4
        for (int bb = b0; bb < b1; ++bb) sum += __ldcg(&p.blockcount[(int64_t)bb * NK + my_key]);
    }
    int32_t inc = sum;
#pragma unroll 1
    for (int o = 1; o < R; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, inc, o, R);
        if (g >= o) inc += u;
    }
    if (own) {
        int32_t ex = inc - sum;
#pragma unroll 1
        for (int bb = b0; bb < b1; ++bb) {
            p.blockoff[(int64_t)bb * NK + my_key] = ex;
            ex += __ldcg(&p.blockcount[(int64_t)bb * NK + my_key]);
        }
        if (g == R - 1) s_tot[my_key] = inc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t off = 0;
        p.offsets[0] = 0;
#pragma unroll 1
        for (int e = 0; e < NK; ++e) {
            p.counts[e] = s_tot[e];
            off += (s_tot[e] + p.seg_align - 1) / p.seg_align * p.seg_align;
            p.offsets[e + 1] = off;
        }
        *p.done = 0u;  // ready for the next forward (kernel boundary orders it)
        if (p.scan_epoch) {  // folded dispatch: the other blocks may read the offsets now
            __threadfence();
            atomicAdd(p.scan_epoch, 1u);
        }
    }
}

// Folded EP dispatch (RouteParams::scan_epoch): after route_block_finish, in every block of a
// router grid whose blocks are all resident (small batches). ep0 = scan_epoch read at kernel
// start (before this block's completion ticket, so before the scan can be published).
template <int NTHREADS, int TB>
__device__ __forceinline__ void route_fold_dispatch(const RouteParams& p, const int32_t (*s_idx)[2], int ntok,
                                                    int tok0, unsigned int ep0) {
    __shared__ int32_t s_ps[TB][2];
    if (threadIdx.x == 0) {
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.scan_epoch) : "memory");
            if (v == ep0) __nanosleep(32);
        } while (v == ep0);
    }
    __syncthreads();
    // positions: destination rank e (the histogram key), slot r = block offset + in-block rank
    if (threadIdx.x < ntok * p.k) {
        const int tl = threadIdx.x / p.k, j = threadIdx.x % p.k;
        const int t = tok0 + tl;
        const int ex = s_idx[tl][j];
        const int e = ex >= 0 ? hist_key(ex, p.key_lo, p.key_div, p.nkeys) : -1;
        int32_t ps = -1;
        if (e >= 0) {
            const int32_t r = __ldcg(&p.blockoff[(int64_t)blockIdx.x * p.nkeys + e]) + __ldcg(&p.rank[(int64_t)t * p.k + j]);
            ps = e * p.cap + r;
            int32_t* meta = reinterpret_cast<int32_t*>(p.peers[e] + p.peer_meta_off) + (int64_t)p.my_rank * p.cap + r;
            *meta = ex - e * p.key_div;  // expert index local to the destination
        }
        p.rank[(int64_t)t * p.k + j] = ps;  // rank[] doubles as the positions array (c->pos)
        if (p.pos_aux) p.pos_aux[(int64_t)t * p.k + j] = ps;
        s_ps[tl][j] = ps;
    }
    __syncthreads();
    // rows: 16-byte vectors of each routed token row into its slots of the destinations' buffers
    const int nvec = p.d / 8;
    for (int tl = 0; tl < ntok; ++tl) {
        const uint4* src = reinterpret_cast<const uint4*>(p.x + (int64_t)(tok0 + tl) * p.d);
        for (int j = 0; j < p.k; ++j) {
            const int32_t ps = s_ps[tl][j];
            if (ps < 0) continue;
            const int e = ps / p.cap, r = ps - e * p.cap;
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.peers[e] + p.peer_rows_off) +
                                                  ((int64_t)p.my_rank * p.cap + r) * p.d);
            for (int v = threadIdx.x; v < nvec; v += NTHREADS) dst[v] = __ldg(src + v);
        }
    }
    // this rank's unused slots [count_e, cap) of every destination's meta -> -1 (grid-stride)
    for (int e = 0; e < p.nkeys; ++e) {
        const int n0 = __ldcg(&p.counts[e]);
        int32_t* meta = reinterpret_cast<int32_t*>(p.peers[e] + p.peer_meta_off) + (int64_t)p.my_rank * p.cap;
        for (int i = n0 + blockIdx.x * NTHREADS + threadIdx.x; i < p.cap; i += gridDim.x * NTHREADS) meta[i] = -1;
    }
    p2p_signal_last_block(p.p2p_ticket, p.peers, p.nkeys, p.sig_off);  // the dispatch exchange is complete
}

// K1: router (a2, a3) + histogram / ranks (a4) + last-block exclusive scan (a5).
// A block owns TB consecutive tokens; its 128 threads split the hidden dimension
// in 8-element (16-byte) chunks, each thread accumulating TB x E partial dot
// products in fp32 (bf16*bf16 products are exact in fp32). W_g chunks are loaded
// once per thread and reused for the TB tokens. Partial sums are reduced with
// warp shuffles, then across the 4 warps in a fixed order (deterministic).
template <int E_MAX, int TB>
__global__ void __launch_bounds__(kRouteThreads) moe_router_kernel(const RouteParams p) {
    __shared__ float s_part[4][TB][E_MAX];
    __shared__ int32_t s_idx[TB][2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * TB;
    const int ntok = min(TB, p.T - tok0);

    ptx::pdl_wait();
    if (p.early_trigger) ptx::pdl_launch_dependents();
    const unsigned int ep0 = p.scan_epoch ? *reinterpret_cast<volatile unsigned int*>(p.scan_epoch) : 0u;

    if (p.in_idx == nullptr) {
        float acc[TB][E_MAX];
#pragma unroll
        for (int t = 0; t < TB; ++t)
#pragma unroll
            for (int e = 0; e < E_MAX; ++e) acc[t][e] = 0.f;
        // All loads of one chunk are issued before any use (rows / experts past the
        // end are clamped to a valid address and their sums ignored), so a thread
        // keeps TB + E 16-byte loads in flight instead of serialising on each.
        const int nchunk = p.d / 8;
        const uint4* xrow[TB];
#pragma unroll
        for (int t = 0; t < TB; ++t)
            xrow[t] = reinterpret_cast<const uint4*>(p.x + (int64_t)(tok0 + min(t, ntok - 1)) * p.d);
#pragma unroll 2
        for (int ci = threadIdx.x; ci < nchunk; ci += kRouteThreads) {
            uint4 xr[TB], wr[E_MAX];
#pragma unroll
            for (int t = 0; t < TB; ++t) xr[t] = __ldg(xrow[t] + ci);
#pragma unroll
            for (int e = 0; e < E_MAX; ++e)
                wr[e] = __ldg(reinterpret_cast<const uint4*>(p.wg + (int64_t)min(e, p.E - 1) * p.d) + ci);
            float xv[TB][8];
#pragma unroll
            for (int t = 0; t < TB; ++t) bf16x8_to_f32(xr[t], xv[t]);
#pragma unroll
            for (int e = 0; e < E_MAX; ++e) {
                float w[8];
                bf16x8_to_f32(wr[e], w);
#pragma unroll
                for (int t = 0; t < TB; ++t)
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[t][e] = fmaf(xv[t][i], w[i], acc[t][e]);
            }
        }
#pragma unroll
        for (int t = 0; t < TB; ++t)
#pragma unroll
            for (int e = 0; e < E_MAX; ++e) {
                float v = acc[t][e];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) s_part[warp][t][e] = v;
            }
        __syncthreads();
        if (threadIdx.x < ntok) {
            const int tb = threadIdx.x, t = tok0 + tb;
            float l[E_MAX];
#pragma unroll
            for (int e = 0; e < E_MAX; ++e)
                l[e] = ((s_part[0][tb][e] + s_part[1][tb][e]) + s_part[2][tb][e]) + s_part[3][tb][e];
            if (p.logits) {
#pragma unroll
                for (int e = 0; e < E_MAX; ++e)
                    if (e < p.E) p.logits[(int64_t)t * p.E + e] = l[e];
            }
            // top-k by (logit desc, index asc): strict '>' keeps the lower index on ties (R3)
            int i0 = 0;
            float b0 = l[0];
#pragma unroll
            for (int e = 1; e < E_MAX; ++e)
                if (e < p.E && l[e] > b0) { b0 = l[e]; i0 = e; }
            int i1 = -1;
            float b1 = 0.f;
            if (p.k > 1) {
#pragma unroll
                for (int e = 0; e < E_MAX; ++e)
                    if (e < p.E && e != i0 && (i1 < 0 || l[e] > b1)) { b1 = l[e]; i1 = e; }
            }
            // softmax over all E renormalised over the selected k (R2): the partition
            // function cancels, w_j = exp(l_j - l_max) / sum_sel exp(l - l_max)
            float w0 = 1.f, w1 = 0.f;
            if (p.k > 1) {
                const float e1 = expf(b1 - b0);
                const float den = 1.f + e1;
                w0 = 1.f / den;
                w1 = e1 / den;
            }
            p.topk_idx[(int64_t)t * p.k] = i0;
            p.topk_w[(int64_t)t * p.k] = w0;
            if (p.k > 1) {
                p.topk_idx[(int64_t)t * p.k + 1] = i1;
                p.topk_w[(int64_t)t * p.k + 1] = w1;
            }
            s_idx[tb][0] = i0;
            s_idx[tb][1] = i1;
        }
    } else {
        // routed mode (caller supplied routing): validate and copy into the workspace
        for (int i = threadIdx.x; i < ntok * p.k; i += kRouteThreads) {
            const int tb = i / p.k, j = i % p.k;
            const int64_t o = (int64_t)(tok0 + tb) * p.k + j;
            const int e = p.in_idx[o];
            if (e >= p.E || (e < 0 && !p.allow_neg)) __trap();
            p.topk_idx[o] = e;
            p.topk_w[o] = p.in_w ? p.in_w[o] : 1.f;
            s_idx[tb][j] = e;
        }
    }
    __syncthreads();
    route_block_finish<kRouteThreads>(p, s_idx, ntok, tok0);
    if (p.scan_epoch) route_fold_dispatch<kRouteThreads, TB>(p, s_idx, ntok, tok0, ep0);
}


// K1 on the legacy tensor-core path (mma.sync m16n8k16, bf16 in, fp32 accumulate)
// for E <= 8: the router GEMM has N = E = 8, exactly one n8 fragment. Each warp
// owns 16 tokens x a 1/KS slice of K. A lane loads 16 contiguous bytes (8 bf16)
// of each of its two token rows and of its expert's W_g row at the same k, and
// feeds them as the fragments of two MMAs: the k order inside the MMA is a
// permutation applied identically to A and B, which leaves the dot products
// unchanged. Products of bf16 are exact in fp32; accumulation is fp32 (R5).
// Tokens per block = 16 * (8 / KS): KS = 8 splits K over all 8 warps (decode:
// many short warps), KS = 1 gives each warp its own 16 tokens (prefill).
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int KS>
__global__ void __launch_bounds__(256) moe_router_mma_kernel(const RouteParams p) {
    constexpr int TOK = 16 * (8 / KS);
    __shared__ float s_log[8 / KS][KS][16][8];
    __shared__ int32_t s_idx[TOK][2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * TOK;
    const int ntok = min(TOK, p.T - tok0);
    const int g = warp / KS, kp = warp % KS;
    const int gid = lane >> 2, q = lane & 3;

    MOE_TL(0, 0);
    ptx::pdl_wait();
    MOE_TL(0, 1);
    if (p.early_trigger) ptx::pdl_launch_dependents();
    const unsigned int ep0 = p.scan_epoch ? *reinterpret_cast<volatile unsigned int*>(p.scan_epoch) : 0u;

    const int r0 = min(tok0 + g * 16 + gid, p.T - 1), r1 = min(tok0 + g * 16 + gid + 8, p.T - 1);
    const uint4* xa = reinterpret_cast<const uint4*>(p.x + (int64_t)r0 * p.d);
    const uint4* xb = reinterpret_cast<const uint4*>(p.x + (int64_t)r1 * p.d);
    const bool has_e = gid < p.E;
    const uint4* wr = reinterpret_cast<const uint4*>(p.wg + (int64_t)min(gid, p.E - 1) * p.d);
    const int ksl = p.d / KS;                  // K slice of this warp (multiple of 32: d % 256 == 0 or KS small)
    const int cb = (kp * ksl) / 8, ce = ((kp + 1) * ksl) / 8;  // 16-byte chunks of this warp's K slice
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    // warp-uniform trip count (mma.sync is .aligned); lanes past the slice feed zeros.
    // Software-pipelined by hand: DEPTH iterations of loads are issued before their
    // MMAs, so each lane keeps 3*DEPTH 16-byte loads in flight (HBM-bound at prefill,
    // latency-bound at decode).
    constexpr int DEPTH = 8;
    for (int g0 = cb; g0 < ce; g0 += 4 * DEPTH) {
        uint4 a[DEPTH], b[DEPTH], w[DEPTH];
#pragma unroll
        for (int u = 0; u < DEPTH; ++u) {
            const int ci = g0 + 4 * u + q;
            a[u] = make_uint4(0u, 0u, 0u, 0u);
            b[u] = a[u];
            w[u] = a[u];
            if (ci < ce) {
                a[u] = __ldg(xa + ci);
                b[u] = __ldg(xb + ci);
                if (has_e) w[u] = __ldg(wr + ci);
            }
        }
#pragma unroll
        for (int u = 0; u < DEPTH; ++u) {
            mma_bf16_16816(c, a[u].x, b[u].x, a[u].y, b[u].y, w[u].x, w[u].y);
            mma_bf16_16816(c, a[u].z, b[u].z, a[u].w, b[u].w, w[u].z, w[u].w);
        }
    }
    // c0,c1: token row gid, experts 2q, 2q+1; c2,c3: row gid+8
    s_log[g][kp][gid][2 * q] = c[0];
    s_log[g][kp][gid][2 * q + 1] = c[1];
    s_log[g][kp][gid + 8][2 * q] = c[2];
    s_log[g][kp][gid + 8][2 * q + 1] = c[3];
    __syncthreads();
    if (threadIdx.x < ntok) {
        const int tb = threadIdx.x, t = tok0 + tb;
        const int gg = tb / 16, rr = tb % 16;
        float l[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float v = s_log[gg][0][rr][e];
#pragma unroll
            for (int s2 = 1; s2 < KS; ++s2) v += s_log[gg][s2][rr][e];  // fixed order over K slices
            l[e] = v;
        }
        if (p.logits) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (e < p.E) p.logits[(int64_t)t * p.E + e] = l[e];
        }
        int i0 = 0;
        float b0 = l[0];
#pragma unroll
        for (int e = 1; e < 8; ++e)
            if (e < p.E && l[e] > b0) { b0 = l[e]; i0 = e; }
        int i1 = -1;
        float b1 = 0.f;
        if (p.k > 1) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (e < p.E && e != i0 && (i1 < 0 || l[e] > b1)) { b1 = l[e]; i1 = e; }
        }
        float w0 = 1.f, w1 = 0.f;
        if (p.k > 1) {
            const float e1 = expf(b1 - b0);
            const float den = 1.f + e1;
            w0 = 1.f / den;
            w1 = e1 / den;
        }
        p.topk_idx[(int64_t)t * p.k] = i0;
        p.topk_w[(int64_t)t * p.k] = w0;
        if (p.k > 1) {
            p.topk_idx[(int64_t)t * p.k + 1] = i1;
            p.topk_w[(int64_t)t * p.k + 1] = w1;
        }
        s_idx[tb][0] = i0;
        s_idx[tb][1] = i1;
    }
    __syncthreads();
#if !MOE_TL_LATE_EXIT
    MOE_TL(0, 2);
#endif
    route_block_finish<256>(p, s_idx, ntok, tok0);
    if (p.scan_epoch) route_fold_dispatch<256, TOK>(p, s_idx, ntok, tok0, ep0);
#if MOE_TL_LATE_EXIT
    MOE_TL(0, 2);  // probe: exit stamp after the histogram / scan hand-off
#endif
}

struct PermuteParams {
    const __nv_bfloat16* x;   // [T, d]
    const int32_t* topk_idx;  // [T, k]
    const int32_t* blockoff;  // [nblk, nkeys] (router blocks of TB tokens)
    const int32_t* offsets;   // [nkeys + 1] (normal mode)
    int32_t T, d, k;
    int32_t key_lo, key_div, nkeys;  // as RouteParams
    int32_t cap;              // EP dispatch mode: rows per destination bucket (0 = normal mode)
    int32_t* meta;            // EP dispatch mode: [nkeys * cap] local expert id at the destination
    int32_t TB;               // router block size (tokens)
    int32_t PT;               // tokens per permute block (1, 2, 4 or 8)
    int32_t* pos;             // [T, k] in: in-block rank (router); out: permuted row (-1: not local)
    int32_t* pos_aux;         // optional copy for the caller
    __nv_bfloat16* x_perm;    // [Cap, d]
    // decode speculative weight prefetch (moe.cu spec_l2): trigger the w1/w3 GEMM before
    // waiting for the router, so its L2 weight prefetch overlaps routing. That GEMM then
    // reads counts / offsets only after its own griddepcontrol.wait.
    int32_t early_trigger;
    // FP8 two-term token split (fp8-weight w1/w3 GEMM on kind::f8f6f4): x8 != nullptr ->
    // row ps is stored as bytes hi = e4m3(x * 2^s) in plane 0 and lo = e4m3(x * 2^s - hi)
    // in plane 1 ([2][plane_rows][d] bytes, reusing x_perm's memory), tok_scale[ps] = 2^-s
    uint8_t* x8;
    float* tok_scale;
    int64_t plane_rows;
    int32_t* src_row;         // gather mode (x_perm == nullptr): [Cap] token of each permuted row
    // EP dispatch over peer memory (MOE_FLAG_P2P): rows / meta go straight into slot
    // (my_rank * cap + r) of the destination rank's receive buffer.
    uint8_t* const* peers;
    int64_t peer_rows_off, peer_meta_off;
    int32_t my_rank;
};

// Two E4M3 codes (lower byte = first element) <-> floats
__device__ __forceinline__ uint16_t f32x2_to_e4m3x2(float first, float second) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(second), "f"(first));
    return r;
}
__device__ __forceinline__ float2 e4m3x2_to_f32x2(uint16_t v) {
    uint32_t h;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(v));
    return __half22float2(*reinterpret_cast<__half2*>(&h));
}

// FP8 two-term split of one token row for the kind::f8f6f4 w1/w3 GEMM (R15):
// s = the power of two putting the row max |x| in (224, 448]; hi = RNE_e4m3(x 2^s),
// lo = RNE_e4m3(x 2^s - hi). For bf16 x the residual x 2^s - hi has at most 4
// significant bits, so hi + lo == x 2^s exactly wherever |x 2^s| >= 2^-2 (lo stays above
// the E4M3 subnormal step 2^-9); smaller elements (below ~1e-3 of the row max) keep an
// error <= 2^-10 / 2^s. The GEMM multiplies its fp32 accumulator by tok_scale = 2^-s.
__device__ __forceinline__ void permute_row_fp8x(const PermuteParams& p, int t, int tl, int sw, int wpt, int lane,
                                              const int32_t (*s_pos)[2]) {
    __shared__ uint32_t s_max[8];
    const int nvec = p.d / 8;
    const int stride = 32 * wpt;
    const bool valid = t < p.T;
    const uint4* src = reinterpret_cast<const uint4*>(p.x + (int64_t)(valid ? t : 0) * p.d);
    // pass 1: row max of |x| on the bf16 bit patterns (magnitude order == integer order)
    uint32_t m = 0;
    if (valid)
        for (int v = sw * 32 + lane; v < nvec; v += stride) {
            const uint4 q = __ldg(src + v);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) m = max(m, max(w[i] & 0x7FFFu, (w[i] >> 16) & 0x7FFFu));
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_max[threadIdx.x / 32] = m;
    __syncthreads();
    if (!valid) return;
    uint32_t rm = 0;
    for (int w = 0; w < wpt; ++w) rm = max(rm, s_max[tl * wpt + w]);
    const float rmax = __uint_as_float(rm << 16);
    int sh = 0;
    if (rmax > 0.f) {  // 448 / rmax = 2^e * 1.xx  ->  s = e, rmax * 2^s in (224, 448]
        const int e = ((__float_as_int(448.f / rmax) >> 23) & 0xFF) - 127;
        sh = max(-60, min(60, e));  // keeps 2^(+-2s) of the fp16 h normalisation in fp32 range
    }
    const float scale = __int_as_float((sh + 127) << 23);
    const int32_t d0 = s_pos[tl][0], d1 = p.k > 1 ? s_pos[tl][1] : -1;
    if (sw == 0 && lane == 0) {
        const float inv = __int_as_float((127 - sh) << 23);
        if (d0 >= 0) p.tok_scale[d0] = inv;
        if (d1 >= 0) p.tok_scale[d1] = inv;
    }
    const int64_t plane = p.plane_rows * p.d;
    uint2* hi0 = d0 >= 0 ? reinterpret_cast<uint2*>(p.x8 + (int64_t)d0 * p.d) : nullptr;
    uint2* hi1 = d1 >= 0 ? reinterpret_cast<uint2*>(p.x8 + (int64_t)d1 * p.d) : nullptr;
    for (int v = sw * 32 + lane; v < nvec; v += stride) {
        float f[8];
        bf16x8_to_f32(__ldg(src + v), f);
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float a = f[2 * i] * scale, b = f[2 * i + 1] * scale;
            const uint16_t h = f32x2_to_e4m3x2(a, b);
            const float2 hf = e4m3x2_to_f32x2(h);
            const uint16_t l = f32x2_to_e4m3x2(a - hf.x, b - hf.y);
            hw[i] = h;
            lw[i] = l;
        }
        const uint2 hv = make_uint2(hw[0] | (hw[1] << 16), hw[2] | (hw[3] << 16));
        const uint2 lv = make_uint2(lw[0] | (lw[1] << 16), lw[2] | (lw[3] << 16));
        if (hi0) { hi0[v] = hv; reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(hi0) + plane)[v] = lv; }
        if (hi1) { hi1[v] = hv; reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(hi1) + plane)[v] = lv; }
    }
}

// K2 (a6): position of each assignment = segment start + rank of its router block
// + stable rank inside the block (#earlier tokens of the block routed to the same
// expert), then a 16-byte-vector copy of the token row to each of its k
// positions (8/PT warps per row, all loads of a row in flight before the stores).
__global__ void __launch_bounds__(kPermuteThreads) moe_permute_kernel(const PermuteParams p) {
    __shared__ int32_t s_pos[8][2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * p.PT;
    MOE_TL(1, 0);
    if (p.early_trigger) ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    MOE_TL(1, 1);
#ifndef MOE_PERMUTE_EARLY_TRIGGER
#define MOE_PERMUTE_EARLY_TRIGGER 1  // r01 A/B: 0.4522 -> 0.4510 ms per decode step
#endif
#if MOE_PERMUTE_EARLY_TRIGGER
    // The router (whose counts the GEMMs schedule from) is complete here, so the
    // w1/w3 GEMM may launch now and start streaming weights while rows are copied;
    // it reads the permuted rows only after its own griddepcontrol.wait.
    ptx::pdl_launch_dependents();
#endif
    if (threadIdx.x < p.PT * p.k) {
        const int tl = threadIdx.x / p.k, j = threadIdx.x % p.k;
        const int t = tok0 + tl;
        if (t < p.T) {
            const int ex = p.topk_idx[(int64_t)t * p.k + j];
            const int e = ex >= 0 ? hist_key(ex, p.key_lo, p.key_div, p.nkeys) : -1;
            int32_t ps = -1;
            if (e >= 0) {
                const int b = t / p.TB;
                const int32_t r = p.blockoff[(int64_t)b * p.nkeys + e] + p.pos[(int64_t)t * p.k + j];
                if (p.cap > 0) {  // EP dispatch: bucket of destination rank e
                    ps = e * p.cap + r;
                    int32_t* meta = p.peers ? reinterpret_cast<int32_t*>(p.peers[e] + p.peer_meta_off) +
                                                  (int64_t)p.my_rank * p.cap + r
                                            : p.meta + ps;
                    *meta = ex - e * p.key_div;  // expert index local to the destination
                } else {
                    ps = p.offsets[e] + r;
                }
            }
            p.pos[(int64_t)t * p.k + j] = ps;
            if (p.pos_aux) p.pos_aux[(int64_t)t * p.k + j] = ps;
            if (p.src_row && ps >= 0) p.src_row[ps] = t;
            s_pos[tl][j] = ps;
        }
    }
    if (p.x_perm == nullptr && p.peers == nullptr) {  // gather mode: the w1/w3 GEMM fetches the rows itself
        ptx::pdl_launch_dependents();
        return;
    }
    __syncthreads();
    const int wpt = 8 / p.PT;            // warps per token row
    const int tl = warp / wpt, sw = warp % wpt;
    const int t = tok0 + tl;
    if (p.x8) {
        permute_row_fp8x(p, t, tl, sw, wpt, lane, s_pos);
        ptx::pdl_launch_dependents();
        return;
    }
    if (t < p.T) {
        const int nvec = p.d / 8;
        const uint4* src = reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.d);
        const int32_t d0 = s_pos[tl][0], d1 = p.k > 1 ? s_pos[tl][1] : -1;
        auto row_ptr = [&](int32_t ps) -> uint4* {
            if (ps < 0) return nullptr;
            if (p.peers) {  // P2P dispatch: the destination rank's receive slot
                const int e = ps / p.cap, r = ps - e * p.cap;
                return reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.peers[e] + p.peer_rows_off) +
                                                ((int64_t)p.my_rank * p.cap + r) * p.d);
            }
            return reinterpret_cast<uint4*>(p.x_perm + (int64_t)ps * p.d);
        };
        uint4* dst0 = row_ptr(d0);
        uint4* dst1 = row_ptr(d1);
        const int stride = 32 * wpt;
        for (int v0 = sw * 32 + lane; v0 < nvec; v0 += 4 * stride) {
            uint4 buf[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v0 + u * stride < nvec) buf[u] = __ldg(src + v0 + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v0 + u * stride < nvec) {
                    if (dst0) dst0[v0 + u * stride] = buf[u];
                    if (dst1) dst1[v0 + u * stride] = buf[u];
                }
        }
    }
    MOE_TL(1, 2);
    ptx::pdl_launch_dependents();
}

struct CombineParams {
    const float* y;           // [splits][Cap, d] fp32 expert outputs
    int64_t split_stride;     // elements
    int32_t splits;
    const int32_t* pos;       // [T, k]
    const float* topk_w;      // [T, k]
    const __nv_bfloat16* x;   // residual source (nullable)
    int32_t T, d, k;
    __nv_bfloat16* out;       // [T, d]
    float* out_f32;           // [T, d] optional (fp32 before rounding)
    // TP reduce-scatter over peer memory (MOE_FLAG_P2P): the fp32 row of token t goes
    // to slot [my_rank][t - row0(owner)] of its owner's region (out/out_f32 unused).
    uint8_t* const* peers;
    int64_t peer_off;
    int32_t G, my_rank, shard_max;
    unsigned int* p2p_ticket;  // P2P: this exchange's completion ticket (p2p_signal_last_block)
    int64_t p2p_sig_off;       // P2P: the exchange counter in every region
};

// K5 (a9): out[t] = bf16_rne( sum_j w_j * (sum_s y_s[pos_j]) (+ x[t]) ), fixed order:
// splits ascending, then r = w_0*s_0, r = fma(w_1, s_1, r), then + x.
// grid = T * ceil(d/4096) blocks: each thread owns 4 float4 column groups of one token
// (strided by 1024 columns), so 8 independent 16-byte loads per thread are in flight.
// VEC = column groups per thread: 4 for large batches; 1 for small ones (T <= 256), so a
// 64-token decode spreads over 4x more blocks (the combine runs after the last GEMM tile:
// its latency is on the step's critical path).
template <int kCombineVec>
__global__ void __launch_bounds__(256) moe_combine_kernel(const CombineParams p) {
    // 1-D grid (T may exceed the 65535 limit of gridDim.y): block b -> token b / nxb
    const int nxb = (p.d + 1024 * kCombineVec - 1) / (1024 * kCombineVec);
    const int t = blockIdx.x / nxb;
    const int c0 = (blockIdx.x % nxb) * 1024 * kCombineVec + threadIdx.x * 4;
    MOE_TL(4, 0);
    ptx::pdl_wait();
    MOE_TL(4, 1);
    int32_t pr[2];
    float w[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        pr[j] = j < p.k ? p.pos[(int64_t)t * p.k + j] : -1;
        w[j] = j < p.k ? p.topk_w[(int64_t)t * p.k + j] : 0.f;
    }
    float4 s[2][kCombineVec];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int v = 0; v < kCombineVec; ++v) {
            const int c = c0 + v * 1024;
            s[j][v] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (pr[j] >= 0 && c < p.d) s[j][v] = __ldcs(reinterpret_cast<const float4*>(p.y + (int64_t)pr[j] * p.d + c));
        }
    for (int sp = 1; sp < p.splits; ++sp)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < kCombineVec; ++v) {
                const int c = c0 + v * 1024;
                if (pr[j] >= 0 && c < p.d) {
                    const float4 u = __ldcs(reinterpret_cast<const float4*>(p.y + sp * p.split_stride +
                                                                            (int64_t)pr[j] * p.d + c));
                    s[j][v].x += u.x; s[j][v].y += u.y; s[j][v].z += u.z; s[j][v].w += u.w;
                }
            }
#pragma unroll
    for (int v = 0; v < kCombineVec; ++v) {
        const int c = c0 + v * 1024;
        if (c >= p.d) break;
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (pr[0] >= 0) r = make_float4(w[0] * s[0][v].x, w[0] * s[0][v].y, w[0] * s[0][v].z, w[0] * s[0][v].w);
        if (pr[1] >= 0) {
            r.x = fmaf(w[1], s[1][v].x, r.x); r.y = fmaf(w[1], s[1][v].y, r.y);
            r.z = fmaf(w[1], s[1][v].z, r.z); r.w = fmaf(w[1], s[1][v].w, r.w);
        }
        if (p.x) {
            const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(p.x + (int64_t)t * p.d + c);
            const float2 a = __bfloat1622float2(xs[0]), b = __bfloat1622float2(xs[1]);
            r.x += a.x; r.y += a.y; r.z += b.x; r.w += b.y;
        }
        if (p.peers) {
            const int o = tp_owner(t, p.T, p.G);
            float* dst = reinterpret_cast<float*>(p.peers[o] + p.peer_off) +
                         ((int64_t)p.my_rank * p.shard_max + (t - tp_row0(o, p.T, p.G))) * p.d + c;
            *reinterpret_cast<float4*>(dst) = r;
        }
        if (p.out_f32) __stcs(reinterpret_cast<float4*>(p.out_f32 + (int64_t)t * p.d + c), r);
        if (p.out) {
            __nv_bfloat162 o0 = __floats2bfloat162_rn(r.x, r.y), o1 = __floats2bfloat162_rn(r.z, r.w);
            uint2 ov;
            ov.x = *reinterpret_cast<uint32_t*>(&o0);
            ov.y = *reinterpret_cast<uint32_t*>(&o1);
            *reinterpret_cast<uint2*>(p.out + (int64_t)t * p.d + c) = ov;
        }
    }
    if (p.peers) p2p_signal_last_block(p.p2p_ticket, p.peers, p.G, p.p2p_sig_off);  // TP reduce-scatter done
    MOE_TL(4, 2);
    ptx::pdl_launch_dependents();
}

// EP return path: ysend[slot] = sum_s y_s[pos[slot]] for every occupied receive
// slot (fp32 rows; splits summed in ascending order, as in the combine).
// P2P (peers != nullptr): the row goes straight to slot (my_rank * cap + r) of the
// return buffer of source rank slot / cap, r = slot % cap.
__global__ void __launch_bounds__(256) moe_ep_gather_kernel(const float* y, int64_t split_stride, int splits,
                                                            const int32_t* pos, int nslots, int d, float* ysend,
                                                            uint8_t* const* peers, int64_t peer_off, int cap,
                                                            int my_rank, int G, unsigned int* ticket, int64_t sig_off) {
    const int nxb = (d + 1023) / 1024;  // 1-D grid: block b -> slot b / nxb
    const int slot = blockIdx.x / nxb;
    const int c = (blockIdx.x % nxb) * 1024 + threadIdx.x * 4;
    ptx::pdl_wait();
    if (slot < nslots && c < d) {
        const int32_t pr = pos[slot];
        if (pr >= 0) {
            const float* yr = y + (int64_t)pr * d + c;
            float4 s = __ldcs(reinterpret_cast<const float4*>(yr));
#pragma unroll 8
            for (int sp = 1; sp < splits; ++sp) {
                const float4 u = __ldcs(reinterpret_cast<const float4*>(yr + sp * split_stride));
                s.x += u.x; s.y += u.y; s.z += u.z; s.w += u.w;
            }
            float* dst = ysend + (int64_t)slot * d + c;
            if (peers) {
                const int src = slot / cap, r = slot - src * cap;
                dst = reinterpret_cast<float*>(peers[src] + peer_off) + ((int64_t)my_rank * cap + r) * d + c;
            }
            *reinterpret_cast<float4*>(dst) = s;
        }
    }
    if (peers) p2p_signal_last_block(ticket, peers, G, sig_off);  // EP return exchange done
    ptx::pdl_launch_dependents();
}

// TP epilogue after the fp32 reduce-scatter: this rank's shard of the summed
// output (+ residual) -> one bf16 RNE rounding, written in place into its slice of
// `out` (all-gathered afterwards); optional fp32 copy into its slice of out_f32.
__global__ void __launch_bounds__(256) moe_tp_finish_kernel(const float* shard, int64_t n, int64_t base,
                                                            const __nv_bfloat16* x, __nv_bfloat16* out,
                                                            float* out_f32) {
    ptx::pdl_wait();
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < n;
         i += (int64_t)gridDim.x * blockDim.x * 4) {
        float4 r = *reinterpret_cast<const float4*>(shard + i);
        if (x) {
            const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(x + base + i);
            const float2 a = __bfloat1622float2(xs[0]), b = __bfloat1622float2(xs[1]);
            r.x += a.x; r.y += a.y; r.z += b.x; r.w += b.y;
        }
        if (out_f32) *reinterpret_cast<float4*>(out_f32 + base + i) = r;
        __nv_bfloat162 o0 = __floats2bfloat162_rn(r.x, r.y), o1 = __floats2bfloat162_rn(r.z, r.w);
        uint2 ov;
        ov.x = *reinterpret_cast<uint32_t*>(&o0);
        ov.y = *reinterpret_cast<uint32_t*>(&o1);
        *reinterpret_cast<uint2*>(out + base + i) = ov;
    }
    ptx::pdl_launch_dependents();
}

// Weight packing (init-time, not on the hot path).
// w13p[e][256*b + i][c] = w1[eg][f_off + 128*b + i][c]        (i < 128)
//                       = w3[eg][f_off + 128*b + i - 128][c]  (i >= 128)
// w2p[e][r][i] = w2[eg][r][f_off + i], eg = e_off + e.
// Packing (moe_pack_weights). Row order of W13: blocks of 256 rows = 128 w1 rows then
// the 128 w3 rows of the same ffn columns (this rank's f slice). `tiled` (bf16): every
// 256-row block of W13 / 128-row block of W2 is stored as K/64 consecutive [rows][64]
// chunks (32 / 16 KB): one K block of one tile is one contiguous HBM range -- a
// streaming read of such chunks runs at 7.26 TB/s vs 6.19 TB/s for 128-byte pieces of
// 128 rows 28 KB apart (the row-major W2), scripts/exp/read_bw.cu. W2 rows are padded
// with zeros to a multiple of 256. tiled = 0 (FP8 packing, 1-byte weights moved as
// 2-byte units): plain row-major [E_l][rows][K].
__global__ void moe_pack_w13_kernel(const __nv_bfloat16* w1, const __nv_bfloat16* w3, __nv_bfloat16* w13p,
                                    int E_local, int e_off, int d, int f, int f_local, int f_off, int tiled) {
    ptx::pdl_wait();  // launched with PDL: the caller's producer of w1/w3 (a cast, a copy) has finished
    const int64_t nvec_row = d / 8;
    const int64_t total = (int64_t)E_local * 2 * f_local * nvec_row;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = v / nvec_row, cv = v % nvec_row;
        const int64_t e = row / (2 * f_local), pr = row % (2 * f_local);
        const int64_t blk = pr / 256, i = pr % 256;
        const __nv_bfloat16* src = (i < 128 ? w1 : w3) +
                                   ((e_off + e) * (int64_t)f + f_off + blk * 128 + (i % 128)) * d;
        int64_t dst = v;
        if (tiled) {
            const int64_t nkb = d / 64, tile = e * (2 * f_local / 256) + blk;
            dst = ((tile * nkb + cv / 8) * 256 + i) * 8 + cv % 8;
        }
        reinterpret_cast<uint4*>(w13p)[dst] = reinterpret_cast<const uint4*>(src)[cv];
    }
}
__global__ void moe_pack_w2_kernel(const __nv_bfloat16* w2, __nv_bfloat16* w2p, int E_local, int e_off, int d,
                                   int f, int f_local, int f_off, int tiled, int pad_rows) {
    ptx::pdl_wait();
    const int64_t nvec_row = f_local / 8;
    const int rows = pad_rows ? (d + 255) / 256 * 256 : d;  // bf16: zero rows up to a multiple of 256
    const int64_t total = (int64_t)E_local * rows * nvec_row;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = v / nvec_row, cv = v % nvec_row;  // row = e*rows + r
        const int64_t e = row / rows, r = row % rows;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (r < d) val = reinterpret_cast<const uint4*>(w2 + ((e_off + e) * (int64_t)d + r) * f + f_off)[cv];
        int64_t dst = v;
        if (tiled) {
            const int64_t nkb = f_local / 64, tile = e * (rows / 128) + r / 128;
            dst = ((tile * nkb + cv / 8) * 128 + r % 128) * 8 + cv % 8;
        }
        reinterpret_cast<uint4*>(w2p)[dst] = val;
    }
}

// FP8 weight scales (one fp32 power of two per output row) in the packed row order:
// s13[e][256*b + i] = s1[eg][f_off + 128*b + i] (i < 128), s3[...][... + i - 128] (i >= 128)
__global__ void moe_pack_scales_kernel(const float* s1, const float* s3, const float* s2, float* s13p, float* s2p,
                                       int E_local, int e_off, int d, int f, int f_local, int f_off) {
    ptx::pdl_wait();
    const int64_t n13 = (int64_t)E_local * 2 * f_local, n2 = (int64_t)E_local * d;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n13 + n2; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n13) {
            const int64_t e = i / (2 * f_local), pr = i % (2 * f_local), b = pr / 256, j = pr % 256;
            const float* src = j < 128 ? s1 : s3;
            s13p[i] = src[(e_off + e) * (int64_t)f + f_off + b * 128 + (j % 128)];
        } else {
            const int64_t k = i - n13, e = k / d, r = k % d;
            s2p[k] = s2[(e_off + e) * (int64_t)d + r];
        }
    }
}

}  // namespace moe
