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
#include <stdint.h>
#include "sm100.cuh"

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
    int32_t* blockcount;      // [nblk, nkeys]
    int32_t* blockoff;        // [nblk, nkeys]
    int32_t* counts;          // [nkeys]
    int32_t* offsets;         // [nkeys + 1]
    unsigned int* done;       // block-completion counter (zero between launches)
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

// K1: router (a2, a3) + per-block histogram (a4) + last-block exclusive scan (a5).
// A block owns TB consecutive tokens; its 128 threads split the hidden dimension
// in 8-element (16-byte) chunks, each thread accumulating TB x E partial dot
// products in fp32 (bf16*bf16 products are exact in fp32). W_g chunks are loaded
// once per thread and reused for the TB tokens. Partial sums are reduced with
// warp shuffles, then across the 4 warps in a fixed order (deterministic).
template <int E_MAX, int TB>
__global__ void __launch_bounds__(kRouteThreads) moe_router_kernel(const RouteParams p) {
    __shared__ float s_part[4][TB][E_MAX];
    __shared__ int32_t s_idx[TB][2];
    __shared__ int s_last;
    __shared__ int32_t s_tot[32];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * TB;
    const int ntok = min(TB, p.T - tok0);
    const int NK = p.nkeys;

    ptx::pdl_wait();

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
#pragma unroll
            for (int t = 0; t < TB; ++t) {
                float xv[8];
                bf16x8_to_f32(xr[t], xv);
#pragma unroll
                for (int e = 0; e < E_MAX; ++e) {
                    float w[8];
                    bf16x8_to_f32(wr[e], w);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[t][e] = fmaf(xv[i], w[i], acc[t][e]);
                }
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

    // ---- a4: per-block histogram over the keys (local experts / destination ranks)
    if (threadIdx.x < NK) {
        int32_t cnt = 0;
        for (int tb = 0; tb < ntok; ++tb) {
            const int e0 = s_idx[tb][0], e1 = p.k > 1 ? s_idx[tb][1] : -1;
            if (p.k > 1 && e0 == e1 && e0 >= 0) __trap();  // duplicate expert in a routing
            cnt += (e0 >= 0 && hist_key(e0, p.key_lo, p.key_div, NK) == (int)threadIdx.x) ? 1 : 0;
            cnt += (e1 >= 0 && hist_key(e1, p.key_lo, p.key_div, NK) == (int)threadIdx.x) ? 1 : 0;
        }
        p.blockcount[(int64_t)blockIdx.x * NK + threadIdx.x] = cnt;
    }

    // ---- a5: the last block to finish runs the exclusive scan (one block, fixed
    // order: deterministic). Classic threadfence-reduction handshake.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int nblk = gridDim.x;
    for (int e = warp; e < NK; e += kRouteThreads / 32) {
        int32_t running = 0;
        for (int base = 0; base < nblk; base += 32) {
            const int b = base + lane;
            const int32_t v = b < nblk ? __ldcg(&p.blockcount[(int64_t)b * NK + e]) : 0;
            int32_t inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            if (b < nblk) p.blockoff[(int64_t)b * NK + e] = running + inc - v;
            running += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_tot[e] = running;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t off = 0;
        p.offsets[0] = 0;
        for (int e = 0; e < NK; ++e) {
            p.counts[e] = s_tot[e];
            off += (s_tot[e] + p.seg_align - 1) / p.seg_align * p.seg_align;
            p.offsets[e + 1] = off;
        }
        *p.done = 0u;  // ready for the next forward (kernel boundary orders it)
    }
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
    int32_t* pos;             // [T, k] permuted row per assignment (-1: not local)
    int32_t* pos_aux;         // optional copy for the caller
    __nv_bfloat16* x_perm;    // [Cap, d]
};

// K2 (a6): position of each assignment = segment start + rank of its router block
// + stable rank inside the block (#earlier tokens of the block routed to the same
// expert), then a 16-byte-vector copy of the token row to each of its k
// positions (8/PT warps per row, all loads of a row in flight before the stores).
__global__ void __launch_bounds__(kPermuteThreads) moe_permute_kernel(const PermuteParams p) {
    __shared__ int32_t s_pos[8][2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * p.PT;
    ptx::pdl_wait();
    if (threadIdx.x < p.PT * p.k) {
        const int tl = threadIdx.x / p.k, j = threadIdx.x % p.k;
        const int t = tok0 + tl;
        if (t < p.T) {
            const int ex = p.topk_idx[(int64_t)t * p.k + j];
            const int e = ex >= 0 ? hist_key(ex, p.key_lo, p.key_div, p.nkeys) : -1;
            int32_t ps = -1;
            if (e >= 0) {
                const int b = t / p.TB;
                int32_t rank = 0;
                // stable order = (token, slot): count earlier assignments with the same key.
                // (A token may put both its rows in one EP destination bucket.)
                for (int t2 = b * p.TB; t2 <= t; ++t2)
                    for (int j2 = 0; j2 < (t2 == t ? j : p.k); ++j2) {
                        const int e2 = p.topk_idx[(int64_t)t2 * p.k + j2];
                        rank += (e2 >= 0 && hist_key(e2, p.key_lo, p.key_div, p.nkeys) == e);
                    }
                const int32_t r = p.blockoff[(int64_t)b * p.nkeys + e] + rank;
                if (p.cap > 0) {  // EP dispatch: bucket of destination rank e
                    ps = e * p.cap + r;
                    p.meta[ps] = ex - e * p.key_div;  // expert index local to the destination
                } else {
                    ps = p.offsets[e] + r;
                }
            }
            p.pos[(int64_t)t * p.k + j] = ps;
            if (p.pos_aux) p.pos_aux[(int64_t)t * p.k + j] = ps;
            s_pos[tl][j] = ps;
        }
    }
    __syncthreads();
    const int wpt = 8 / p.PT;            // warps per token row
    const int tl = warp / wpt, sw = warp % wpt;
    const int t = tok0 + tl;
    if (t < p.T) {
        const int nvec = p.d / 8;
        const uint4* src = reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.d);
        const int32_t d0 = s_pos[tl][0], d1 = p.k > 1 ? s_pos[tl][1] : -1;
        uint4* dst0 = d0 >= 0 ? reinterpret_cast<uint4*>(p.x_perm + (int64_t)d0 * p.d) : nullptr;
        uint4* dst1 = d1 >= 0 ? reinterpret_cast<uint4*>(p.x_perm + (int64_t)d1 * p.d) : nullptr;
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
};

// K5 (a9): out[t] = bf16_rne( sum_j w_j * (sum_s y_s[pos_j]) (+ x[t]) ), fixed order:
// splits ascending, then r = w_0*s_0, r = fma(w_1, s_1, r), then + x.
// grid = (ceil(d/1024), T): each thread owns 4 consecutive columns of one token.
__global__ void __launch_bounds__(256) moe_combine_kernel(const CombineParams p) {
    const int t = blockIdx.y;
    const int c = blockIdx.x * 1024 + threadIdx.x * 4;
    ptx::pdl_wait();
    if (c < p.d) {
        int32_t pr[2];
        float w[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pr[j] = j < p.k ? p.pos[(int64_t)t * p.k + j] : -1;
            w[j] = j < p.k ? p.topk_w[(int64_t)t * p.k + j] : 0.f;
        }
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (pr[j] < 0) continue;
            const float* yr = p.y + (int64_t)pr[j] * p.d + c;
            float4 s = __ldcs(reinterpret_cast<const float4*>(yr));
#pragma unroll 8
            for (int sp = 1; sp < p.splits; ++sp) {
                const float4 u = __ldcs(reinterpret_cast<const float4*>(yr + sp * p.split_stride));
                s.x += u.x; s.y += u.y; s.z += u.z; s.w += u.w;
            }
            if (j == 0) {
                r = make_float4(w[0] * s.x, w[0] * s.y, w[0] * s.z, w[0] * s.w);
            } else {
                r.x = fmaf(w[j], s.x, r.x); r.y = fmaf(w[j], s.y, r.y);
                r.z = fmaf(w[j], s.z, r.z); r.w = fmaf(w[j], s.w, r.w);
            }
        }
        if (p.x) {
            const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(p.x + (int64_t)t * p.d + c);
            const float2 a = __bfloat1622float2(xs[0]), b = __bfloat1622float2(xs[1]);
            r.x += a.x; r.y += a.y; r.z += b.x; r.w += b.y;
        }
        if (p.out_f32) __stcs(reinterpret_cast<float4*>(p.out_f32 + (int64_t)t * p.d + c), r);
        if (p.out == nullptr) return;
        __nv_bfloat162 o0 = __floats2bfloat162_rn(r.x, r.y), o1 = __floats2bfloat162_rn(r.z, r.w);
        uint2 ov;
        ov.x = *reinterpret_cast<uint32_t*>(&o0);
        ov.y = *reinterpret_cast<uint32_t*>(&o1);
        *reinterpret_cast<uint2*>(p.out + (int64_t)t * p.d + c) = ov;
    }
    ptx::pdl_launch_dependents();
}

// EP return path: ysend[slot] = sum_s y_s[pos[slot]] for every occupied receive
// slot (fp32 rows; splits summed in ascending order, as in the combine).
__global__ void __launch_bounds__(256) moe_ep_gather_kernel(const float* y, int64_t split_stride, int splits,
                                                            const int32_t* pos, int nslots, int d, float* ysend) {
    const int slot = blockIdx.y;
    const int c = blockIdx.x * 1024 + threadIdx.x * 4;
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
            *reinterpret_cast<float4*>(ysend + (int64_t)slot * d + c) = s;
        }
    }
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
__global__ void moe_pack_w13_kernel(const __nv_bfloat16* w1, const __nv_bfloat16* w3, __nv_bfloat16* w13p,
                                    int E_local, int e_off, int d, int f, int f_local, int f_off) {
    const int64_t nvec_row = d / 8;
    const int64_t total = (int64_t)E_local * 2 * f_local * nvec_row;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = v / nvec_row, cv = v % nvec_row;
        const int64_t e = row / (2 * f_local), pr = row % (2 * f_local);
        const int64_t blk = pr / 256, i = pr % 256;
        const __nv_bfloat16* src = (i < 128 ? w1 : w3) +
                                   ((e_off + e) * (int64_t)f + f_off + blk * 128 + (i % 128)) * d;
        reinterpret_cast<uint4*>(w13p)[v] = reinterpret_cast<const uint4*>(src)[cv];
    }
}
__global__ void moe_pack_w2_kernel(const __nv_bfloat16* w2, __nv_bfloat16* w2p, int E_local, int e_off, int d,
                                   int f, int f_local, int f_off) {
    const int64_t nvec_row = f_local / 8;
    const int64_t total = (int64_t)E_local * d * nvec_row;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = v / nvec_row, cv = v % nvec_row;  // row = e*d + r
        const int64_t e = row / d, r = row % d;
        const __nv_bfloat16* src = w2 + ((e_off + e) * (int64_t)d + r) * f + f_off;
        reinterpret_cast<uint4*>(w2p)[v] = reinterpret_cast<const uint4*>(src)[cv];
    }
}

}  // namespace moe
