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

constexpr int kRouteTokPerBlock = 64;   // tokens per router / permute block
constexpr int kRouteThreads = 256;      // 8 warps
constexpr int kSegAlign = 128;          // expert segments padded to the GEMM M tile

struct RouteParams {
    const __nv_bfloat16* x;   // [T, d]
    const __nv_bfloat16* wg;  // [E, d]
    const int32_t* in_idx;    // routed mode: caller's [T, k] (else nullptr)
    const float* in_w;        // routed mode: caller's gates [T, k]
    int32_t T, d, E, k;
    int32_t e_lo, e_hi;       // experts owned by this rank: [e_lo, e_hi) (all for NONE/TP)
    float* logits;            // [T, E] optional debug output
    int32_t* topk_idx;        // [T, k] workspace
    float* topk_w;            // [T, k] workspace
    int32_t* blockcount;      // [nblk, E_local]
    int32_t* blockoff;        // [nblk, E_local]
    int32_t* counts;          // [E_local]
    int32_t* offsets;         // [E_local + 1]
    unsigned int* done;       // block-completion counter (zero between launches)
};

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// Per-warp, stable (by token index) rank of each of the warp's 32 tokens inside
// each local expert: rank = #{lanes l' < l whose token is routed to that expert}.
// Writes wcnt[e] = #tokens of this warp routed to local expert e.
template <int KMAX>
__device__ __forceinline__ void warp_expert_ranks(const int32_t (&le)[KMAX], int k, int E_local, bool valid,
                                                  int32_t (&rank)[KMAX], int32_t* wcnt, int lane) {
    const uint32_t lt = (1u << lane) - 1u;
    for (int e = 0; e < E_local; ++e) {
        bool mine = false;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) mine |= (j < k) && (le[j] == e);
        const uint32_t m = __ballot_sync(0xffffffffu, valid && mine);
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
            if (j < k && le[j] == e) rank[j] = __popc(m & lt);
        if (lane == 0) wcnt[e] = __popc(m);
    }
}

// K1: router + histogram + (last block) scan.  E_MAX bounds E (register arrays).
template <int E_MAX>
__global__ void __launch_bounds__(kRouteThreads) moe_router_kernel(const RouteParams p) {
    __shared__ int32_t s_idx[kRouteTokPerBlock][2];
    __shared__ int32_t s_wcnt[2][32];
    __shared__ int s_last;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * kRouteTokPerBlock;
    const int E_local = p.e_hi - p.e_lo;

    ptx::pdl_wait();

    if (p.in_idx == nullptr) {
        // ---- a2/a3: logits by warp-cooperative dot products, 2 tokens per pass.
        // Lane owns 8 consecutive hidden elements per 256-element slab (16-byte loads).
        for (int pass = 0; pass < kRouteTokPerBlock / 16; ++pass) {
            const int tl0 = warp * (kRouteTokPerBlock / 8) + 2 * pass;
            const int t0 = tok0 + tl0, t1 = t0 + 1;
            float acc0[E_MAX], acc1[E_MAX];
#pragma unroll
            for (int e = 0; e < E_MAX; ++e) { acc0[e] = 0.f; acc1[e] = 0.f; }
            if (t0 < p.T) {
                const bool has1 = t1 < p.T;
                for (int c = lane * 8; c < p.d; c += 256) {
                    float x0[8], x1[8];
                    bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t0 * p.d + c)), x0);
                    if (has1) bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)t1 * p.d + c)), x1);
                    else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) x1[i] = 0.f;
                    }
#pragma unroll
                    for (int e = 0; e < E_MAX; ++e) {
                        if (e < p.E) {
                            float w[8];
                            bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(p.wg + (int64_t)e * p.d + c)), w);
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                acc0[e] = fmaf(x0[i], w[i], acc0[e]);  // bf16*bf16 is exact in fp32
                                acc1[e] = fmaf(x1[i], w[i], acc1[e]);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < E_MAX; ++e) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    acc0[e] += __shfl_xor_sync(0xffffffffu, acc0[e], o);
                    acc1[e] += __shfl_xor_sync(0xffffffffu, acc1[e], o);
                }
            }
            // lane 0 finalises token t0, lane 1 token t1 (each from its own, fixed-order sums)
            if (lane < 2) {
                const int t = lane == 0 ? t0 : t1;
                if (t < p.T) {
                    float l[E_MAX];
#pragma unroll
                    for (int e = 0; e < E_MAX; ++e) l[e] = lane == 0 ? acc0[e] : acc1[e];
                    if (p.logits) {
#pragma unroll
                        for (int e = 0; e < E_MAX; ++e)
                            if (e < p.E) p.logits[(int64_t)t * p.E + e] = l[e];
                    }
                    // top-k by (logit desc, index asc): strict '>' keeps the lower index on ties
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
                    // softmax over all E renormalised over the selected k: the partition
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
                    s_idx[t - tok0][0] = i0;
                    s_idx[t - tok0][1] = i1;
                }
            }
        }
    } else {
        // routed mode (caller supplied routing): validate and copy into the workspace
        for (int i = threadIdx.x; i < kRouteTokPerBlock * p.k; i += blockDim.x) {
            const int tl = i / p.k, j = i % p.k;
            const int t = tok0 + tl;
            if (t < p.T) {
                const int e = p.in_idx[(int64_t)t * p.k + j];
                if (e < 0 || e >= p.E) __trap();
                p.topk_idx[(int64_t)t * p.k + j] = e;
                p.topk_w[(int64_t)t * p.k + j] = p.in_w[(int64_t)t * p.k + j];
                s_idx[tl][j] = e;
            }
        }
    }
    __syncthreads();

    // ---- a4: per-block histogram over local experts (warps 0,1 x 32 tokens)
    if (warp < 2) {
        const int tl = warp * 32 + lane;
        const bool valid = tok0 + tl < p.T;
        int32_t le[2], rank[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) le[j] = valid && j < p.k ? s_idx[tl][j] - p.e_lo : -1;
        if (valid && p.k > 1 && le[0] == le[1]) __trap();  // duplicate expert in a routing
        warp_expert_ranks<2>(le, p.k, E_local, valid, rank, s_wcnt[warp], lane);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E_local; e += blockDim.x)
        p.blockcount[(int64_t)blockIdx.x * E_local + e] = s_wcnt[0][e] + s_wcnt[1][e];

    // ---- a5: the last block to finish runs the exclusive scan (deterministic: one
    // block, fixed order). Classic threadfence-reduction handshake.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ int32_t s_tot[32];
    const int nblk = gridDim.x;
    for (int e = warp; e < E_local; e += kRouteThreads / 32) {
        int32_t running = 0;
        for (int base = 0; base < nblk; base += 32) {
            const int b = base + lane;
            const int32_t v = b < nblk ? __ldcg(&p.blockcount[(int64_t)b * E_local + e]) : 0;
            int32_t inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            if (b < nblk) p.blockoff[(int64_t)b * E_local + e] = running + inc - v;
            running += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_tot[e] = running;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t off = 0;
        p.offsets[0] = 0;
        for (int e = 0; e < E_local; ++e) {
            p.counts[e] = s_tot[e];
            off += (s_tot[e] + kSegAlign - 1) / kSegAlign * kSegAlign;
            p.offsets[e + 1] = off;
        }
        *p.done = 0u;  // ready for the next forward (kernel boundary orders it)
    }
}

struct PermuteParams {
    const __nv_bfloat16* x;   // [T, d]
    const int32_t* topk_idx;  // [T, k]
    const float* topk_w;      // [T, k]
    const int32_t* blockoff;  // [nblk, E_local]
    const int32_t* offsets;   // [E_local + 1]
    int32_t T, d, k, e_lo, E_local;
    int32_t* pos;             // [T, k] permuted row per assignment (-1: not local)
    int32_t* pos_aux;         // optional copy for the caller
    __nv_bfloat16* x_perm;    // [Cap, d]
};

// K2: stable rank -> position, then copy each token row to its k segments with
// 16-byte vectors (one warp per token row; all loads of a row in flight first).
__global__ void __launch_bounds__(kRouteThreads) moe_permute_kernel(const PermuteParams p) {
    __shared__ int32_t s_wcnt[2][32];
    __shared__ int32_t s_pos[kRouteTokPerBlock][2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tok0 = blockIdx.x * kRouteTokPerBlock;
    ptx::pdl_wait();
    int32_t le[2] = {-1, -1}, rank[2] = {0, 0};
    const int tl = warp * 32 + lane;
    const bool valid = warp < 2 && tok0 + tl < p.T;
    if (warp < 2) {
        if (valid) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
                if (j < p.k) {
                    const int e = p.topk_idx[(int64_t)(tok0 + tl) * p.k + j] - p.e_lo;
                    le[j] = (e >= 0 && e < p.E_local) ? e : -1;
                }
        }
        warp_expert_ranks<2>(le, p.k, p.E_local, valid, rank, s_wcnt[warp], lane);
    }
    __syncthreads();
    if (valid) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (j >= p.k) break;
            int32_t ps = -1;
            if (le[j] >= 0) {
                const int e = le[j];
                ps = p.offsets[e] + p.blockoff[(int64_t)blockIdx.x * p.E_local + e] +
                     (warp == 1 ? s_wcnt[0][e] : 0) + rank[j];
            }
            p.pos[(int64_t)(tok0 + tl) * p.k + j] = ps;
            if (p.pos_aux) p.pos_aux[(int64_t)(tok0 + tl) * p.k + j] = ps;
            s_pos[tl][j] = ps;
        }
    }
    __syncthreads();
    // row copies: warp w handles tokens [w*8, w*8+8) of the block
    const int nvec = p.d / 8;  // uint4 per row
    for (int i = 0; i < kRouteTokPerBlock / 8; ++i) {
        const int tl2 = warp * (kRouteTokPerBlock / 8) + i;
        const int t = tok0 + tl2;
        if (t >= p.T) break;
        const uint4* src = reinterpret_cast<const uint4*>(p.x + (int64_t)t * p.d);
        int32_t dst_row[2] = {s_pos[tl2][0], p.k > 1 ? s_pos[tl2][1] : -1};
        for (int v0 = 0; v0 < nvec; v0 += 32 * 8) {
            uint4 buf[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < nvec) buf[u] = __ldg(src + v);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (dst_row[j] < 0) continue;
                uint4* dst = reinterpret_cast<uint4*>(p.x_perm + (int64_t)dst_row[j] * p.d);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int v = v0 + u * 32 + lane;
                    if (v < nvec) dst[v] = buf[u];
                }
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

// K5: out[t] = bf16_rne( sum_j w_j * (sum_s y_s[pos_j]) (+ x[t]) ), fixed order:
// splits ascending, then r = w_0*s_0, r = fma(w_1, s_1, r), then + x.
__global__ void __launch_bounds__(256) moe_combine_kernel(const CombineParams p) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int t = blockIdx.x * 8 + warp;
    ptx::pdl_wait();
    if (t < p.T) {
        int32_t pr[2];
        float w[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pr[j] = j < p.k ? p.pos[(int64_t)t * p.k + j] : -1;
            w[j] = j < p.k ? p.topk_w[(int64_t)t * p.k + j] : 0.f;
        }
        for (int c = lane * 4; c < p.d; c += 128) {
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (pr[j] < 0) continue;
                const float* yr = p.y + (int64_t)pr[j] * p.d + c;
                float4 s = __ldcs(reinterpret_cast<const float4*>(yr));
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
                float xv[4];
                const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(p.x + (int64_t)t * p.d + c);
                float2 a = __bfloat1622float2(xs[0]), b = __bfloat1622float2(xs[1]);
                xv[0] = a.x; xv[1] = a.y; xv[2] = b.x; xv[3] = b.y;
                r.x += xv[0]; r.y += xv[1]; r.z += xv[2]; r.w += xv[3];
            }
            if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + (int64_t)t * p.d + c) = r;
            __nv_bfloat162 o0 = __floats2bfloat162_rn(r.x, r.y), o1 = __floats2bfloat162_rn(r.z, r.w);
            uint2 ov;
            ov.x = *reinterpret_cast<uint32_t*>(&o0);
            ov.y = *reinterpret_cast<uint32_t*>(&o1);
            *reinterpret_cast<uint2*>(p.out + (int64_t)t * p.d + c) = ov;
        }
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
