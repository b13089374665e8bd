// Peer-memory transport (MOE_FLAG_P2P, SURVEY 8(f) NEXT #3 "communication fusion").
//
// Every rank of the group owns one symmetric device region (same layout and size on
// all ranks) and holds a device table `peers[G]` of the base addresses of all G
// regions, mapped into its address space (CUDA IPC across processes; the plain
// pointers when the ranks share a process). The exchange steps of the EP and TP
// paths then become stores into the peers' regions issued by the kernels that
// produce the data -- no separate collective, no staging copy:
//
//   EP dispatch : the permute kernel writes each routed token row straight into its
//                 slot of the destination rank's receive buffer (P2P 16-byte stores)
//   EP return   : the gather kernel writes each expert-output row straight into the
//                 source rank's return buffer
//   TP reduce   : the combine kernel writes each token's fp32 partial into the
//                 owner rank's slot for this rank (reduce-scatter by stores); the
//                 owner sums the G slots in rank order, rounds once to bf16 (R7),
//                 and the other ranks pull the finished rows (all-gather by loads)
//
// Completion (round 2: inside the producing kernel): every block of the producing kernel
// fences its peer stores (system scope) and takes a ticket; the LAST block adds 1 to
// counter `sig` of every rank's region (release, system scope) -- p2p_signal_last_block.
// Each rank's stream then waits (cuStreamWaitValue64 >= G, no SM spinning) and resets its
// counter for the next forward (moe.cu p2p_wait). No separate signal kernel.
#pragma once
#include "sm100.cuh"

namespace moe {

__device__ __forceinline__ void red_release_sys_add_u64(uint64_t* p, uint64_t v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exchange completion from inside a producing kernel, called by EVERY thread of EVERY
// block at its end (no early returns before it). Each thread's stores (local or peer) are
// fenced at system scope before its block takes a ticket (classic last-block pattern); the
// block that takes the last ticket resets it and signals counter `sig_off` of every
// region with a release at system scope, which (cumulatively) orders all blocks' fenced
// stores before the count the peers wait for. ticket: this rank's, zero between launches.
__device__ __forceinline__ void p2p_signal_last_block(unsigned int* ticket, uint8_t* const* peers, int G,
                                                      int64_t sig_off) {
    __shared__ int s_last;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int nblk = gridDim.x * gridDim.y * gridDim.z;
        s_last = atomicAdd(ticket, 1u) == nblk - 1;
    }
    __syncthreads();
    if (s_last) {
        if (threadIdx.x == 0) *ticket = 0u;
        __threadfence_system();
        for (int g = threadIdx.x; g < G; g += blockDim.x)
            red_release_sys_add_u64(reinterpret_cast<uint64_t*>(peers[g] + sig_off), 1ull);
    }
}

// EP dispatch, empty slots: this rank's meta entries [count_e, cap) in the receive
// buffer of every destination e are set to -1 (count_e from the router; counts ==
// nullptr: no rows at all, every slot empty).
// The dispatch exchange completes here (the permute kernel, which stored the occupied
// slots, has finished before this grid passes its griddepcontrol.wait).
__global__ void moe_ep_p2p_fill_kernel(uint8_t* const* peers, int64_t meta_off, const int32_t* counts, int G,
                                       int cap, int my_rank, unsigned int* ticket, int64_t sig_off) {
    ptx::pdl_wait();
    const int e = blockIdx.y;
    if (e < G) {
        const int n0 = counts ? counts[e] : 0;
        int32_t* meta = reinterpret_cast<int32_t*>(peers[e] + meta_off) + (int64_t)my_rank * cap;
        for (int i = n0 + blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) meta[i] = -1;
    }
    p2p_signal_last_block(ticket, peers, G, sig_off);
    ptx::pdl_launch_dependents();
}

// TP row ownership: rank r finishes tokens [r*T/G, (r+1)*T/G).
__device__ __forceinline__ int tp_owner(int t, int T, int G) {
    return (int)((((int64_t)t + 1) * G + T - 1) / T) - 1;
}
__device__ __forceinline__ int tp_row0(int r, int T, int G) { return (int)(((int64_t)r * T) / G); }

// TP finish (owner side): out rows [t0, t0+n) = bf16_rne(sum_{r=0..G-1} slot_r (+ x)),
// slots summed in ascending rank order; the rows are also kept in this rank's region
// (bf16 and fp32) for the peers to pull.
__global__ void __launch_bounds__(256) moe_tp_p2p_finish_kernel(const float* slots, int G, int shard_max, int t0,
                                                                int n, int d, const __nv_bfloat16* x,
                                                                __nv_bfloat16* out, float* out_f32,
                                                                __nv_bfloat16* keep16, float* keep32,
                                                                uint8_t* const* peers, unsigned int* ticket,
                                                                int64_t sig_off) {
    ptx::pdl_wait();
    const int64_t total = (int64_t)n * d;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < total;
         i += (int64_t)gridDim.x * blockDim.x * 4) {
        float4 r = *reinterpret_cast<const float4*>(slots + i);
        for (int g = 1; g < G; ++g) {
            const float4 u = *reinterpret_cast<const float4*>(slots + (int64_t)g * shard_max * d + i);
            r.x += u.x; r.y += u.y; r.z += u.z; r.w += u.w;
        }
        const int64_t o = (int64_t)t0 * d + i;
        if (x) {
            const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(x + o);
            const float2 a = __bfloat1622float2(xs[0]), b = __bfloat1622float2(xs[1]);
            r.x += a.x; r.y += a.y; r.z += b.x; r.w += b.y;
        }
        __nv_bfloat162 o0 = __floats2bfloat162_rn(r.x, r.y), o1 = __floats2bfloat162_rn(r.z, r.w);
        uint2 ov;
        ov.x = *reinterpret_cast<uint32_t*>(&o0);
        ov.y = *reinterpret_cast<uint32_t*>(&o1);
        *reinterpret_cast<uint2*>(out + o) = ov;
        *reinterpret_cast<uint2*>(keep16 + o) = ov;
        *reinterpret_cast<float4*>(keep32 + o) = r;
        if (out_f32) *reinterpret_cast<float4*>(out_f32 + o) = r;
    }
    p2p_signal_last_block(ticket, peers, G, sig_off);  // the finished rows may be pulled
    ptx::pdl_launch_dependents();
}

// TP all-gather by loads: rows owned by the other ranks are read from their regions.
__global__ void __launch_bounds__(256) moe_tp_p2p_pull_kernel(uint8_t* const* peers, int64_t keep16_off,
                                                              int64_t keep32_off, int G, int my_rank, int T, int d,
                                                              __nv_bfloat16* out, float* out_f32) {
    ptx::pdl_wait();
    const int vec = d / 8;  // 16-byte vectors of bf16 per row
    const int64_t total = (int64_t)T * vec;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(i / vec);
        const int o = tp_owner(t, T, G);
        if (o == my_rank) continue;
        const int64_t e = (int64_t)t * d + (i % vec) * 8;
        reinterpret_cast<uint4*>(out + e)[0] =
            reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(peers[o] + keep16_off) + e)[0];
        if (out_f32) {
            const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(peers[o] + keep32_off) + e);
            float4* dst = reinterpret_cast<float4*>(out_f32 + e);
            dst[0] = src[0];
            dst[1] = src[1];
        }
    }
    ptx::pdl_launch_dependents();
}

}  // namespace moe
