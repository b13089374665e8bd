// nvls.h -- internal interface of nvls.cu (no NCCL or torch types): the tensor-parallel
// all-reduce of the MoE block fused into its combine kernel through NVLink SHARP
// (multimem) on NCCL 2.28 symmetric memory. SURVEY.md 8(f) NEXT #3
// (Sec. 4.1, "tensor parallelism ... splitting tensors"), P:171 (Sec. 5, NVLink).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace moe_nvls {

struct State;  // symmetric window + device communicator of one context (opaque)

// What the fused kernel needs from the combine step (kernels.cuh CombineParams, same
// meaning): this rank's fp32 expert outputs y (split-K partials), the routing of every
// token, the residual source and the caller's outputs.
struct CombineArgs {
    const float* y;
    int64_t split_stride;
    int32_t splits;
    const int32_t* pos;
    const float* topk_w;
    const __nv_bfloat16* x;   // residual (nullable)
    int32_t T, d, k;
    __nv_bfloat16* out;       // [T, d]
    float* out_f32;           // [T, d] (nullable)
};

// Collective over the TP communicator (every rank calls it): allocates a symmetric window
// of 2 fp32 + 1 bf16 [max_T, d] buffers with ncclMemAlloc, registers it
// (NCCL_WIN_COLL_SYMMETRIC) and creates a device communicator with LSA multimem and
// `max_blocks` LSA barriers. Returns 0, or nonzero with a message in err when the NCCL
// in the process has no device API (< 2.28) or the ranks have no multicast object
// (NVLS needs >= 2 GPUs on one NVSwitch domain).
int setup(void* nccl_comm, int max_T, int d, int max_blocks, State** out, char* err, size_t errlen);
void destroy(State* s);
int max_blocks(const State* s);

// One launch: fp32 partial combine of every token row into the window, LSA barrier,
// multimem.ld_reduce of this rank's column slice (switch-side fp32 sum over the ranks),
// + residual, one bf16 rounding, multimem.st of the bf16 (and fp32) rows to every rank,
// LSA barrier, copy of the rows into the caller's buffers.
cudaError_t launch_tp_combine(State* s, const CombineArgs& a, int nblocks, bool pdl, cudaStream_t st);

}  // namespace moe_nvls
