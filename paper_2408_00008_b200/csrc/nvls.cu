// nvls.cu -- the tensor-parallel all-reduce of the MoE block fused into the combine
// kernel through NVLink SHARP multimem ("all-reduce fused into
// the K4 epilogue via NVLS multimem"; Sec. 4.1 tensor parallelism
// Sec. 5 NVLink). Separate translation unit: it includes NCCL 2.28's headers (device API:
// symmetric windows, LSA barriers, multimem pointers), which clash with the handful of
// NCCL declarations moe.cu makes for its dlopen'd host calls. libnccl is never linked:
// the host entry points come from the library torch (or the caller) already loaded.
//
// TP step (reading R7: fp32 reduction, exactly one bf16 rounding) of one launch:
//   1. every block forms the fp32 partial output of its token rows from this rank's
//      expert outputs (the combine of kernels.cuh, same summation order) into the
//      symmetric window;
//   2. LSA barrier (multimem release / acquire) across the TP ranks, per block index;
//   3. each rank owns a column slice of every row: multimem.ld_reduce.add.f32 makes the
//      NVSwitch sum the G partials, + residual, one bf16 rounding, multimem.st writes the
//      bf16 (and fp32) row slice into every rank's window (all-gather by multicast);
//   4. LSA barrier; every block copies its rows from the window to the caller's buffers.
// One kernel instead of combine + fp32 reduce-scatter + finish + bf16 all-gather; no
// host involvement, so the TP forward stays CUDA-graph capturable.
// The NVSwitch sums in its own order: results equal the ascending-rank fp32 sum of the
// collective path up to fp32 rounding (tested against the oracle, not bit-exact).
#include "nvls.h"

#include <dlfcn.h>
#include <cstdio>
#include <cstring>
#include <new>

#if defined(MOE_HAVE_NCCL_DEVICE)
#include <cuda/atomic>
#include <nccl.h>
#include <nccl_device.h>
#endif

namespace moe_nvls {

#if defined(MOE_HAVE_NCCL_DEVICE)

namespace {
struct Api {
    ncclResult_t (*MemAlloc)(void**, size_t);
    ncclResult_t (*MemFree)(void*);
    ncclResult_t (*WindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int);
    ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t);
    ncclResult_t (*DevCommCreate)(ncclComm_t, ncclDevCommRequirements_t const*, ncclDevComm_t*);
    ncclResult_t (*DevCommDestroy)(ncclComm_t, ncclDevComm_t const*);
    ncclResult_t (*CommCount)(const ncclComm_t, int*);
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
    const char* (*GetErrorString)(ncclResult_t);
};

bool load_api(Api& a, char* err, size_t errlen) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the NCCL the communicator came from
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        snprintf(err, errlen, "NVLS: cannot dlopen libnccl.so.2");
        return false;
    }
#define SYM(f, n)                                                            \
    a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, n));                      \
    if (!a.f) {                                                              \
        snprintf(err, errlen, "NVLS: NCCL without %s (needs NCCL >= 2.28)", n); \
        return false;                                                        \
    }
    SYM(MemAlloc, "ncclMemAlloc");
    SYM(MemFree, "ncclMemFree");
    SYM(WindowRegister, "ncclCommWindowRegister");
    SYM(WindowDeregister, "ncclCommWindowDeregister");
    SYM(DevCommCreate, "ncclDevCommCreate");
    SYM(DevCommDestroy, "ncclDevCommDestroy");
    SYM(CommCount, "ncclCommCount");
    SYM(CommUserRank, "ncclCommUserRank");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    return true;
}
}  // namespace

struct State {
    Api api{};
    ncclComm_t comm = nullptr;
    void* buf = nullptr;          // symmetric: [partial f32 | out f32 | out bf16], each max_T x d
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm_t dc{};
    bool dc_made = false;
    int max_T = 0, d = 0, nb = 0, G = 1, rank = 0;
};

namespace {

struct KParams {
    CombineArgs a;
    ncclWindow_t win;
    float* part;                  // local window pointers
    float* of32;
    __nv_bfloat16* ob16;
    size_t off_part, off_f32, off_b16;  // window byte offsets of the three buffers
    int G, rank;
};

__device__ __forceinline__ void mm_ld_reduce_f32x4(const float* mc, float4& v) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(mc)
                 : "memory");
}
__device__ __forceinline__ void mm_st_f32x4(float* mc, const float4& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void mm_st_bf16x4(__nv_bfloat16* mc, uint32_t lo, uint32_t hi) {
    asm volatile("multimem.st.relaxed.sys.global.v2.bf16x2 [%0], {%1, %2};" ::"l"(mc), "r"(lo), "r"(hi) : "memory");
}

__global__ void __launch_bounds__(256) moe_tp_nvls_combine_kernel(const KParams p, const ncclDevComm dc) {
    const CombineArgs& a = p.a;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int nvec = a.d / 4;
    // 1. fp32 partial rows of this rank (kernels.cuh moe_combine_kernel's order: splits
    //    ascending, r = w0 s0, r = fma(w1, s1, r)) -> the window
    for (int t = blockIdx.x; t < a.T; t += gridDim.x) {
        int32_t pr[2];
        float w[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pr[j] = j < a.k ? a.pos[(int64_t)t * a.k + j] : -1;
            w[j] = j < a.k ? a.topk_w[(int64_t)t * a.k + j] : 0.f;
        }
        for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
            float4 s[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (pr[j] >= 0) {
                    const float* yr = a.y + (int64_t)pr[j] * a.d + 4 * v;
                    s[j] = __ldcs(reinterpret_cast<const float4*>(yr));
                    for (int sp = 1; sp < a.splits; ++sp) {
                        const float4 u = __ldcs(reinterpret_cast<const float4*>(yr + sp * a.split_stride));
                        s[j].x += u.x; s[j].y += u.y; s[j].z += u.z; s[j].w += u.w;
                    }
                }
            }
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (pr[0] >= 0) r = make_float4(w[0] * s[0].x, w[0] * s[0].y, w[0] * s[0].z, w[0] * s[0].w);
            if (pr[1] >= 0) {
                r.x = fmaf(w[1], s[1].x, r.x); r.y = fmaf(w[1], s[1].y, r.y);
                r.z = fmaf(w[1], s[1].z, r.z); r.w = fmaf(w[1], s[1].w, r.w);
            }
            reinterpret_cast<float4*>(p.part + (int64_t)t * a.d)[v] = r;
        }
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, /*multimem=*/true);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    // 2. this rank's column slice of every row: switch-side fp32 sum, + residual, one
    //    rounding, multicast stores of the finished slice to every rank
    const int slice = nvec / p.G, v0 = p.rank * slice;
    float* mc_part = static_cast<float*>(ncclGetLsaMultimemPointer(p.win, p.off_part, dc));
    float* mc_f32 = static_cast<float*>(ncclGetLsaMultimemPointer(p.win, p.off_f32, dc));
    __nv_bfloat16* mc_b16 = static_cast<__nv_bfloat16*>(ncclGetLsaMultimemPointer(p.win, p.off_b16, dc));
    const int my_rows = a.T > (int)blockIdx.x ? (a.T - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    for (int i = threadIdx.x; i < my_rows * slice; i += blockDim.x) {
        const int t = blockIdx.x + (i / slice) * gridDim.x, v = v0 + i % slice;
        const int64_t e = (int64_t)t * a.d + 4 * v;
        float4 r;
        mm_ld_reduce_f32x4(mc_part + e, r);
        if (a.x) {
            const __nv_bfloat162* xs = reinterpret_cast<const __nv_bfloat162*>(a.x + e);
            const float2 u = __bfloat1622float2(xs[0]), z = __bfloat1622float2(xs[1]);
            r.x += u.x; r.y += u.y; r.z += z.x; r.w += z.y;
        }
        if (a.out_f32) mm_st_f32x4(mc_f32 + e, r);
        __nv_bfloat162 o0 = __floats2bfloat162_rn(r.x, r.y), o1 = __floats2bfloat162_rn(r.z, r.w);
        mm_st_bf16x4(mc_b16 + e, *reinterpret_cast<uint32_t*>(&o0), *reinterpret_cast<uint32_t*>(&o1));
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    // 3. the finished rows (all slices, from every rank's multicast stores) -> caller
    for (int t = blockIdx.x; t < a.T; t += gridDim.x) {
        const int64_t e = (int64_t)t * a.d;
        for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
            reinterpret_cast<uint2*>(a.out + e)[v] = reinterpret_cast<const uint2*>(p.ob16 + e)[v];
            if (a.out_f32) reinterpret_cast<float4*>(a.out_f32 + e)[v] = reinterpret_cast<const float4*>(p.of32 + e)[v];
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace

int setup(void* nccl_comm, int max_T, int d, int max_blocks, State** out, char* err, size_t errlen) {
    *out = nullptr;
    State* s = new (std::nothrow) State();
    if (!s) {
        snprintf(err, errlen, "NVLS: host allocation failed");
        return 1;
    }
    if (!load_api(s->api, err, errlen)) {
        delete s;
        return 1;
    }
    s->comm = static_cast<ncclComm_t>(nccl_comm);
    s->max_T = max_T;
    s->d = d;
    s->nb = max_blocks;
    const Api& A = s->api;
    auto nfail = [&](const char* what, ncclResult_t r) {
        snprintf(err, errlen, "NVLS: %s failed: %s", what, A.GetErrorString(r));
        destroy(s);
        return 1;
    };
    ncclResult_t r;
    if ((r = A.CommCount(s->comm, &s->G)) || (r = A.CommUserRank(s->comm, &s->rank))) return nfail("comm query", r);
    const size_t one = (size_t)max_T * d * 4;
    s->bytes = (2 * one + (size_t)max_T * d * 2 + 4095) / 4096 * 4096;
    if ((r = A.MemAlloc(&s->buf, s->bytes))) return nfail("ncclMemAlloc", r);
    if ((r = A.WindowRegister(s->comm, s->buf, s->bytes, &s->win, NCCL_WIN_COLL_SYMMETRIC)))
        return nfail("ncclCommWindowRegister", r);
    ncclDevCommRequirements_t req;
    memset(&req, 0, sizeof(req));
    req.lsaMultimem = true;
    req.lsaBarrierCount = max_blocks;
    if ((r = A.DevCommCreate(s->comm, &req, &s->dc))) return nfail("ncclDevCommCreate", r);
    s->dc_made = true;
    if (s->dc.lsaSize != s->G || s->dc.lsaMultimem.mcBasePtr == nullptr) {
        snprintf(err, errlen,
                 "NVLS: no multicast object over the %d TP ranks (LSA team %d, multimem %s): NVLink SHARP needs "
                 ">= 2 GPUs of one NVSwitch domain",
                 s->G, s->dc.lsaSize, s->dc.lsaMultimem.mcBasePtr ? "yes" : "no");
        destroy(s);
        return 1;
    }
    *out = s;
    return 0;
}

void destroy(State* s) {
    if (!s) return;
    if (s->dc_made) s->api.DevCommDestroy(s->comm, &s->dc);
    if (s->win) s->api.WindowDeregister(s->comm, s->win);
    if (s->buf) s->api.MemFree(s->buf);
    delete s;
}

int max_blocks(const State* s) { return s ? s->nb : 0; }

cudaError_t launch_tp_combine(State* s, const CombineArgs& a, int nblocks, bool pdl, cudaStream_t st) {
    KParams p{};
    p.a = a;
    p.win = s->win;
    const size_t one = (size_t)s->max_T * s->d * 4;
    p.off_part = 0;
    p.off_f32 = one;
    p.off_b16 = 2 * one;
    p.part = static_cast<float*>(s->buf);
    p.of32 = reinterpret_cast<float*>(static_cast<char*>(s->buf) + one);
    p.ob16 = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(s->buf) + 2 * one);
    p.G = s->G;
    p.rank = s->dc.lsaRank;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nblocks < s->nb ? nblocks : s->nb);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, moe_tp_nvls_combine_kernel, p, s->dc);
}

#else  // built without NCCL 2.28's device API headers

struct State {};
int setup(void*, int, int, int, State** out, char* err, size_t errlen) {
    *out = nullptr;
    snprintf(err, errlen, "NVLS: libmoe was built without NCCL 2.28 device-API headers");
    return 1;
}
void destroy(State*) {}
int max_blocks(const State*) { return 0; }
cudaError_t launch_tp_combine(State*, const CombineArgs&, int, bool, cudaStream_t) { return cudaErrorNotSupported; }

#endif

}  // namespace moe_nvls
