"""Power / clock comparison at prefill: cuBLAS bf16 GEMM of the GEMM1 shape vs libmoe's
prefill forward, each run back to back for a few seconds with nvidia-smi sampling.

Question it answers: under the 1 kW cap, does the prefill w1/w3 GEMM (kG1Pair) run at a
lower SM clock than a library GEMM of the same FLOPs (i.e. is it spending more power per
FLOP), or only at a lower fraction of its clock's peak?

usage (GPU box): python scripts/exp/power_ab.py [seconds]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402  (ClockSampler)
import synth  # noqa: E402


def sampler_stats(cs):
    rows = [r for r in cs.rows if len(r) >= 9]
    sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
    pw = sorted(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
    med = lambda v: v[len(v) // 2] if v else None  # noqa: E731
    return {"sm_mhz_med": med(sm), "power_w_med": med(pw), "n": len(sm)}


def run_loop(fn, seconds, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    cs = bench.ClockSampler(0)
    cs.start()
    t0 = time.perf_counter()
    n = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(4):
            fn()
            n += 1
        torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / n
    cs.stop()
    s = sampler_stats(cs)
    s.update({"ms": ms, "tflops": flops / ms / 1e9})
    return s


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    T, d, f, E, k = 32768, 4096, 14336, 8, 2
    # 1. cuBLAS: all 65536 assignments through one [2f, d] weight (same FLOPs as GEMM1)
    a = torch.randn(T * k, d, device=dev, dtype=torch.bfloat16)
    b = (torch.randn(2 * f, d, device=dev) / d ** 0.5).to(torch.bfloat16)
    c = torch.empty(T * k, 2 * f, device=dev, dtype=torch.bfloat16)
    fl = 2.0 * T * k * 2 * f * d
    print("cublas_g1_shape", run_loop(lambda: torch.matmul(a, b.t(), out=c), secs, fl), flush=True)
    del a, b, c
    torch.cuda.empty_cache()
    # 2. libmoe prefill forward (all five kernels); GEMM1 share from kernel events
    import paper_2408_00008_b200 as moe
    w = synth.make_weights(d, f, E, seed=0, device=dev)
    x = synth.make_tokens(T, d, seed=1, device=dev)
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=k, max_tokens=T)
    del w
    torch.cuda.empty_cache()
    out = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
    st = torch.cuda.current_stream()

    def fwd():
        moe.moe_forward(blk.ctx, x, T, blk.router_w, blk.w13, blk.w2, out, None, st, blk.s13, blk.s2)

    fl_all = 2.0 * T * k * 3 * d * f + 2.0 * T * d * E
    print("libmoe_prefill", run_loop(fwd, secs, fl_all), flush=True)
    moe.moe_reset_profile(blk.ctx)
    moe.moe_set_profiling(blk.ctx, True)
    for _ in range(5):
        fwd()
    torch.cuda.synchronize()
    print("libmoe_kernel_ms", moe.moe_kernel_times(blk.ctx), flush=True)
    moe.moe_set_profiling(blk.ctx, False)
    blk.close()


if __name__ == "__main__":
    main()
