"""Router / pipeline latency at decode sizes: python scripts/exp/router_lat.py
Per-kernel event times (profiling breaks PDL overlap) and the whole-step time of a
small-ffn block (d=4096, f=1024, E=8: GEMMs tiny, so the step is the fixed latency of
the five-kernel chain), for the tensor-core router and the CUDA-core router
(moe_tuning.router_cc_max_T = T_max)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402

f = int(os.environ.get("RL_FFN", "1024"))
w = synth.make_weights(4096, f, 8, seed=0, device="cuda")


def run(T, cc):
    x = synth.make_tokens(T, 4096, seed=1, device="cuda")
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], max_tokens=max(T, 64),
                       tuning={"router_cc_max_T": T} if cc else None)
    for _ in range(10):
        blk.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        blk.forward(x)
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 200 * 1000
    moe.moe_set_profiling(blk.ctx, True)
    moe.moe_reset_profile(blk.ctx)
    for _ in range(100):
        blk.forward(x)
    torch.cuda.synchronize()
    kt = moe.moe_kernel_times(blk.ctx)
    blk.close()
    print(f"T={T:4d} router={'cc ' if cc else 'mma'} step {step:6.1f} us  ",
          {k: round(v[0] / max(v[1], 1) * 1000, 1) for k, v in kt.items() if v[1]}, flush=True)


for T in (1, 16, 64, 256):
    for cc in (False, True):
        run(T, cc)
