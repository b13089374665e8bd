"""C5 stack (32 Mixtral layers, T = 575): eager launches vs one CUDA graph of the whole
32-layer forward, interleaved; with a MOE_TIMELINE build (MOE_LIB) also the per-kernel
stamps of the last layer. Synthetic stack recipe (synth.STACK_W2_SCALE)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2408_00008_b200 as moe  # noqa: E402
import synth  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 575
L = 32
d, f, E = 4096, 14336, 8
dev = torch.device("cuda", 0)
st = moe.MoEStack([synth.make_weights(d, f, E, 1, 0, device=dev, w2_scale=synth.STACK_W2_SCALE)], max_tokens=T)
for l in range(1, L):
    lw = synth.make_weights(d, f, E, 1, l, device=dev, w2_scale=synth.STACK_W2_SCALE)
    st.add_layer(lw)
    del lw
torch.cuda.empty_cache()
x = synth.make_tokens(T, d, 2, device=dev)
out = torch.empty_like(x)


def step():
    st.forward(x, out, torch.cuda.current_stream())


for _ in range(3):
    step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
g.replay()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(3):
    for name, fn in (("eager", step), ("graph", g.replay)):
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(5):
            fn()
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / 5
        print(f"{name} round {r}: {ms:.3f} ms per 32-layer step, {ms / L * 1000:.1f} us per layer, {T / ms * 1000:.0f} tok/s")
lib = moe._lib
if hasattr(lib, "moe_debug_timeline"):
    lib.moe_debug_timeline.argtypes = [ctypes.c_void_p]
    buf = np.zeros(5 * 3 * 4096, np.uint64)
    for name, fn in (("eager", step), ("graph", g.replay)):
        fn()
        torch.cuda.synchronize()
        lib.moe_debug_timeline(buf.ctypes.data)
        tl = buf.reshape(5, 3, 4096).astype(np.int64)
        t0 = tl[0, 0][tl[0, 0] > 0].min()
        print(f"{name}: last layer, us from its router entry")
        for s, kn in enumerate(["router", "permute", "gemm1", "gemm2", "combine"]):
            e, w_, x_ = ((a[a > 0] - t0) / 1000.0 for a in tl[s])
            if e.size:
                print(f"  {kn:8s} {e.size:5d} entry {e.min():8.1f}..{e.max():8.1f} waited {w_.min():8.1f}..{w_.max():8.1f} "
                      f"exit {x_.min():8.1f}..{x_.max():8.1f}")
