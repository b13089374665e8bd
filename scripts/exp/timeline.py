"""Per-block kernel timeline of one graph-replayed MoE forward (probe build only).

Build:  python paper_2408_00008_b200/_build.py --force --out build_ab/libmoe_tl.so -DMOE_TIMELINE=1
Run:    MOE_LIB=build_ab/libmoe_tl.so python scripts/exp/timeline.py T [tuning k=v,...|-] [--residual] [--fp8]
        [--shard ep2|ep4|ep8|tp2|tp4|tp8]   (one rank's share: E/G experts top-1 over its rows, or f/G columns)
With tuning fused=2 the w1/w3 slot is the fused FFN kernel and slot 3 holds its producer
probes: first w2-tile claim, last (failing) claim, and the time spent waiting for h tiles.

The probe build stamps %globaltimer (ns) in thread 0 of every block at kernel entry,
after griddepcontrol.wait and at exit (csrc/sm100.cuh MOE_TL). After back-to-back graph
replays of one layer forward the last replay's stamps are read back and summarised per
kernel: first/last entry, first/last post-wait, first/last exit, relative to the router's
first entry -- where the step's time goes between and inside the kernels (PDL overlap,
tails, waves). Synthetic Mixtral 8x7B layer (synth recipe), inputs resident in HBM.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2408_00008_b200 as moe  # noqa: E402
import synth  # noqa: E402

SLOTS = ["router", "permute", "gemm1", "gemm2", "combine"]
TL_BLOCKS = 4096


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 575
    tuning = None
    if len(sys.argv) > 2 and sys.argv[2] != "-":
        tuning = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[2].split(","))}
    flags = moe.MOE_FLAG_RESIDUAL if "--residual" in sys.argv else 0
    fp8 = "--fp8" in sys.argv
    lib = moe._lib
    if not hasattr(lib, "moe_debug_timeline"):
        raise SystemExit("not a MOE_TIMELINE build (set MOE_LIB=build_ab/libmoe_tl.so)")
    lib.moe_debug_timeline.argtypes = [ctypes.c_void_p]
    lib.moe_debug_timeline.restype = ctypes.c_int
    d, f, E = 4096, 14336, 8
    w = synth.make_weights(d, f, E, 1, 0, device="cuda", w2_scale=synth.STACK_W2_SCALE)
    if fp8:  # E4M3 weights with per-row scales (bench.py --fp8)
        flags |= moe.MOE_FLAG_FP8_WEIGHTS
        for n in ("w1", "w3", "w2"):
            w[n] = synth.quantize_fp8_rows(w[n])
    x = synth.make_tokens(T, d, 1, 0, device="cuda")
    shard = next((a.split("=", 1)[1] if "=" in a else sys.argv[sys.argv.index(a) + 1]
                  for a in sys.argv if a.startswith("--shard")), None)
    k = 2
    if shard and shard.startswith("tp"):  # this rank's f/G ffn slice of every expert, whole batch
        fl = f // int(shard[2:])
        w = {"wg": w["wg"], "w1": w["w1"][:, :fl].contiguous(), "w3": w["w3"][:, :fl].contiguous(),
             "w2": w["w2"][:, :, :fl].contiguous()}
    elif shard and shard.startswith("ep"):  # E/G experts; the rows routed to them (~T*k/G), top-1
        G = int(shard[2:])
        el = E // G
        w = {n: w[n][:el].contiguous() for n in ("wg", "w1", "w3", "w2")}
        T = max(1, T * 2 // G)
        x = x[:T].contiguous()
        k = 1
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=k, max_tokens=T, flags=flags, tuning=tuning)
    del w
    out = torch.empty_like(x)

    def step():
        blk.forward(x, out, stream=torch.cuda.current_stream())

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    buf = np.zeros(5 * 3 * TL_BLOCKS, np.uint64)
    lib.moe_debug_timeline(buf.ctypes.data)  # clears the stamps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(20):
        g.replay()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 20
    assert lib.moe_debug_timeline(buf.ctypes.data) == 0
    tl = buf.reshape(5, 3, TL_BLOCKS).astype(np.int64)
    t0 = tl[0, 0][tl[0, 0] > 0].min()
    print(f"T={T} tuning={tuning} graph step {ms * 1000:.1f} us (20 replays); stamps of the last replay, us from router entry")
    print(f"{'kernel':8s} {'blocks':>6s} {'entry first..last':>20s} {'waited first..last':>20s} {'exit first..last':>20s}")
    ends = {}
    for s, name in enumerate(SLOTS):
        ent, wt, ex = tl[s]
        m = ent > 0
        if not m.any():
            continue
        r = lambda a: (a[a > 0] - t0) / 1000.0  # noqa: E731
        e, w_, x_ = r(ent), r(wt), r(ex)
        fmt = lambda a: f"{a.min():8.1f}..{a.max():8.1f}" if a.size else " " * 20  # noqa: E731
        print(f"{name:8s} {int(m.sum()):6d} {fmt(e)} {fmt(w_)} {fmt(x_)}")
        ends[name] = x_
        if name == "gemm2" and tuning and tuning.get("fused") == 2:
            stall = (tl[s][2][m] - tl[2][0][m]) / 1000.0
            print(f"  (fused producer: first w2 claim {fmt(e)}, last claim {fmt(w_)}, "
                  f"h-wait us p50/p90/max {np.percentile(stall, 50):.1f}/{np.percentile(stall, 90):.1f}/{stall.max():.1f})")
            continue
        if name in ("gemm1", "gemm2") and x_.size:
            q = np.percentile(x_, [0, 10, 50, 90, 100])
            print(f"         exit percentiles 0/10/50/90/100: " + " ".join(f"{v:.1f}" for v in q))
    if "--teardown" in sys.argv:  # MOE_TL_TEARDOWN build: slot 3 = fused FFN exit hand-off stamps
        a, b, c = tl[3]
        x = tl[2][2]
        m = (a > 0) & (x > 0)
        last = np.argmax(np.where(m, x, 0))
        us = lambda v: (v - t0) / 1000.0  # noqa: E731
        print(f"fused exit hand-off, last CTA {last}: fence done {us(a[last]):.1f}, atomic back {us(b[last]):.1f}, "
              f"barrier {us(c[last]):.1f}, exit {us(x[last]):.1f}")
        for lbl, v in (("fence->atomic", b - a), ("atomic->barrier", c - b), ("barrier->exit", x - c)):
            q = np.percentile(v[m] / 1000.0, [50, 90, 100])
            print(f"  {lbl:16s} p50/p90/max us {q[0]:.2f}/{q[1]:.2f}/{q[2]:.2f}")
    blk.close()


if __name__ == "__main__":
    main()
