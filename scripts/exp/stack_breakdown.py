"""Per-kernel times of the mid-size (stack, T=575) forward on one Mixtral layer:
python scripts/exp/stack_breakdown.py [T] [flags] [field=v,... (moe_tuning)]  (profiling events break PDL overlap)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 575
flags = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0
tuning = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
w = synth.make_weights(4096, 14336, 8, seed=0, device="cuda")
x = synth.make_tokens(T, 4096, seed=1, device="cuda")
blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], max_tokens=T, flags=flags, tuning=tuning)
counts = torch.empty(8, dtype=torch.int32, device="cuda")
for _ in range(5):
    blk.forward(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    blk.forward(x)
e1.record()
torch.cuda.synchronize()
print(f"T={T} flags={flags:#x} step {e0.elapsed_time(e1) / 50 * 1000:.1f} us")
moe.moe_set_profiling(blk.ctx, True)
moe.moe_reset_profile(blk.ctx)
for _ in range(20):
    blk.forward(x, aux={"expert_counts": counts})
torch.cuda.synchronize()
kt = moe.moe_kernel_times(blk.ctx)
print({k: round(v[0] / max(v[1], 1) * 1000, 1) for k, v in kt.items() if v[1]}, "us/launch")
print("counts", counts.tolist())
