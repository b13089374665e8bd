"""Debug driver for MOE_FLAG_P2P on one GPU: G in-process ranks, per-rank progress
printed, run under `timeout`. usage: python scripts/exp/p2p_debug.py ep|tp G"""
import os
import sys
import threading
import traceback

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402

par, G = sys.argv[1], int(sys.argv[2])
shape = synth.MoEShape(T=96, d=256, f=512, E=8, k=2)
inp = synth.make_inputs(shape, 70 + G, device="cuda")
pm = moe.MOE_PAR_EP if par == "ep" else moe.MOE_PAR_TP
blocks = [moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=96, par=pm, world_size=G,
                       rank=r, flags=moe.MOE_FLAG_P2P | 0x2) for r in range(G)]
hs = [b.p2p_handle() for b in blocks]
for b in blocks:
    b.p2p_connect(hs)
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in range(G)]
print("setup ok", flush=True)


def work(r):
    try:
        x = inp["x"] if par == "tp" else inp["x"][r * 96 // G:(r + 1) * 96 // G]
        out = torch.empty_like(x)
        for it in range(2):
            with torch.cuda.stream(streams[r]):
                moe.moe_forward(blocks[r].ctx, x, x.shape[0], blocks[r].router_w, blocks[r].w13, blocks[r].w2, out,
                                None, streams[r])
            print(f"rank {r} it {it} enqueued", flush=True)
            streams[r].synchronize()
            print(f"rank {r} it {it} done", flush=True)
    except Exception:
        traceback.print_exc()
        sys.stdout.flush()


ths = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(G)]
for t in ths:
    t.start()
for t in ths:
    t.join(30)
print("alive:", [t.is_alive() for t in ths], flush=True)
os._exit(0)
