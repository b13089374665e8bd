"""Worker for tests/test_gpu_parity.py::test_p2p_multiprocess_ipc (launched by
torch.distributed.run, 2 processes, gloo for the host exchange, both on cuda:0).

Each process owns one EP or TP rank with MOE_FLAG_P2P; the symmetric regions are
connected through CUDA IPC handles all-gathered on the gloo group, so the exchange
steps run as stores/loads into the other process's device memory. Writes this
rank's outputs to <outdir>/rank<r>.pt."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402


def main():
    par, outdir = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    r, G = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    shape = synth.MoEShape(T=96, d=256, f=512, E=8, k=2)
    inp = synth.make_inputs(shape, 81, device="cuda")
    if par == "ep":
        cuts = np.linspace(0, shape.T, G + 1).astype(int)
        x = inp["x"][cuts[r]:cuts[r + 1]]
        pm = moe.MOE_PAR_EP
    else:
        x = inp["x"]
        pm = moe.MOE_PAR_TP
    blk = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=shape.T, par=pm,
                       world_size=G, rank=r, flags=moe.MOE_FLAG_P2P)
    moe.p2p_connect_process_group(blk.ctx)
    T = x.shape[0]
    st = torch.cuda.Stream()
    aux = {"topk_idx": torch.empty(max(T, 1), 2, dtype=torch.int32, device="cuda"),
           "out_f32": torch.empty(max(T, 1), shape.d, dtype=torch.float32, device="cuda")}
    outs = []
    for _ in range(3):
        out = torch.empty(max(T, 1), shape.d, dtype=torch.bfloat16, device="cuda")
        with torch.cuda.stream(st):
            moe.moe_forward(blk.ctx, x, T, blk.router_w, blk.w13, blk.w2, out, aux, st)
        st.synchronize()
        outs.append(out[:T].cpu())
    torch.save({"outs": outs, "out_f32": aux["out_f32"][:T].cpu(), "topk_idx": aux["topk_idx"][:T].cpu()},
               os.path.join(outdir, f"rank{r}.pt"))
    dist.barrier()  # every peer is done with my region before it is freed
    blk.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
