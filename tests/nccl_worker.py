"""Worker for tests/test_gpu_parity.py::test_real_nccl_multigpu (launched by
torch.distributed.run, one process per GPU, NCCL for the collectives): the EP, TP
and hybrid EP x TP variants over REAL NCCL communicators (libmoe's own, built from
the process group with nccl_comm_from_process_group / nccl_hybrid_comms), capacity
and exact-count EP exchanges, the peer-memory (MOE_FLAG_P2P) transport across
GPUs and the NVLink SHARP TP all-reduce fused into the combine (MOE_FLAG_NVLS). Writes this rank's outputs per case to <outdir>/rank<r>.pt."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402

SHAPE = synth.MoEShape(T=96, d=512, f=1024, E=8, k=2)


def cases(G):
    yield "ep", dict(par=moe.MOE_PAR_EP, flags=0)
    yield "ep_exact", dict(par=moe.MOE_PAR_EP, flags=moe.MOE_FLAG_EP_EXACT)
    yield "tp", dict(par=moe.MOE_PAR_TP, flags=0)
    yield "ep_p2p", dict(par=moe.MOE_PAR_EP, flags=moe.MOE_FLAG_P2P)
    yield "tp_p2p", dict(par=moe.MOE_PAR_TP, flags=moe.MOE_FLAG_P2P)
    yield "tp_nvls", dict(par=moe.MOE_PAR_TP, flags=moe.MOE_FLAG_NVLS)
    if G % 2 == 0:
        yield "hybrid", dict(par=moe.MOE_PAR_HYBRID, flags=0, tp=2)


def main():
    outdir = sys.argv[1]
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    r, G = dist.get_rank(), dist.get_world_size()
    inp = synth.make_inputs(SHAPE, 91, device="cuda")
    res = {}
    for name, c in cases(G):
        tp = c.get("tp", 0)
        comm = tp_comm = None
        if c["par"] == moe.MOE_PAR_HYBRID:
            comm, tp_comm = moe.nccl_hybrid_comms(G, r, tp, local)
            shard, nshard = r // tp, G // tp
        elif not c["flags"] & moe.MOE_FLAG_P2P:
            comm = moe.nccl_comm_from_process_group(G, r, local)
        if c["par"] == moe.MOE_PAR_TP:
            shard, nshard = 0, 1
        elif c["par"] == moe.MOE_PAR_EP:
            shard, nshard = r, G
        cuts = np.linspace(0, SHAPE.T, nshard + 1).astype(int)
        x = inp["x"][cuts[shard]:cuts[shard + 1]]
        blk = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=SHAPE.T, par=c["par"],
                           world_size=G, rank=r, nccl_comm=comm, flags=c["flags"], tp_size=tp, tp_comm=tp_comm)
        if c["flags"] & moe.MOE_FLAG_P2P:
            moe.p2p_connect_process_group(blk.ctx)
        T = x.shape[0]
        aux = {"topk_idx": torch.empty(max(T, 1), 2, dtype=torch.int32, device="cuda"),
               "out_f32": torch.empty(max(T, 1), SHAPE.d, dtype=torch.float32, device="cuda")}
        outs = []
        for _ in range(2):
            out = torch.empty(max(T, 1), SHAPE.d, dtype=torch.bfloat16, device="cuda")
            moe.moe_forward(blk.ctx, x, T, blk.router_w, blk.w13, blk.w2, out, aux, None)
            torch.cuda.synchronize()
            outs.append(out[:T].cpu())
        res[name] = {"shard": shard, "nshard": nshard, "outs": outs, "out_f32": aux["out_f32"][:T].cpu(),
                     "topk_idx": aux["topk_idx"][:T].cpu()}
        dist.barrier()
        blk.close()
        for cm in (comm, tp_comm):
            if cm is not None:
                moe.moe_nccl_comm_destroy(cm)
    torch.save(res, os.path.join(outdir, f"rank{r}.pt"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
