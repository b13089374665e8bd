"""World-size-2 CPU tests (gloo) of the multi-process host logic of the EP / TP
variants (Sec. 4.1):
  * the NCCL unique-id handshake libmoe's communicator needs (rank 0 draws it
    through the C ABI, the host process group broadcasts it);
  * the EP token sharding / expert ownership and the TP ffn slicing, exercised
    end to end across two real processes with gloo collectives standing in for
    NCCL: each rank computes its share with the fp64 oracle's partition
    emulation (EP: its experts' contributions; TP: its ffn slice), the ranks
    exchange (EP: all-to-all of per-token partials back to the owner; TP:
    all-reduce), and the result must equal the single-process oracle;
  * bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = fn(rank, world)
        q.put((rank, "ok", out))
    except Exception as ex:  # surfaced to the parent
        import traceback
        q.put((rank, "err", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, st, out = q.get(timeout=300)
        assert st == "ok", out
        res[r] = out
    for p in ps:
        p.join(timeout=60)
    return res


def _uid_fn(rank, world):
    import paper_2408_00008_b200 as moe
    obj = [moe.moe_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def test_nccl_unique_id_handshake():
    res = _spawn(_uid_fn)
    assert len(res[0]) == 128 and res[0] == res[1]


def _inputs():
    import synth
    shape = synth.MoEShape(T=24, d=64, f=256, E=4, k=2)
    inp = synth.make_inputs(shape, seed=77)
    return {k: synth.bf16_bits(v) for k, v in inp.items()}


def _ep_fn(rank, world):
    """EP: tokens sharded across ranks; every rank evaluates ITS experts for every
    token routed to them (partition mode 'ep' of the oracle over the global batch
    it receives), then the per-token partial rows go back to their source rank
    (all_to_all), which sums them -- the dispatch / combine round trip."""
    import oracle
    h = _inputs()
    T = h["x"].shape[0]
    # token shard of each rank (contiguous, uneven)
    cuts = [0, 10, T]
    # dispatch: every rank needs the rows routed to its experts -> here every rank
    # gathers all shards (all_gather of token rows), then computes its experts' part
    mine = torch.from_numpy(h["x"][cuts[rank]:cuts[rank + 1]].astype(np.int32))
    sizes = [cuts[r + 1] - cuts[r] for r in range(world)]
    gathered = [torch.zeros(s, h["x"].shape[1], dtype=torch.int32) for s in sizes]
    _all_gather_uneven(gathered, mine, rank)
    xg = torch.cat(gathered).numpy().astype(np.uint16)
    assert np.array_equal(xg, h["x"])
    P = oracle.partition(xg, h["wg"], h["w1"], h["w3"], h["w2"], k=2, G=world, mode="ep")[rank]  # [T, d]
    # combine: send each source rank the partial rows of its tokens, sum at the source
    send = [torch.from_numpy(P[cuts[r]:cuts[r + 1]].copy()) for r in range(world)]
    recv = [torch.zeros(sizes[rank], h["x"].shape[1], dtype=torch.float64) for _ in range(world)]
    _all_to_all(send, recv, rank, world)
    y_mine = sum(recv)
    y_ref = oracle.moe_forward(h["x"], h["wg"], h["w1"], h["w3"], h["w2"], 2)[cuts[rank]:cuts[rank + 1]]
    return float(np.max(np.abs(y_mine.numpy() - y_ref)))


def _all_gather_uneven(gathered, mine, rank):
    for r in range(len(gathered)):
        buf = mine.clone() if r == rank else gathered[r]
        dist.broadcast(buf, src=r)
        gathered[r] = buf


def _all_to_all(send, recv, rank, world):
    """recv[p] <- send of rank p addressed to me (point-to-point on gloo)."""
    reqs = []
    for p in range(world):
        if p == rank:
            recv[p].copy_(send[p])
            continue
        reqs.append(dist.isend(send[p].contiguous(), dst=p))
        reqs.append(dist.irecv(recv[p], src=p))
    for r in reqs:
        r.wait()


def test_ep_two_process_exchange():
    res = _spawn(_ep_fn)
    assert res[0] < 1e-12 and res[1] < 1e-12, res


def _tp_fn(rank, world):
    """TP: every rank holds the full batch and its ffn slice; the fp32 partials are
    summed by an all-reduce (libmoe: reduce-scatter + all-gather)."""
    import oracle
    h = _inputs()
    P = oracle.partition(h["x"], h["wg"], h["w1"], h["w3"], h["w2"], k=2, G=world, mode="tp")[rank]
    t = torch.from_numpy(P.copy())
    dist.all_reduce(t)
    y = oracle.moe_forward(h["x"], h["wg"], h["w1"], h["w3"], h["w2"], 2)
    return float(np.max(np.abs(t.numpy() - y)))


def test_tp_two_process_allreduce():
    res = _spawn(_tp_fn)
    assert res[0] < 1e-12 and res[1] < 1e-12, res


def _timing_fn(rank, world):
    """bench.py reports the MAX over ranks of the device-timed step."""
    ms = torch.tensor([1.0 + rank, 5.0 - rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return ms.tolist()


def test_max_over_ranks_reduction():
    res = _spawn(_timing_fn)
    assert res[0] == res[1] == [2.0, 5.0]
