"""Small forwards over every kernel family, for compute-sanitizer (scripts/sanitize.sh):
swap-AB decode GEMMs, CTA-pair and 1-CTA prefill tiles, tile::gather4 token fetch,
FP8 weights, and the EP / TP paths over the loopback and the
peer-memory (MOE_FLAG_P2P) transports at G = 2."""
import os
import sys
import threading

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402


def single(shape, flags, tuning=None):
    inp = synth.make_inputs(shape, 5, device="cuda")
    w = dict(inp)
    if flags & moe.MOE_FLAG_FP8_WEIGHTS:
        for n in ("w1", "w3", "w2"):
            w[n] = synth.quantize_fp8_rows(w[n])
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], max_tokens=shape.T, flags=flags, tuning=tuning)
    blk.forward(inp["x"])
    torch.cuda.synchronize()
    blk.close()
    print("ok", shape, hex(flags), tuning, flush=True)


def group(par, G, p2p, tuning=None):
    shape = synth.MoEShape(T=48, d=256, f=512, E=4, k=2)
    inp = synth.make_inputs(shape, 6, device="cuda")
    flags = moe.MOE_FLAG_P2P if p2p else 0
    grp = None if p2p else moe.moe_loopback_comm_create(G)
    comms = [None] * G if p2p else [moe.moe_loopback_comm_rank(grp, r) for r in range(G)]
    pm = moe.MOE_PAR_EP if par == "ep" else moe.MOE_PAR_TP
    blocks = [moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], max_tokens=48, par=pm, world_size=G, rank=r,
                           nccl_comm=comms[r], flags=flags, tuning=tuning) for r in range(G)]
    if p2p:
        hs = [b.p2p_handle() for b in blocks]
        for b in blocks:
            b.p2p_connect(hs)
    streams = [torch.cuda.Stream() for _ in range(G)]
    torch.cuda.synchronize()

    def work(r):
        x = inp["x"][r * 24:(r + 1) * 24] if par == "ep" else inp["x"]
        with torch.cuda.stream(streams[r]):
            for _ in range(2):
                blocks[r].forward(x, stream=streams[r])
        streams[r].synchronize()

    ths = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for b in blocks:
        b.close()
    if grp is not None:
        for c in comms:
            moe.moe_loopback_comm_destroy(c)
        moe.moe_loopback_comm_destroy(grp)
    print("ok", par, G, "p2p" if p2p else "loopback", tuning, flush=True)


if __name__ == "__main__":
    small = synth.MoEShape(T=40, d=256, f=512, E=4, k=2)
    single(small, 0x2)                       # swap-AB
    single(small, 0x4)                       # CTA pair
    single(small, 0x4 | 0x10)                # 1-CTA tiles
    single(small, 0x2 | moe.MOE_FLAG_GATHER)  # gather4, swap
    single(small, 0x4 | moe.MOE_FLAG_GATHER)  # gather4, pair
    single(synth.MoEShape(T=64, d=1024, f=2560, E=8, k=2), 0x2)  # speculative L2 prefetch, auto grids
    single(synth.MoEShape(T=32, d=256, f=512, E=4, k=2), moe.MOE_FLAG_FP8_WEIGHTS)   # FP8, block-scaled w2
    single(synth.MoEShape(T=200, d=256, f=512, E=4, k=2), moe.MOE_FLAG_FP8_WEIGHTS, {"swap_nb_cap": 32})
    single(synth.MoEShape(T=600, d=256, f=512, E=8, k=2), 0x2)   # token tile 192 (T=575-like): CTA-pair swap
    single(synth.MoEShape(T=600, d=256, f=512, E=8, k=2), 0x2, {"swap_pair": 1})  # same on single-CTA swap tiles
    single(synth.MoEShape(T=300, d=256, f=512, E=8, k=2), 0x2)   # CTA-pair swap, token tile 128
    single(synth.MoEShape(T=1000, d=320, f=512, E=8, k=2), 0x2, {"swap_pair": 2})  # pair tile 256 + 2nd tiles, padded d
    # fused decode FFN (ffn_fused.cuh): cross-CTA h readiness / tile claims / counter resets
    fz = synth.MoEShape(T=64, d=1024, f=2560, E=8, k=2)
    single(fz, 0, {"fused": 2})                                   # tapered splits, 256-row w1/w3 tiles
    single(fz, 0, {"fused": 2, "fused_half": 2})                  # 128-row w1/w3 tiles (smem a/b exchange)
    single(fz, 0, {"fused": 2, "fused_chain": 1, "fused_splits": 8})  # split chaining
    single(fz, moe.MOE_FLAG_RESIDUAL, {"fused": 2, "fused_combine": 1})  # in-kernel combine
    single(synth.MoEShape(T=100, d=512, f=1024, E=4, k=2), 0, {"fused": 2, "swap_nb_cap": 32})  # several token tiles
    for par in ("ep", "tp"):
        for p2p in (False, True):
            group(par, 2, p2p)
    group("tp", 2, False, {"fused": 2})
