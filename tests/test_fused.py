"""GPU parity of the fused decode FFN (moe_ffn_fused_kernel, csrc/ffn_fused.cuh; tuning
fused=2): the w1/w3 + SwiGLU tiles and the w2 tiles of every expert in ONE persistent
launch, w2 tiles waiting per 128-column h tile through counters in global memory.

Checks, all through the C ABI:
- oracle parity (routing, out_f32 within 2e-2 of the row RMS, bf16 out = RNE(out_f32))
  over ragged token counts, odd ffn-tile counts, uneven K splits, empty experts, several
  token tiles per expert (a w2 tile then waits for every token tile of its h columns);
- bit-identity with the two-kernel swap path at the same K split where the split
  boundaries coincide (the same MMAs per output element in the same K order);
- repeated forwards and CUDA-graph replays (the device-side claim / ready counters are
  reset by the last CTA of each launch);
- EP / TP contexts (loopback transport) and the Mixtral-size 64-token decode.
"""
import numpy as np
import pytest
import torch

import synth
from parity import GpuRun, check_forward, to_host_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def moe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2408_00008_b200 as m
    return m


def _block(moe, inp, k, T, tuning, split_k=0, flags=0):
    return moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=k, max_tokens=T, flags=flags,
                        split_k=split_k, tuning=tuning)


def _launches(moe, blk, x):
    n0 = moe.moe_launch_count(blk.ctx)
    blk.forward(x)
    torch.cuda.synchronize()
    return moe.moe_launch_count(blk.ctx) - n0


@pytest.mark.parametrize("half", [1, 2])
@pytest.mark.parametrize("uniform,chain", [(0, 0), (1, 0), (0, 1), (1, 1), (4, 0), (2, 0)])
@pytest.mark.parametrize("T,d,f,E,k,splits", [
    (64, 512, 1024, 8, 2, 0),    # decode-like: one token tile per expert (NB 64), auto splits
    (1, 256, 512, 4, 2, 1),      # one token: 2 experts used, 2 empty
    (40, 256, 1024, 8, 2, 2),
    (40, 256, 1024, 8, 2, 3),    # 8 ffn tiles over 3 splits: 2 / 3 / 3 tiles
    (100, 256, 384, 2, 2, 2),    # 3 ffn tiles: splits of 1 and 2 tiles; NB 128
    (77, 768, 256, 8, 1, 4),     # top-1, 2 ffn tiles over 4 splits -> 2 (capped by the tile count)
    (16, 256, 256, 4, 2, 1),     # NB 32 (16 rows bound), single ffn tile pair
    (128, 512, 512, 6, 2, 4),    # NB 128, ragged expert segments
    (48, 256, 2048, 8, 2, 8),    # 16 ffn tiles over 8 tapered splits (8 partial buffers)
])
def test_fused_parity(moe, T, d, f, E, k, splits, uniform, chain, half):
    """Tapered (default: geometric or linear by shape; 4 / 2 forced), uniform and chained w2 K
    splits, incl. more splits than ffn tiles allow;
    256-row w1/w3 tiles (fused_half 1) and 128-row ones (2: 64 w1 + 64 w3 rows, a/b paired
    through shared memory)."""
    shape = synth.MoEShape(T=T, d=d, f=f, E=E, k=k)
    inp = synth.make_inputs(shape, 7100 + T + d + splits, device="cuda")
    host = to_host_inputs(inp)
    blk = _block(moe, inp, k, T, {"fused": 2, "fused_splits": splits, "fused_uniform": uniform, "fused_chain": chain,
                                  "fused_half": half})
    run = GpuRun(blk, inp["x"])
    check_forward(run, host, k)
    assert _launches(moe, blk, inp["x"]) == 4  # router, permute, fused FFN, combine
    for _ in range(3):  # counters reset by the last CTA: repeated forwards agree bit for bit
        out2 = blk.forward(inp["x"])
        torch.cuda.synchronize()
        assert torch.equal(out2.view(torch.int16), run.out.view(torch.int16))
    blk.close()


@pytest.mark.parametrize("half", [1, 2])
@pytest.mark.parametrize("chain", [0, 1])
@pytest.mark.parametrize("T,splits", [(64, 1), (64, 2), (64, 4), (100, 2), (13, 4)])
def test_fused_bit_identical_to_two_kernels(moe, T, splits, chain, half):
    """f = 1024 (8 ffn tiles), uniform splits (tuning fused_uniform): K splits 1 / 2 / 4 fall on
    ffn-tile boundaries in both paths, so each fp32 partial is the same sum in the same order
    and the outputs match bit for bit."""
    shape = synth.MoEShape(T=T, d=512, f=1024, E=8, k=2)
    inp = synth.make_inputs(shape, 7200 + T + splits, device="cuda")
    outs = []
    for tu in ({"fused": 2, "fused_splits": splits, "fused_uniform": 1, "fused_chain": chain, "fused_half": half},
               {"fused": 1}):
        blk = _block(moe, inp, 2, T, tu, split_k=splits, flags=moe.MOE_FLAG_FORCE_SWAP)
        run = GpuRun(blk, inp["x"])
        outs.append((run.np("out_f32").copy(), run.out.clone()))
        blk.close()
    assert np.array_equal(outs[0][0].view(np.int32), outs[1][0].view(np.int32))
    assert torch.equal(outs[0][1].view(torch.int16), outs[1][1].view(torch.int16))


@pytest.mark.parametrize("n", [33, 100, 256])
def test_fused_multi_token_tiles(moe, n):
    """Every token routed to experts (0, 1) of 4 with the token tile capped at 32 rows
    (tuning swap_nb_cap): the two busy experts run ceil(n/32) token tiles each, so an h
    tile is finished only when all of its token tiles are, and two experts are empty."""
    shape = synth.MoEShape(T=n, d=256, f=512, E=4, k=2)
    inp = synth.make_inputs(shape, 7300 + n, device="cuda")
    host = to_host_inputs(inp)
    import oracle
    idx = np.tile(np.array([[0, 1]], np.int32), (n, 1))
    l = oracle.router(host["x"], host["wg"], 1)["logits"]
    li = np.take_along_axis(l, idx.astype(np.int64), 1)
    p = np.exp(li - li.max(1, keepdims=True))
    gw = (p / p.sum(1, keepdims=True)).astype(np.float32)
    blk = _block(moe, inp, 2, n, {"fused": 2, "swap_nb_cap": 32, "fused_splits": 4, "fused_half": 2})
    run = GpuRun(blk, inp["x"], routed=(torch.from_numpy(idx).cuda(), torch.from_numpy(gw).cuda()))
    check_forward(run, host, 2, routed=True)
    assert run.np("expert_counts").tolist() == [n, n, 0, 0]
    blk.close()


def test_fused_graph_replay(moe):
    """CUDA-graph capture of the fused forward, replayed 20 times: identical outputs."""
    shape = synth.MoEShape(T=64, d=512, f=1024, E=8, k=2)
    inp = synth.make_inputs(shape, 7400, device="cuda")
    blk = _block(moe, inp, 2, 64, {"fused": 2})
    ref = blk.forward(inp["x"]).clone()
    out = torch.empty_like(ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        blk.forward(inp["x"], out, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        blk.forward(inp["x"], out, stream=s)
    for _ in range(20):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
    blk.close()


@pytest.mark.parametrize("half", [1, 2])
@pytest.mark.parametrize("par,G", [("ep", 2), ("ep", 4), ("tp", 2), ("tp", 4)])
def test_fused_group(moe, par, G, half):
    """Fused FFN inside EP (receive-side expert segments) and TP (ffn slice) contexts."""
    from test_gpu_parity import _check_group_outputs, _run_group
    shape = synth.MoEShape(T=96, d=256, f=1024, E=8, k=2)
    inp = synth.make_inputs(shape, 7500 + G, device="cuda")
    host = to_host_inputs(inp)
    n_two, n_fused = [0] * G, [0] * G
    if par == "ep":
        cuts = np.linspace(0, shape.T, G + 1).astype(int)
        shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
        _run_group(moe, inp, moe.MOE_PAR_EP, G, shards, max_tokens=shape.T, tuning={"fused": 1}, launches=n_two)
        res = _run_group(moe, inp, moe.MOE_PAR_EP, G, shards, max_tokens=shape.T, tuning={"fused": 2, "fused_half": half},
                         launches=n_fused)
        _check_group_outputs(host, 2, host["x"], [r[0] for r in res], [r[1] for r in res])
    else:
        _run_group(moe, inp, moe.MOE_PAR_TP, G, [inp["x"]] * G, tuning={"fused": 1}, launches=n_two)
        res = _run_group(moe, inp, moe.MOE_PAR_TP, G, [inp["x"]] * G, tuning={"fused": 2, "fused_half": half},
                         launches=n_fused)
        for r in range(1, G):
            assert torch.equal(res[r][0].view(torch.int16), res[0][0].view(torch.int16))
        _check_group_outputs(host, 2, host["x"], [res[0][0]], [res[0][1]])
    assert all(f == t - 1 for f, t in zip(n_fused, n_two)), (n_fused, n_two)  # one launch for both GEMMs


@pytest.mark.parametrize("par,G", [("ep", 2), ("tp", 2), ("tp", 4)])
def test_fused_p2p_equals_collectives(moe, par, G):
    """Fused FFN inside EP / TP over peer memory (MOE_FLAG_P2P): bit-identical to the same
    contexts over the loopback collectives, over 3 back-to-back forwards."""
    from test_gpu_parity import _run_group
    shape = synth.MoEShape(T=64, d=256, f=1024, E=8, k=2)
    inp = synth.make_inputs(shape, 7900 + G, device="cuda")
    if par == "ep":
        cuts = np.linspace(0, shape.T, G + 1).astype(int)
        shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
        pm = moe.MOE_PAR_EP
    else:
        shards = [inp["x"]] * G
        pm = moe.MOE_PAR_TP
    tu = {"fused": 2}
    ref = _run_group(moe, inp, pm, G, shards, max_tokens=shape.T, tuning=tu)
    got = _run_group(moe, inp, pm, G, shards, max_tokens=shape.T, p2p=True, iters=3, tuning=tu)
    for r in range(G):
        assert torch.equal(ref[r][0].view(torch.int16), got[r][0].view(torch.int16)), r
        assert torch.equal(ref[r][1]["out_f32"], got[r][1]["out_f32"]), r


def test_fused_mixtral_decode(moe):
    """BASELINE configs[1]: Mixtral layer, 64-token decode, fused FFN (sampled tokens vs the
    oracle, every token's routing) and bit-identical to the two-kernel path at 4 splits
    (112 ffn tiles -> 28 per split in both)."""
    w = synth.make_weights(4096, 14336, 8, seed=42, device="cuda")
    x = synth.make_tokens(64, 4096, seed=9001, device="cuda")
    inp = dict(w, x=x)
    host = to_host_inputs(inp)
    outs = []
    for tu in ({"fused": 2, "fused_splits": 4, "fused_uniform": 1}, {"fused": 1}):
        blk = _block(moe, inp, 2, 64, tu, split_k=4)
        run = GpuRun(blk, x)
        if tu["fused"] == 2:
            check_forward(run, host, 2, tokens=[0, 1, 31, 62, 63])
        outs.append(run.np("out_f32").copy())
        blk.close()
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32))


@pytest.mark.parametrize("chain", [0, 1])
@pytest.mark.parametrize("T,residual", [(64, False), (64, True), (1, False), (37, True), (256, False)])
def test_fused_combine_bit_identical(moe, T, residual, chain):
    """In-kernel combine (tuning fused_combine=1: step a9 inside the fused FFN, one combine task
    of 256 columns x a token chunk per CTA, each waiting for every w2 tile of its slice) vs the
    combine kernel: the same sums in the same order -> bf16 out and out_f32 bit for bit, with
    and without the residual; and oracle parity."""
    shape = synth.MoEShape(T=T, d=512, f=1024, E=8, k=2)
    inp = synth.make_inputs(shape, 7600 + T, device="cuda")
    flags = moe.MOE_FLAG_RESIDUAL if residual else 0
    res = []
    for fc in (1, 0):
        blk = _block(moe, inp, 2, T, {"fused": 2, "fused_combine": fc, "fused_chain": chain}, flags=flags)
        run = GpuRun(blk, inp["x"])
        if fc == 1 and not residual:
            check_forward(run, to_host_inputs(inp), 2)
        n = _launches(moe, blk, inp["x"])
        assert n == (3 if fc == 1 else 4), n  # router, permute, fused FFN (+ combine)
        out_noaux = blk.forward(inp["x"])  # no aux: out only
        torch.cuda.synchronize()
        assert torch.equal(out_noaux.view(torch.int16), run.out.view(torch.int16))
        res.append((run.np("out_f32").copy(), run.out.clone()))
        blk.close()
    assert np.array_equal(res[0][0].view(np.int32), res[1][0].view(np.int32))
    assert torch.equal(res[0][1].view(torch.int16), res[1][1].view(torch.int16))


@pytest.mark.parametrize("par,G", [("ep", 8), ("tp", 8)])
def test_fused_half_mixtral_ranks(moe, par, G):
    """Mixtral-size EP8 / TP8 rank shapes with the fused FFN on 128-row w1/w3 tiles (the
    per-rank shapes it is meant for) vs the two-kernel path: routing and outputs bit-identical
    (uniform splits), and oracle parity on sampled tokens."""
    w = synth.make_weights(4096, 14336, 8, seed=42, device="cuda")
    x = synth.make_tokens(64, 4096, seed=9100 + G, device="cuda")
    if par == "tp":
        f_l = 14336 // G
        ws = {"wg": w["wg"], "w1": w["w1"][:, :f_l].contiguous(), "w3": w["w3"][:, :f_l].contiguous(),
              "w2": w["w2"][:, :, :f_l].contiguous()}
        k, xs = 2, x
    else:  # one expert, the rows it receives (top-1 over a single expert)
        ws = {n: w[n][:1].contiguous() for n in ("wg", "w1", "w3", "w2")}
        k, xs = 1, x[:21].contiguous()
    inp = dict(ws, x=xs)
    outs = []
    S = 2 if par == "tp" else 4  # split boundaries on whole ffn tiles in both paths (f/G = 1792: 14 tiles)
    for tu in ({"fused": 2, "fused_half": 2, "fused_uniform": 1, "fused_splits": S}, {"fused": 1}):
        blk = _block(moe, inp, k, xs.shape[0], tu, split_k=S)
        run = GpuRun(blk, xs)
        if tu["fused"] == 2:
            check_forward(run, to_host_inputs(inp), k, tokens=[0, 5, xs.shape[0] - 1])
        outs.append(run.np("out_f32").copy())
        blk.close()
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32))


def _fp8_block_inputs(shape, seed):
    """bf16 inputs + their E4M3 row-quantised weights and the oracle's exact-dequant host copy
    (tests/test_gpu_parity.py _fp8_inputs)."""
    from test_gpu_parity import _fp8_inputs
    return _fp8_inputs(shape, seed)


@pytest.mark.parametrize("T,d,f,E", [(64, 512, 1024, 8), (37, 256, 1024, 8), (64, 1024, 2560, 8), (16, 256, 512, 4)])
def test_fused_fp8(moe, T, d, f, E):
    """FP8 E4M3 weights through the fused FFN (FusedCfg FP8: kind::f8f6f4 w1/w3 tiles, block-scaled
    w2 tiles with the B scales copied into TMEM per stage): oracle parity on the exact-dequant
    weights, and bit-identity with the two-kernel FP8 path at uniform splits (same MMAs, same
    K-chunk order, same scale placement)."""
    shape = synth.MoEShape(T=T, d=d, f=f, E=E, k=2)
    inp, qs, host = _fp8_block_inputs(shape, 7700 + T + d)
    outs = []
    for tu in ({"fused": 2, "fused_uniform": 1, "fused_splits": 4}, {"fused": 1}):
        blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T,
                           flags=moe.MOE_FLAG_FP8_WEIGHTS, split_k=4, tuning=tu)
        run = GpuRun(blk, inp["x"])
        check_forward(run, host, 2)
        if tu["fused"] == 2:
            assert _launches(moe, blk, inp["x"]) == 4
            out2 = blk.forward(inp["x"])
            torch.cuda.synchronize()
            assert torch.equal(out2.view(torch.int16), run.out.view(torch.int16))
        outs.append(run.np("out_f32").copy())
        blk.close()
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32))


@pytest.mark.parametrize("T,residual", [(64, False), (37, True)])
def test_fused_fp8_combine_bit_identical(moe, T, residual):
    """FP8 fused FFN with the in-kernel combine: its w2 tiles are 128 rows, two per 256-column
    combine slice, so a slice's combine task must wait for both (arrive[m * 128 / 256]);
    bit-identical to the combine kernel after the same fused FFN, and oracle parity."""
    shape = synth.MoEShape(T=T, d=512, f=1024, E=8, k=2)
    inp, qs, host = _fp8_block_inputs(shape, 7800 + T)
    flags = moe.MOE_FLAG_FP8_WEIGHTS | (moe.MOE_FLAG_RESIDUAL if residual else 0)
    res = []
    for fc in (1, 0):
        blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T, flags=flags,
                           split_k=4, tuning={"fused": 2, "fused_combine": fc})
        run = GpuRun(blk, inp["x"])
        if not residual:
            check_forward(run, host, 2)
        assert _launches(moe, blk, inp["x"]) == (3 if fc == 1 else 4)
        res.append((run.np("out_f32").copy(), run.out.clone()))
        blk.close()
    assert np.array_equal(res[0][0].view(np.int32), res[1][0].view(np.int32))
    assert torch.equal(res[0][1].view(torch.int16), res[1][1].view(torch.int16))


@pytest.mark.parametrize("par,G", [("tp", 2), ("tp", 4)])
def test_fused_fp8_group(moe, par, G):
    """FP8 weights through the fused FFN (tuning fused=2) inside TP contexts (ffn slice, fp32
    partials reduced across ranks; loopback transport): one launch replaces the two FP8 GEMMs,
    oracle parity on the exact-dequant weights, every rank with the same output, 3 back-to-back
    forwards. (EP capacity-mode ranks size their token tile for the capacity, above the FP8
    fused kernel's 32 rows, and keep the two FP8 kernels.)"""
    from test_gpu_parity import _check_group_outputs, _run_group
    shape = synth.MoEShape(T=64, d=512, f=1024, E=8, k=2)
    inp, qs, host = _fp8_block_inputs(shape, 7950 + G)
    inp8 = dict(inp, w1=qs["w1"], w3=qs["w3"], w2=qs["w2"])
    if par == "ep":
        cuts = np.linspace(0, shape.T, G + 1).astype(int)
        shards, pm, mt = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)], moe.MOE_PAR_EP, shape.T
    else:
        shards, pm, mt = [inp["x"]] * G, moe.MOE_PAR_TP, None
    n_two = [0] * G
    _run_group(moe, inp8, pm, G, shards, flags=moe.MOE_FLAG_FP8_WEIGHTS, max_tokens=mt, tuning={"fused": 1},
               launches=n_two)
    n_fused = [0] * G
    res = _run_group(moe, inp8, pm, G, shards, flags=moe.MOE_FLAG_FP8_WEIGHTS, max_tokens=mt, iters=3,
                     tuning={"fused": 2}, launches=n_fused)
    assert all(f == t - 1 for f, t in zip(n_fused, n_two)), (n_fused, n_two)  # one launch for both GEMMs
    if par == "ep":
        _check_group_outputs(host, 2, host["x"], [r[0] for r in res], [r[1] for r in res])
    else:
        for r in range(1, G):
            assert torch.equal(res[r][0].view(torch.int16), res[0][0].view(torch.int16))
        _check_group_outputs(host, 2, host["x"], [res[0][0]], [res[0][1]])


def test_fused_fp8_mixtral(moe):
    """FP8 Mixtral-size 64-token decode: the fused FFN (uniform 4 splits) bit-identical to the
    two-kernel FP8 path, and oracle parity on sampled tokens (exact-dequant weights); the default
    tapered splits against the oracle too (tests/test_gpu_parity.py test_fp8_mixtral_decode
    checks every token of the default path)."""
    w = synth.make_weights(4096, 14336, 8, seed=42, device="cuda")
    x = synth.make_tokens(64, 4096, seed=9200, device="cuda")
    qs = {n: synth.quantize_fp8_rows(w[n]) for n in ("w1", "w3", "w2")}
    host = {n: synth.dequantize_fp8_rows(*qs[n]).cpu().numpy() for n in qs}
    host["x"] = x.float().cpu().numpy()
    host["wg"] = w["wg"].float().cpu().numpy()
    outs = []
    for tu in ({"fused": 2, "fused_uniform": 1, "fused_splits": 4}, {"fused": 1}, {"fused": 2}):
        blk = moe.MoEBlock(w["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=64,
                           flags=moe.MOE_FLAG_FP8_WEIGHTS, split_k=4, tuning=tu)
        run = GpuRun(blk, x)
        check_forward(run, host, 2, tokens=[0, 1, 33, 62, 63])
        outs.append(run.np("out_f32").copy())
        blk.close()
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32))
