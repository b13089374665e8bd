"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (R4/R8, BASELINE.json north_star): routing bit-exact outside
the 1e-3 margin band; permutation integers exact; out_f32 within 2e-2 of the
oracle normalised by the row RMS; the stored bf16 output exactly RNE(out_f32);
and, at C1/C2 sizes, the literal bf16 output within 2e-2 too.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from parity import GpuRun, check_forward, to_host_inputs

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def moe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2408_00008_b200 as m
    return m


def _block(moe, inp, k, max_tokens, flags=0, split_k=0, tuning=None):
    return moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=k, max_tokens=max_tokens,
                        flags=flags, split_k=split_k, tuning=tuning)


def _inputs(shape, seed, device="cuda"):
    return synth.make_inputs(shape, seed, device=device)


# 0x80 = MOE_FLAG_GATHER: token rows gathered by the w1/w3 GEMM (tile::gather4), no permuted copy
MODES = {"auto": 0, "swap": 0x2, "tiled": 0x4, "tiled1cta": 0x4 | 0x10,
         "swap_gather": 0x2 | 0x80, "tiled_gather": 0x4 | 0x80, "tiled1cta_gather": 0x4 | 0x10 | 0x80}


# ---------------------------------------------------------------- worked example
def test_worked_example_on_gpu(moe):
    """Tie-break + closed form (tests/golden/worked_example.json), zero-padded to C1 shapes."""
    g = json.load(open(os.path.join(GOLDEN, "worked_example.json")))
    d, f, E = 64, 128, 4
    x = torch.zeros(16, d)
    x[0, :2] = torch.tensor(g["x"][0])
    wg = torch.zeros(E, d)
    wg[:, :2] = torch.tensor(g["wg"])
    w1 = torch.zeros(E, f, d)
    w3 = torch.zeros(E, f, d)
    w2 = torch.zeros(E, d, f)
    for e in range(E):
        w1[e, 0, :2] = torch.tensor(g["w1"][e][0])
        w3[e, 0, :2] = torch.tensor(g["w3"][e][0])
        w2[e, :2, 0] = torch.tensor([r[0] for r in g["w2"][e]])
    inp = {n: v.to(torch.bfloat16).cuda() for n, v in dict(x=x, wg=wg, w1=w1, w3=w3, w2=w2).items()}
    for flags in MODES.values():
        blk = _block(moe, inp, 2, 16, flags)
        run = GpuRun(blk, inp["x"])
        assert run.np("topk_idx")[0].tolist() == g["expect_idx"]
        np.testing.assert_allclose(run.np("topk_w")[0], g["expect_w"], rtol=0, atol=1e-6)
        of = run.np("out_f32")
        assert abs(of[0, 0] - g["gpu_expect"]["out_f32_approx"]) < 2e-6
        assert run.np("out")[0, 0] == g["gpu_expect"]["out_bf16"]
        assert np.all(of[0, 1:] == 0) and np.all(of[1:] == 0)
        assert abs(of[0, 0] - g["expect_y"][0]) / abs(g["expect_y"][0]) < 2e-2
        blk.close()


# ---------------------------------------------------------------- C1 (BASELINE configs[0])
@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("seed", list(range(20)))
def test_c1_parity(moe, seed, mode):
    inp = _inputs(synth.TINY, seed)
    blk = _block(moe, inp, 2, synth.TINY.T, MODES[mode])
    run = GpuRun(blk, inp["x"])
    check_forward(run, to_host_inputs(inp), 2)
    blk.close()


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("T,d,f,E,k", [(1, 64, 128, 4, 2), (7, 64, 128, 4, 2), (63, 64, 128, 8, 2),
                                       (65, 128, 256, 8, 2), (129, 64, 128, 4, 2), (300, 128, 256, 8, 2),
                                       (200, 64, 128, 1, 1), (77, 64, 128, 8, 1), (100, 64, 384, 2, 2),
                                       (333, 320, 256, 6, 2)])
def test_ragged_shapes(moe, T, d, f, E, k, mode):
    """Ragged token counts, odd tile tails (d=320 -> 2.5 N-tiles), E=1 k=1 (dense SwiGLU)."""
    shape = synth.MoEShape(T=T, d=d, f=f, E=E, k=k)
    inp = _inputs(shape, 1000 + T)
    blk = _block(moe, inp, k, T + 5, MODES[mode])
    run = GpuRun(blk, inp["x"])
    check_forward(run, to_host_inputs(inp), k)
    blk.close()


@pytest.mark.parametrize("mode", ["auto", "swap", "tiled"])
@pytest.mark.parametrize("T,E,k", [(1, 16, 2), (37, 16, 2), (200, 16, 2), (64, 32, 2), (333, 32, 2), (90, 32, 1),
                                   (129, 12, 2), (50, 9, 2)])
def test_many_experts(moe, T, E, k, mode):
    """8 < E <= 32: the CUDA-core routers moe_router_kernel<16,2> / <32,2> (the
    tensor-core router covers E <= 8), 16- and 32-key histograms and scans, and grouped
    GEMMs over up to 32 expert segments (some empty at small T)."""
    shape = synth.MoEShape(T=T, d=128, f=256, E=E, k=k)
    inp = _inputs(shape, 3000 + 7 * T + E)
    blk = _block(moe, inp, k, T, MODES[mode])
    check_forward(GpuRun(blk, inp["x"]), to_host_inputs(inp), k)
    blk.close()


@pytest.mark.parametrize("G", [1, 2])
def test_ep_many_experts(moe, G):
    """EP with E = 32 (16 local experts per rank at G = 2, 32 at G = 1): the receive-side
    routing histogram spans E_local keys over G*max_tokens*k slots (the workspace sizing
    of ADVICE r01: EP-like contexts at ep_world 1 included)."""
    shape = synth.MoEShape(T=64, d=128, f=256, E=32, k=2)
    inp = _inputs(shape, 3100 + G)
    host = to_host_inputs(inp)
    cuts = np.linspace(0, shape.T, G + 1).astype(int)
    shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
    res = _run_group(moe, inp, moe.MOE_PAR_EP, G, shards, max_tokens=shape.T)
    _check_group_outputs(host, 2, host["x"], [r[0] for r in res], [r[1] for r in res])


@pytest.mark.parametrize("mode", ["swap", "tiled", "tiled1cta"])
def test_multi_tile_mid_size(moe, mode):
    """Several M/N/K tiles per expert plus ragged tails (d=512, f=1024, E=8, T=1000)."""
    shape = synth.MoEShape(T=1000, d=512, f=1024, E=8, k=2)
    inp = _inputs(shape, 7)
    blk = _block(moe, inp, 2, 1000, MODES[mode])
    run = GpuRun(blk, inp["x"])
    check_forward(run, to_host_inputs(inp), 2)
    blk.close()


@pytest.mark.parametrize("flags", [0, 0x10])
def test_mixed_gemm_paths(moe, flags):
    """Per-GEMM path choice: ~150 rows per expert with the w2 threshold at 40 runs the
    w1/w3 GEMM swap-AB and the w2 GEMM on tokens-as-M tiles (CTA pairs, or single
    CTAs with MOE_FLAG_NO_PAIR) -- the h buffer hand-off between the two families."""
    shape = synth.MoEShape(T=600, d=512, f=1024, E=8, k=2)
    inp = _inputs(shape, 17)
    blk = _block(moe, inp, 2, 600, flags, tuning={"g2_swap_rows": 40})  # w2 GEMM on tiles from 40 rows/expert
    run = GpuRun(blk, inp["x"])
    check_forward(run, to_host_inputs(inp), 2)
    blk.close()


@pytest.mark.parametrize("T,d,f,E,k", [(16, 64, 128, 4, 2), (333, 320, 256, 6, 2), (1000, 512, 1024, 8, 2),
                                       (700, 768, 384, 4, 2), (129, 64, 128, 4, 2)])
def test_pair_wide_tiles(moe, T, d, f, E, k):
    """CTA-pair GEMMs with 256 x 512 tiles (tuning pair_nblk=2, single-buffered TMEM,
    block-0-first catch-up) vs 256 x 256 tiles (NBLK=1, two accumulators): both against
    the oracle, and bit-identical to each other (the same MMAs accumulate each 256-column
    block in the same K order). Odd block counts (f/128 = 3, ceil(d/256) = 3) leave a
    half-empty last tile."""
    shape = synth.MoEShape(T=T, d=d, f=f, E=E, k=k)
    inp = _inputs(shape, 4000 + T)
    outs = []
    for nblk in (1, 2):
        blk = _block(moe, inp, k, T, moe.MOE_FLAG_FORCE_TILED, tuning={"pair_nblk": nblk})
        run = GpuRun(blk, inp["x"])
        check_forward(run, to_host_inputs(inp), k)
        outs.append(run.np("out_f32").copy())
        out2 = blk.forward(inp["x"])  # second forward: barrier phases carried across calls
        torch.cuda.synchronize()
        assert torch.equal(out2.view(torch.int16), run.out.view(torch.int16))
        blk.close()
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32))


@pytest.mark.parametrize("T,d,f,E,k,split_k", [
    (300, 256, 512, 8, 2, 0),     # ~75 rows / expert: token tile 128 on the pair (64 rows per CTA)
    (575, 512, 1024, 8, 2, 0),    # the stack batch: token tile 192 (96 per CTA)
    (1000, 512, 1024, 8, 2, 0),   # ~250 rows / expert: tile 256, busy experts run a 2nd token tile
    (400, 320, 384, 4, 2, 3),     # f/128 odd: w1/w3 on single CTAs, w2 pairs over d = 320 (a padding tile), 3 K splits
    (130, 256, 512, 8, 1, 0),     # top-1, small experts: N = 32 tiles with a few valid tokens
    (700, 768, 256, 6, 2, 2)])
def test_swap_pair(moe, T, d, f, E, k, split_k):
    """Swap-AB GEMMs on CTA pairs (moe_gemm_swap_pair_kernel, tuning swap_pair): each CTA
    streams its own weight tile and stages half of the token tile, the pair's M = 256 MMA
    fills both CTAs' TMEM. Oracle parity with the pair kernels forced (2) and off (1),
    and the two runs bit-identical (same MMAs per output element, same K order)."""
    shape = synth.MoEShape(T=T, d=d, f=f, E=E, k=k)
    inp = _inputs(shape, 6100 + T + d)
    host = to_host_inputs(inp)
    outs = []
    for mode in (2, 1):
        blk = _block(moe, inp, k, T, moe.MOE_FLAG_FORCE_SWAP, split_k=split_k, tuning={"swap_pair": mode})
        run = GpuRun(blk, inp["x"])
        check_forward(run, host, k)
        outs.append(run.np("out_f32").copy())
        out2 = blk.forward(inp["x"])  # second forward: barrier phases carried across calls
        torch.cuda.synchronize()
        assert torch.equal(out2.view(torch.int16), run.out.view(torch.int16))
        blk.close()
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32))


@pytest.mark.parametrize("n", [129, 256, 300])
def test_swap_pair_pathological(moe, n):
    """Forced routing of every token to experts (0, 1) of 4 with the pair kernels: the
    token tile is sized for the expected n/2 rows per expert, so each of the two busy
    experts runs two token tiles (129 rows: a 1-token tail tile)."""
    shape = synth.MoEShape(T=n, d=256, f=512, E=4, k=2)
    inp = _inputs(shape, 6200 + n)
    host = to_host_inputs(inp)
    idx = np.tile(np.array([[0, 1]], np.int32), (n, 1))
    gw = _forced_gates(host, idx)
    blk = _block(moe, inp, 2, n, moe.MOE_FLAG_FORCE_SWAP, tuning={"swap_pair": 2})
    run = GpuRun(blk, inp["x"], routed=(torch.from_numpy(idx).cuda(), torch.from_numpy(gw).cuda()))
    check_forward(run, host, 2, routed=True)
    assert run.np("expert_counts").tolist() == [n, n, 0, 0]
    blk.close()


@pytest.mark.parametrize("fp8", [False, True])
@pytest.mark.parametrize("T,d,f,E", [(64, 512, 1024, 8), (300, 256, 512, 8), (100, 256, 512, 2)])
def test_swap_nb_cap(moe, T, d, f, E, fp8):
    """Swap-AB token tile capped at 32 (tuning swap_nb_cap): experts with more rows run
    several token tiles (device-side tile count), bf16 and FP8 weights."""
    shape = synth.MoEShape(T=T, d=d, f=f, E=E, k=2)
    tu = {"swap_nb_cap": 32}
    if fp8:
        inp, qs, host = _fp8_inputs(shape, 5000 + T)
        blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T,
                           flags=moe.MOE_FLAG_FP8_WEIGHTS, tuning=tu)
    else:
        inp = _inputs(shape, 5000 + T)
        host = to_host_inputs(inp)
        blk = _block(moe, inp, 2, T, moe.MOE_FLAG_FORCE_SWAP, tuning=tu)
    run = GpuRun(blk, inp["x"])
    check_forward(run, host, 2)
    blk.close()


@pytest.mark.parametrize("split_k", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("T", [40, 200])
def test_split_k(moe, T, split_k):
    """Decode w2 GEMM with an explicit K split (moe_config.split_k; fixed-order fp32
    partials summed by the combine), incl. uneven splits of 1024/64 = 16 K blocks."""
    shape = synth.MoEShape(T=T, d=256, f=1024, E=8, k=2)
    inp = _inputs(shape, 29)
    blk = _block(moe, inp, 2, T, 0x2, split_k=split_k)
    run = GpuRun(blk, inp["x"])
    check_forward(run, to_host_inputs(inp), 2)
    blk.close()


def _forced_gates(host, idx):
    l = oracle.router(host["x"], host["wg"], 1)["logits"]
    li = np.take_along_axis(l, idx.astype(np.int64), 1)
    p = np.exp(li - li.max(1, keepdims=True))
    return (p / p.sum(1, keepdims=True)).astype(np.float32)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("n", [127, 128, 129, 256])
def test_pathological_routing(moe, n, mode):
    """Forced routing (oracle step 8): every token to experts (0, 1): counts 127/128/129/256, others empty."""
    shape = synth.MoEShape(T=n, d=128, f=256, E=4, k=2)
    inp = _inputs(shape, n)
    host = to_host_inputs(inp)
    idx = np.tile(np.array([[1, 0]], np.int32), (n, 1))
    gw = _forced_gates(host, idx)
    blk = _block(moe, inp, 2, n, MODES[mode])
    run = GpuRun(blk, inp["x"], routed=(torch.from_numpy(idx).cuda(), torch.from_numpy(gw).cuda()))
    np.testing.assert_array_equal(run.np("topk_idx"), idx)
    check_forward(run, host, 2, routed=True)
    assert run.np("expert_counts").tolist() == [n, n, 0, 0]
    blk.close()


@pytest.mark.parametrize("T", [16, 48, 128])
def test_speculative_prefetch_wrong_guess(moe, T):
    """Decode speculative L2 prefetch (16 <= T <= 128, bf16 swap path): the w1/w3 GEMM
    launches before routing completes and guesses one token tile per expert. Forced
    routing to experts (3, 6) of 8 leaves six experts empty, so every guess is wrong;
    the GEMM must still read counts only after its wait (oracle parity)."""
    shape = synth.MoEShape(T=T, d=256, f=512, E=8, k=2)
    inp = _inputs(shape, 200 + T)
    host = to_host_inputs(inp)
    idx = np.tile(np.array([[6, 3]], np.int32), (T, 1))
    gw = _forced_gates(host, idx)
    blk = _block(moe, inp, 2, T, MODES["swap"])
    run = GpuRun(blk, inp["x"], routed=(torch.from_numpy(idx).cuda(), torch.from_numpy(gw).cuda()))
    check_forward(run, host, 2, routed=True)
    assert run.np("expert_counts").tolist() == [0, 0, 0, T, 0, 0, T, 0]
    blk.close()
    run = GpuRun(_block(moe, inp, 2, T, MODES["swap"]), inp["x"])  # router path, same shapes
    check_forward(run, host, 2)


def test_t_zero_and_determinism(moe):
    inp = _inputs(synth.TINY, 3)
    blk = _block(moe, inp, 2, 16)
    out = torch.full((1, 64), 7.0, dtype=torch.bfloat16, device="cuda")
    moe.moe_forward(blk.ctx, inp["x"], 0, blk.router_w, blk.w13, blk.w2, out)
    torch.cuda.synchronize()
    assert torch.all(out == 7.0)  # T = 0 enqueues nothing
    a = blk.forward(inp["x"]).clone()
    b = blk.forward(inp["x"]).clone()
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))  # bit-identical reruns
    blk.close()


def test_invalid_arguments_enqueue_nothing(moe):
    inp = _inputs(synth.TINY, 4)
    blk = _block(moe, inp, 2, 16)
    out = torch.zeros(16, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(moe.MoEError) as ei:
        moe.moe_forward(blk.ctx, inp["x"], 17, blk.router_w, blk.w13, blk.w2, out)  # T > max_tokens
    assert ei.value.status == moe.MOE_ERR_INVALID
    with pytest.raises(moe.MoEError):
        moe.moe_forward(blk.ctx, inp["x"][:, 1:], 16, blk.router_w, blk.w13, blk.w2, out)  # misaligned
    torch.cuda.synchronize()
    assert torch.all(out == 0)
    blk.close()


def test_residual_flag(moe):
    inp = _inputs(synth.TINY, 5)
    blk = _block(moe, inp, 2, 16, flags=moe.MOE_FLAG_RESIDUAL)
    run = GpuRun(blk, inp["x"])
    host = to_host_inputs(inp)
    y = oracle.moe_forward(host["x"], host["wg"], host["w1"], host["w3"], host["w2"], 2,
                           forced_idx=run.np("topk_idx"), residual=True)
    from parity import rel_err
    assert rel_err(run.np("out_f32"), y).max() <= 2e-2
    blk.close()


def test_host_entry_point(moe):
    """moe_forward_host (the e2e call bench.py times) == moe_forward."""
    inp = _inputs(synth.TINY, 6)
    blk = _block(moe, inp, 2, 16)
    ref = blk.forward(inp["x"]).cpu()
    xh = inp["x"].cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()      # pinned: the combine kernel writes it directly
    moe.moe_forward_host(blk.ctx, xh, 16, blk.router_w, blk.w13, blk.w2, oh)
    torch.cuda.synchronize()
    assert torch.equal(oh.view(torch.int16), ref.view(torch.int16))
    op = torch.zeros_like(inp["x"].cpu())       # pageable: staging buffer + copy
    xp = inp["x"].cpu()
    for _ in range(3):                          # back-to-back calls rotate the two input slots
        moe.moe_forward_host(blk.ctx, xp, 16, blk.router_w, blk.w13, blk.w2, op)
        moe.moe_forward_host(blk.ctx, xh, 16, blk.router_w, blk.w13, blk.w2, oh)
    torch.cuda.synchronize()
    assert torch.equal(op.view(torch.int16), ref.view(torch.int16))
    assert torch.equal(oh.view(torch.int16), ref.view(torch.int16))
    blk.close()


@pytest.mark.parametrize("residual", [False, True])
def test_host_entry_point_fused_combine(moe, residual):
    """moe_forward_host into pinned (mapped) host memory with the fused FFN: the auto mode of
    tuning fused_combine runs step a9 inside the fused kernel there (one launch fewer, each
    output slice crossing the host link as its w2 tiles finish) -- bit-identical to the device
    forward with the combine kernel; pageable output keeps the combine kernel."""
    shape = synth.MoEShape(T=64, d=512, f=1024, E=8, k=2)
    inp = synth.make_inputs(shape, 8100 + residual, device="cuda")
    flags = moe.MOE_FLAG_RESIDUAL if residual else 0
    blk = _block(moe, inp, 2, 64, flags=flags, tuning={"fused": 2})
    n0 = moe.moe_launch_count(blk.ctx)
    ref = blk.forward(inp["x"]).cpu()
    torch.cuda.synchronize()
    n_dev = moe.moe_launch_count(blk.ctx) - n0
    xh = inp["x"].cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    for _ in range(3):
        n0 = moe.moe_launch_count(blk.ctx)
        moe.moe_forward_host(blk.ctx, xh, 64, blk.router_w, blk.w13, blk.w2, oh)
        torch.cuda.synchronize()
        n_host = moe.moe_launch_count(blk.ctx) - n0
        assert torch.equal(oh.view(torch.int16), ref.view(torch.int16))
    assert n_dev == 4 and n_host == 3, (n_dev, n_host)  # router, permute, fused FFN (+ combine kernel)
    op = torch.zeros_like(inp["x"].cpu())  # pageable: staging buffer + copy, combine kernel
    n0 = moe.moe_launch_count(blk.ctx)
    moe.moe_forward_host(blk.ctx, inp["x"].cpu(), 64, blk.router_w, blk.w13, blk.w2, op)
    torch.cuda.synchronize()
    assert moe.moe_launch_count(blk.ctx) - n0 == 4
    assert torch.equal(op.view(torch.int16), ref.view(torch.int16))
    blk.close()


# ---------------------------------------------------------------- full size (BASELINE configs[1], [2])
@pytest.fixture(scope="module")
def mixtral_weights():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = synth.make_weights(4096, 14336, 8, seed=42, device="cuda")
    host = {n: synth.bf16_bits(v) for n, v in w.items()}
    return w, host


def test_c2_host_entry_point(moe, mixtral_weights):
    """The e2e call bench.py times (moe_forward_host, pinned host buffers) at Mixtral size in the
    bench's default configuration (fused FFN; in-kernel combine for the mapped host output):
    bit-identical to the device-resident forward over back-to-back calls."""
    w, _ = mixtral_weights
    x = synth.make_tokens(64, 4096, seed=8200, device="cuda")
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=2, max_tokens=64)
    ref = blk.forward(x).cpu()
    xh = x.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    for _ in range(4):
        oh.zero_()
        moe.moe_forward_host(blk.ctx, xh, 64, blk.router_w, blk.w13, blk.w2, oh)
        torch.cuda.synchronize()
        assert torch.equal(oh.view(torch.int16), ref.view(torch.int16))
    blk.close()


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])  # C2 x 5 parity seeds
def test_c2_decode_full(moe, mixtral_weights, seed):
    """64-token decode at Mixtral size, all tokens checked against the oracle."""
    w, host = mixtral_weights
    x = synth.make_tokens(64, 4096, seed=100 + seed, device="cuda")
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=2, max_tokens=64)
    run = GpuRun(blk, x)
    h = dict(host, x=synth.bf16_bits(x))
    st = check_forward(run, h, 2)
    print("C2", seed, st)
    blk.close()


@pytest.mark.parametrize("T", [64, 575])
def test_skewed_routing(moe, mixtral_weights, T):
    """SURVEY 8(d) optional skew variant: tokens with a 4:1 popularity of expert 0
    (synth.make_tokens_skewed) at Mixtral size, decode (T=64) and the stack batch (T=575,
    where the popular expert overflows the statistical 192-row token tile and runs
    several token tiles): routing exact, every output vs the oracle."""
    w, host = mixtral_weights
    x = synth.make_tokens_skewed(T, 4096, w["wg"], seed=400 + T, device="cuda")
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=2, max_tokens=T)
    run = GpuRun(blk, x)
    counts = run.np("expert_counts")
    assert counts[0] > 2.5 * np.mean(counts[1:]), counts
    toks = np.arange(T) if T <= 64 else np.unique(np.concatenate([[0, T - 1], np.random.default_rng(T).choice(T, 48, replace=False)]))
    st = check_forward(run, dict(host, x=synth.bf16_bits(x)), 2, tokens=toks, literal_bf16=T <= 64)
    print("skewed", T, counts.tolist(), st)
    blk.close()


def test_c2_speculative_prefetch_bit_identical(moe, mixtral_weights):
    """The speculative L2 prefetch (tuning spec_l2) changes only timing: 64-token decode
    outputs are bit-identical with it off and at two depths."""
    w, _ = mixtral_weights
    x = synth.make_tokens(64, 4096, seed=321, device="cuda")
    outs = []
    for v in (-1, 16, 64):
        blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=2, max_tokens=64, tuning={"spec_l2": v})
        for _ in range(2):
            o = blk.forward(x)
        torch.cuda.synchronize()
        outs.append(o.clone())
        blk.close()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    assert torch.equal(outs[0].view(torch.int16), outs[2].view(torch.int16))


def stratified_tokens(run, rng, tile=256):
    """Tokens whose permuted rows cover every expert segment of a GPU run: for each local
    expert its first row, its last row (the ragged tail) and one random row inside every
    `tile`-row block of the segment (the CTA-pair M tile is 256 rows), mapped back to
    their tokens through the permutation `pos`."""
    pos = run.np("pos")
    counts, offs = run.np("expert_counts"), run.np("expert_offsets")
    row_tok = {}
    for t, rows in enumerate(pos):
        for r in rows:
            if r >= 0:
                row_tok[int(r)] = t
    rows = []
    for e, c in enumerate(counts):
        if c <= 0:
            continue
        o = int(offs[e])
        rows += [o, o + int(c) - 1]
        for b0 in range(0, int(c), tile):
            rows.append(o + b0 + int(rng.integers(0, min(tile, int(c) - b0))))
    return np.unique([row_tok[r] for r in rows])


@pytest.mark.parametrize("seed", [0, 1])  # C3 x 2 parity seeds
def test_c3_prefill_full(moe, mixtral_weights, seed):
    """32k-token prefill: full routing + permutation exact; outputs element by element on
    a stratified token set that touches every 256-row tile of every expert segment (its
    first and last rows included) plus fixed and random tokens."""
    w, host = mixtral_weights
    T = 32768
    x = synth.make_tokens(T, 4096, seed=200 + seed, device="cuda")
    blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=2, max_tokens=T)
    run = GpuRun(blk, x)
    h = dict(host, x=synth.bf16_bits(x))
    rng = np.random.default_rng(seed)
    strat = stratified_tokens(run, rng)
    toks = np.unique(np.concatenate([[0, 1, 63, 64, T - 1], rng.choice(T, 27, replace=False), strat]))
    assert len(strat) >= 200, len(strat)  # ~8 experts x (32 tiles + 2 ends)
    st = check_forward(run, h, 2, tokens=toks, literal_bf16=False)
    st["tokens_checked"] = int(len(toks))
    print("C3", st)
    # determinism at full size
    out2 = blk.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(out2.view(torch.int16), run.out.view(torch.int16))
    blk.close()


@pytest.mark.parametrize("T,flags", [(64, 0), (300, 0x2), (4096, 0), (4096, 0x10), (1000, 0x4 | 0x10)])
def test_gather_equals_copy(moe, mixtral_weights, T, flags):
    """The tile::gather4 token fetch and the materialised permuted copy feed the same
    bytes to the same MMAs: outputs must agree bit for bit (Mixtral size)."""
    w, _ = mixtral_weights
    x = synth.make_tokens(T, 4096, seed=300 + T, device="cuda")
    outs = []
    for extra in (0, moe.MOE_FLAG_GATHER):
        # two-kernel GEMM path for both (the fused decode FFN has no gather variant)
        blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], top_k=2, max_tokens=T, flags=flags | extra,
                           tuning={"fused": 1})
        outs.append(blk.forward(x).clone())
        torch.cuda.synchronize()
        blk.close()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))


# ---------------------------------------------------------------- EP / TP device path (loopback transport)
def _run_group(moe, inp, par, G, shards, k=2, flags=0, max_tokens=None, p2p=False, iters=1, tuning=None, launches=None):
    """G contexts on one GPU, each driven by its own thread (and stream), exchanging
    through the loopback transport, or through peer memory (p2p: MOE_FLAG_P2P, the
    handles of the G regions connected in-process). shards[r] = token tensor of rank
    r. Returns per-rank (out, aux) of the last of `iters` forwards (all must agree);
    launches (a list of G), when given, receives each rank's kernel launches of that forward."""
    import threading
    if p2p:
        grp, comms, flags = None, [None] * G, flags | moe.MOE_FLAG_P2P
    else:
        grp = moe.moe_loopback_comm_create(G)
        comms = [moe.moe_loopback_comm_rank(grp, r) for r in range(G)]
    mt = max_tokens or max(1, max(s.shape[0] for s in shards))
    blocks = [moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=k, max_tokens=mt, par=par,
                           world_size=G, rank=r, nccl_comm=comms[r], flags=flags, tuning=tuning) for r in range(G)]
    if p2p:
        handles = [b.p2p_handle() for b in blocks]
        for b in blocks:
            b.p2p_connect(handles)
    torch.cuda.synchronize()
    E, d = inp["wg"].shape
    res = [None] * G
    errs = []
    streams = [torch.cuda.Stream() for _ in range(G)]  # consecutive pool streams: distinct hardware queues

    def work(r):
        try:
            st = streams[r]
            x = shards[r]
            T = x.shape[0]
            aux = {"topk_idx": torch.empty(max(T, 1), k, dtype=torch.int32, device="cuda"),
                   "pos": torch.empty(max(T, 1), k, dtype=torch.int32, device="cuda"),
                   "out_f32": torch.empty(max(T, 1), d, dtype=torch.float32, device="cuda")}
            out = torch.empty(max(T, 1), d, dtype=torch.bfloat16, device="cuda")
            first = None
            for it in range(iters):
                n0 = moe.moe_launch_count(blocks[r].ctx)
                with torch.cuda.stream(st):
                    moe.moe_forward(blocks[r].ctx, x if T else out, T, blocks[r].router_w, blocks[r].w13,
                                    blocks[r].w2, out, aux, st, blocks[r].s13, blocks[r].s2)
                st.synchronize()
                if launches is not None:
                    launches[r] = moe.moe_launch_count(blocks[r].ctx) - n0
                res[r] = (out[:T].clone(), {n: v[:T].clone() for n, v in aux.items()})
                if first is None:
                    first = res[r][0]
                elif not torch.equal(first.view(torch.int16), res[r][0].view(torch.int16)):
                    raise AssertionError(f"rank {r}: iteration {it} differs from iteration 0")
        except Exception as ex:  # pragma: no cover - surfaced below
            errs.append((r, ex))

    ths = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    for b in blocks:
        b.close()
    if grp is not None:
        for cm in comms:
            moe.moe_loopback_comm_destroy(cm)
        moe.moe_loopback_comm_destroy(grp)
    assert not errs, errs
    return res


def _check_group_outputs(host, k, x_rows, outs, auxs):
    """Concatenated per-rank outputs vs the single-GPU oracle on the global batch."""
    from parity import rel_err
    idx = np.concatenate([a["topk_idx"].cpu().numpy() for a in auxs]) if auxs else None
    h = dict(host, x=x_rows)
    ref = oracle.router(h["x"], h["wg"], k)
    from parity import routing_check
    excl, bad = routing_check(idx, ref)
    assert not bad, bad
    y = oracle.moe_forward(h["x"], h["wg"], h["w1"], h["w3"], h["w2"], k, forced_idx=idx)
    of32 = np.concatenate([a["out_f32"].cpu().numpy() for a in auxs])
    ob16 = np.concatenate([o.float().cpu().numpy() for o in outs]).astype(np.float64)
    e32, e16 = rel_err(of32, y).max(), rel_err(ob16, y).max()
    assert e32 <= 2e-2 and e16 <= 2e-2, (e32, e16)
    rne = torch.from_numpy(of32).to(torch.bfloat16).float().numpy().astype(np.float64)
    np.testing.assert_array_equal(ob16, rne)
    return e32, e16


@pytest.mark.parametrize("par,G", [("ep", 2), ("ep", 4), ("tp", 2), ("ep_exact", 2)])
def test_fp8_group(moe, par, G):
    """FP8 weights under expert / tensor parallelism (loopback transport): each rank packs
    its expert range / ffn slice of the E4M3 weights and scales; the receive-side permute
    splits tokens into the two E4M3 terms of the kind::f8f6f4 w1/w3 GEMM."""
    shape = synth.MoEShape(T=96, d=256, f=512, E=8, k=2)
    inp, qs, host = _fp8_inputs(shape, 70 + G)
    inp8 = dict(inp, w1=qs["w1"], w3=qs["w3"], w2=qs["w2"])
    flags = moe.MOE_FLAG_FP8_WEIGHTS | (moe.MOE_FLAG_EP_EXACT if par == "ep_exact" else 0)
    if par == "tp":
        res = _run_group(moe, inp8, moe.MOE_PAR_TP, G, [inp["x"]] * G, flags=flags)
        outs, auxs = [res[0][0]], [res[0][1]]
    else:
        cuts = np.linspace(0, shape.T, G + 1).astype(int)
        shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
        res = _run_group(moe, inp8, moe.MOE_PAR_EP, G, shards, flags=flags, max_tokens=shape.T)
        outs, auxs = [r[0] for r in res], [r[1] for r in res]
    _check_group_outputs(host, 2, host["x"], outs, auxs)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["swap", "tiled", "exact"])
def test_ep_loopback(moe, G, mode):
    """Expert parallel (one process per GPU emulated by G threads on one device):
    tokens sharded unevenly across ranks (incl. a rank with no tokens)."""
    shape = synth.MoEShape(T=96, d=256, f=512, E=8, k=2)
    inp = _inputs(shape, 50 + G)
    host = to_host_inputs(inp)
    cuts = np.linspace(0, shape.T, G + 1).astype(int)
    if G >= 2:
        cuts[1] = 0  # rank 0 gets no tokens, rank 1 gets the first share
    shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
    flags = moe.MOE_FLAG_EP_EXACT if mode == "exact" else MODES[mode]
    res = _run_group(moe, inp, moe.MOE_PAR_EP, G, shards, flags=flags, max_tokens=shape.T)
    outs = [r[0] for r in res]
    auxs = [r[1] for r in res]
    _check_group_outputs(host, 2, host["x"], outs, auxs)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("par", ["ep", "tp"])
@pytest.mark.parametrize("mode", ["swap", "tiled"])
def test_p2p_equals_collectives(moe, G, par, mode):
    """Peer-memory transport (MOE_FLAG_P2P): the same slots and the same summation
    order as the collective path, so outputs must match it bit for bit (and the
    oracle within tolerance), over 3 back-to-back forwards (counter epochs, buffer
    reuse), with a rank that has no tokens (EP)."""
    if par == "tp" and G == 8:
        pytest.skip("f=512 / 8 < 128")
    shape = synth.MoEShape(T=96, d=256, f=512, E=8, k=2)
    inp = _inputs(shape, 70 + G)
    host = to_host_inputs(inp)
    if par == "ep":
        cuts = np.linspace(0, shape.T, G + 1).astype(int)
        if G >= 2:
            cuts[1] = 0
        shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
        pm = moe.MOE_PAR_EP
    else:
        shards = [inp["x"]] * G
        pm = moe.MOE_PAR_TP
    ref = _run_group(moe, inp, pm, G, shards, flags=MODES[mode], max_tokens=shape.T)
    got = _run_group(moe, inp, pm, G, shards, flags=MODES[mode], max_tokens=shape.T, p2p=True, iters=3)
    for r in range(G):
        assert torch.equal(ref[r][0].view(torch.int16), got[r][0].view(torch.int16)), r
        assert torch.equal(ref[r][1]["out_f32"], got[r][1]["out_f32"]), r
    if par == "ep":
        _check_group_outputs(host, 2, host["x"], [g[0] for g in got], [g[1] for g in got])
    else:
        for r in range(1, G):
            assert torch.equal(got[0][0], got[r][0])
        _check_group_outputs(host, 2, host["x"], [got[0][0]], [got[0][1]])


@pytest.mark.parametrize("G", [2, 4, 8])
def test_ep_router_dispatch(moe, G):
    """EP over peer memory with the dispatch folded into the router (tuning ep_fold = 2, T <= 64
    per rank): the router's blocks wait for the scan and store their rows and meta into the
    destinations' buffers themselves (no permute / fill launch). Bit-identical to the
    permute-kernel dispatch (ep_fold = 1) over 3 forwards, an empty rank and a 64-token rank
    included, and the oracle within tolerance."""
    shape = synth.MoEShape(T=64 * G // 2, d=256, f=512, E=8, k=2)
    inp = _inputs(shape, 7800 + G)
    host = to_host_inputs(inp)
    cuts = np.linspace(0, shape.T, G + 1).astype(int)
    cuts[1] = 0  # rank 0: no tokens; the others up to 64
    shards = [inp["x"][cuts[r]:cuts[r + 1]] for r in range(G)]
    outs = []
    for tu in ({"ep_fold": 2}, {"ep_fold": 1}):
        res = _run_group(moe, inp, moe.MOE_PAR_EP, G, shards, max_tokens=64, p2p=True, iters=3, tuning=tu)
        outs.append(res)
    for r in range(G):
        assert torch.equal(outs[0][r][0].view(torch.int16), outs[1][r][0].view(torch.int16)), r
        assert torch.equal(outs[0][r][1]["out_f32"], outs[1][r][1]["out_f32"]), r
        assert torch.equal(outs[0][r][1]["pos"], outs[1][r][1]["pos"]), r
    _check_group_outputs(host, 2, host["x"], [g[0] for g in outs[0]], [g[1] for g in outs[0]])


@pytest.mark.parametrize("par", ["ep", "tp"])
def test_p2p_multiprocess_ipc(moe, par, tmp_path):
    """MOE_FLAG_P2P across two PROCESSES (CUDA IPC mappings of each other's region,
    handles all-gathered over gloo), both on this GPU: bitwise equal to the
    in-process collective path and to itself over 3 forwards."""
    import socket
    import subprocess
    import sys
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tests", "p2p_worker.py"), par, str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = [torch.load(tmp_path / f"rank{i}.pt") for i in range(2)]
    shape = synth.MoEShape(T=96, d=256, f=512, E=8, k=2)
    inp = _inputs(shape, 81)
    if par == "ep":
        cuts = np.linspace(0, shape.T, 3).astype(int)
        shards = [inp["x"][cuts[i]:cuts[i + 1]] for i in range(2)]
        ref = _run_group(moe, inp, moe.MOE_PAR_EP, 2, shards, max_tokens=shape.T)
    else:
        ref = _run_group(moe, inp, moe.MOE_PAR_TP, 2, [inp["x"]] * 2, max_tokens=shape.T)
    for i in range(2):
        for o in got[i]["outs"]:
            assert torch.equal(o.view(torch.int16), ref[i][0].cpu().view(torch.int16)), i
        assert torch.equal(got[i]["out_f32"], ref[i][1]["out_f32"].cpu())


def test_real_nccl_multigpu(moe, tmp_path):
    """EP (capacity + exact), TP, hybrid EP2xTPn and the P2P transport over REAL NCCL /
    CUDA peer memory, one process per GPU (torchrun), every rank's output against the
    single-GPU oracle on the global batch. Needs >= 2 GPUs: NCCL refuses two ranks on one
    device, so on a 1-GPU box this is skipped (the same device paths are covered there by
    the loopback / in-process P2P tests and test_nccl_world1)."""
    import socket
    import subprocess
    import sys
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (NCCL: one rank per device)")
    G = min(n, 8)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(G),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tests", "nccl_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = [torch.load(tmp_path / f"rank{i}.pt") for i in range(G)]
    import nccl_worker
    inp = _inputs(nccl_worker.SHAPE, 91)
    host = to_host_inputs(inp)
    for name in got[0]:
        per = [g[name] for g in got]
        for p in per:
            assert torch.equal(p["outs"][0].view(torch.int16), p["outs"][1].view(torch.int16)), name
        firsts = {}
        for p in per:  # ranks holding the same token shard (TP, hybrid tp group) agree bit for bit
            if p["shard"] in firsts:
                assert torch.equal(firsts[p["shard"]]["outs"][0].view(torch.int16), p["outs"][0].view(torch.int16))
            else:
                firsts[p["shard"]] = p
        order = [firsts[s] for s in sorted(firsts)]
        _check_group_outputs(host, 2, host["x"], [p["outs"][0] for p in order],
                             [{"topk_idx": p["topk_idx"], "out_f32": p["out_f32"]} for p in order])


def test_p2p_errors(moe):
    """MOE_FLAG_P2P: forward before connect, wrong world, hybrid, foreign handle."""
    shape = synth.MoEShape(T=8, d=64, f=256, E=4, k=2)
    inp = _inputs(shape, 3)
    mk = lambda r, G=2: moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], max_tokens=8, par=moe.MOE_PAR_EP,
                                     world_size=G, rank=r, flags=moe.MOE_FLAG_P2P)
    a, b = mk(0), mk(1)
    with pytest.raises(moe.MoEError, match="connect"):
        a.forward(inp["x"])
    with pytest.raises(moe.MoEError):
        a.p2p_connect([a.p2p_handle()])                      # world 1 != 2
    with pytest.raises(moe.MoEError):
        a.p2p_connect([b.p2p_handle(), a.p2p_handle()])      # rank order swapped
    c4 = mk(0, 4)
    with pytest.raises(moe.MoEError):
        a.p2p_connect([c4.p2p_handle(), b.p2p_handle()])     # region of another config
    with pytest.raises(moe.MoEError):
        moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], max_tokens=8, par=moe.MOE_PAR_HYBRID,
                     world_size=2, rank=0, tp_size=2, flags=moe.MOE_FLAG_P2P)
    plain = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], max_tokens=8)
    with pytest.raises(moe.MoEError):
        plain.p2p_handle()
    one = mk(0, 1)
    one.p2p_connect([one.p2p_handle()])
    with pytest.raises(moe.MoEError):
        one.p2p_connect([one.p2p_handle()])                  # connected twice
    one.forward(inp["x"])
    torch.cuda.synchronize()
    for blk in (a, b, c4, plain, one):
        blk.close()


@pytest.mark.parametrize("par", ["ep", "tp"])
def test_p2p_graph_capture(moe, par):
    """MOE_FLAG_P2P forwards are graph-capturable (each exchange waits for its counter to
    reach G and resets it): a 1-rank group (the signal kernel, the wait and the reset are
    all in the captured forward) captured once, replayed several times, bit-identical to
    the eager forwards, then eager again (counters left consistent)."""
    shape = synth.MoEShape(T=48, d=256, f=512, E=4, k=2)
    inp = _inputs(shape, 33)
    pm = moe.MOE_PAR_EP if par == "ep" else moe.MOE_PAR_TP
    one = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], max_tokens=48, par=pm, world_size=1, rank=0,
                       flags=moe.MOE_FLAG_P2P)
    one.p2p_connect([one.p2p_handle()])
    ref = one.forward(inp["x"]).clone()
    out = torch.empty_like(ref)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        one.forward(inp["x"], out=out)
    for _ in range(4):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
    again = one.forward(inp["x"])                            # eager after the replays: counters consistent
    torch.cuda.synchronize()
    assert torch.equal(again.view(torch.int16), ref.view(torch.int16))
    one.close()


@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("mode", ["swap", "tiled"])
def test_tp_loopback(moe, G, mode):
    """Tensor parallel: ffn sharded, fp32 reduce-scatter + bf16 all-gather; every
    rank's output identical and equal to the oracle's."""
    shape = synth.MoEShape(T=80, d=256, f=512, E=4, k=2)
    inp = _inputs(shape, 60 + G)
    host = to_host_inputs(inp)
    res = _run_group(moe, inp, moe.MOE_PAR_TP, G, [inp["x"]] * G, flags=MODES[mode])
    for r in range(1, G):
        assert torch.equal(res[r][0].view(torch.int16), res[0][0].view(torch.int16))
    _check_group_outputs(host, 2, host["x"], [res[0][0]], [res[0][1]])


@pytest.mark.parametrize("par", ["ep", "ep_exact", "tp", "ep_p2p", "tp_p2p"])
def test_mixtral_decode_8_ranks(moe, mixtral_weights, par):
    """BASELINE configs[3]/[4] shapes at G=8 (loopback / in-process peer memory):
    64-token decode, Mixtral layer."""
    w, host = mixtral_weights
    x = synth.make_tokens(64, 4096, seed=300, device="cuda")
    G = 8
    p2p = par.endswith("p2p")
    if par.startswith("ep"):
        shards = [x[8 * r:8 * (r + 1)] for r in range(G)]
        res = _run_group(moe, w, moe.MOE_PAR_EP, G, shards, max_tokens=8,
                         flags=moe.MOE_FLAG_EP_EXACT if par == "ep_exact" else 0, p2p=p2p, iters=2 if p2p else 1)
        outs, auxs = [r[0] for r in res], [r[1] for r in res]
    else:
        res = _run_group(moe, w, moe.MOE_PAR_TP, G, [x] * G, max_tokens=64, p2p=p2p, iters=2 if p2p else 1)
        for r in range(1, G):
            assert torch.equal(res[r][0].view(torch.int16), res[0][0].view(torch.int16))
        outs, auxs = [res[0][0]], [res[0][1]]
    e32, e16 = _check_group_outputs(host, 2, synth.bf16_bits(x), outs, auxs)
    print(par, "G=8", e32, e16)


@pytest.mark.parametrize("par", ["ep", "tp"])
def test_nccl_world1(moe, par):
    """The production NCCL transport (libnccl loaded at run time) on a 1-rank communicator."""
    uid = moe.moe_nccl_unique_id()
    comm = moe.moe_nccl_comm_init(uid, 1, 0, torch.cuda.current_device())
    inp = _inputs(synth.MoEShape(T=40, d=128, f=256, E=4, k=2), 91)
    p = moe.MOE_PAR_EP if par == "ep" else moe.MOE_PAR_TP
    blk = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=40, par=p, world_size=1,
                       rank=0, nccl_comm=comm)
    run = GpuRun(blk, inp["x"])
    host = to_host_inputs(inp)
    y = oracle.moe_forward(host["x"], host["wg"], host["w1"], host["w3"], host["w2"], 2,
                           forced_idx=run.np("topk_idx"))
    from parity import rel_err
    assert rel_err(run.np("out_f32"), y).max() <= 2e-2
    assert rel_err(run.np("out"), y).max() <= 2e-2
    blk.close()
    moe.moe_nccl_comm_destroy(comm)


def test_nvls_world1(moe):
    """MOE_FLAG_NVLS on a 1-rank NCCL communicator: NVLink SHARP needs a multicast object
    over >= 2 GPUs, so moe_init must refuse cleanly with MOE_ERR_UNSUPPORTED (nothing
    leaks: a plain TP context on the same communicator still works afterwards); if the
    platform does give a 1-GPU multicast object, the fused path must pass the oracle.
    The >= 2-GPU run is test_real_nccl_multigpu's tp_nvls case."""
    uid = moe.moe_nccl_unique_id()
    comm = moe.moe_nccl_comm_init(uid, 1, 0, torch.cuda.current_device())
    inp = _inputs(synth.MoEShape(T=40, d=128, f=256, E=4, k=2), 92)
    host = to_host_inputs(inp)
    try:
        blk = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=40, par=moe.MOE_PAR_TP,
                           world_size=1, rank=0, nccl_comm=comm, flags=moe.MOE_FLAG_NVLS)
    except moe.MoEError as ex:
        assert ex.status == moe.MOE_ERR_UNSUPPORTED and "NVLS" in str(ex), str(ex)
        print("NVLS at world 1:", ex)
        blk = None
    if blk is not None:
        check_forward(GpuRun(blk, inp["x"]), host, 2)
        blk.close()
    plain = moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=40, par=moe.MOE_PAR_TP,
                         world_size=1, rank=0, nccl_comm=comm)
    check_forward(GpuRun(plain, inp["x"]), host, 2)
    plain.close()
    moe.moe_nccl_comm_destroy(comm)


# ---------------------------------------------------------------- C5: layer stack with residual
def _stack_aux(L, T, d, k):
    return [{"topk_idx": torch.empty(T, k, dtype=torch.int32, device="cuda"),
             "out_f32": torch.empty(T, d, dtype=torch.float32, device="cuda")} for _ in range(L)]


def _check_stack_layers(layers, x, outs, auxs, k, literal_bf16):
    """Per-layer teacher-forced parity of x_{l+1} = x_l + MoE_l(x_l) (reading R12): layer
    l's GPU output vs the oracle applied to the GPU's own input of that layer. Routing
    bit-exact outside the margin band (R4); EVERY token's output -- margin-band ones
    included -- checked against the oracle under the GPU's routing (forced-routing mode,
    SURVEY 8(c) s4 strengthening): out_f32 within 2e-2, bf16 out == RNE(out_f32), and at
    decode sizes the literal bf16 output within 2e-2."""
    from parity import rel_err, routing_check
    cur = x
    stats = []
    for l, lw in enumerate(layers):
        h = {n: synth.bf16_bits(v) for n, v in lw.items()}
        xin = synth.bf16_bits(cur)
        gidx = auxs[l]["topk_idx"].cpu().numpy()
        excl, bad = routing_check(gidx, oracle.router(xin, h["wg"], k))
        assert not bad, (l, bad[:10])
        ref = oracle.moe_forward(xin, h["wg"], h["w1"], h["w3"], h["w2"], k, forced_idx=gidx, residual=True)
        of32 = auxs[l]["out_f32"].cpu().numpy()
        ob16 = outs[l].float().cpu().numpy().astype(np.float64)
        e32, e16 = rel_err(of32, ref).max(), rel_err(ob16, ref).max()
        assert e32 <= 2e-2, (l, e32)
        rne = torch.from_numpy(of32).to(torch.bfloat16).float().numpy().astype(np.float64)
        np.testing.assert_array_equal(ob16, rne)
        if literal_bf16:
            assert e16 <= 2e-2, (l, e16)
        stats.append((l, int(excl.sum()), float(e32), float(e16)))
        cur = outs[l]
    return stats


@pytest.mark.parametrize("L,shape", [(6, synth.MoEShape(T=100, d=256, f=512, E=8, k=2)),
                                     (3, synth.MoEShape(T=64, d=4096, f=14336, E=8, k=2)),
                                     (2, synth.MoEShape(T=575, d=4096, f=14336, E=8, k=2))])
def test_stack_teacher_forced(moe, L, shape):
    """C5 composition on one shared context (BASELINE configs[4] per-layer shape; T = 575
    is the M1 mixed batch): every layer teacher-forced against the oracle, margin-band
    tokens under forced routing, out_f32 checked too."""
    layers = [synth.make_weights(shape.d, shape.f, shape.E, seed=500, layer=l, device="cuda") for l in range(L)]
    x = synth.make_tokens(shape.T, shape.d, seed=501, device="cuda")
    st = moe.MoEStack(layers, top_k=shape.k, max_tokens=shape.T)
    outs, auxs = [], _stack_aux(L, shape.T, shape.d, shape.k)
    y = st.forward(x, layer_outputs=outs, layer_aux=auxs)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), outs[-1].view(torch.int16))
    print("stack", shape.T, _check_stack_layers(layers, x, outs, auxs, shape.k, literal_bf16=shape.T <= 128))
    st.close()


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("T", [64, 575])
def test_tp_stack_loopback(moe, G, T):
    """C5 is a TENSOR-PARALLEL stack (BASELINE configs[4]): G ranks (threads, loopback
    transport) each hold an f/G slice of 2 Mixtral-size layers; every layer ends in the
    fp32 reduce-scatter + one rounding + bf16 all-gather. All ranks' outputs bit-identical;
    each layer teacher-forced against the oracle."""
    import threading
    L, d, f, E, k = 2, 4096, 14336, 8, 2
    layers = [synth.make_weights(d, f, E, seed=510, layer=l, device="cuda") for l in range(L)]
    x = synth.make_tokens(T, d, seed=511, device="cuda")
    grp = moe.moe_loopback_comm_create(G)
    comms = [moe.moe_loopback_comm_rank(grp, r) for r in range(G)]
    stacks = [moe.MoEStack(layers, top_k=k, max_tokens=T, par=moe.MOE_PAR_TP, world_size=G, rank=r,
                           nccl_comm=comms[r]) for r in range(G)]
    torch.cuda.synchronize()
    res, errs = [None] * G, []
    streams = [torch.cuda.Stream() for _ in range(G)]

    def work(r):
        try:
            outs, auxs = [], _stack_aux(L, T, d, k)
            with torch.cuda.stream(streams[r]):
                stacks[r].forward(x, stream=streams[r], layer_outputs=outs, layer_aux=auxs)
            streams[r].synchronize()
            res[r] = (outs, auxs)
        except Exception as ex:  # pragma: no cover
            errs.append((r, ex))

    ths = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=900)
    for s_ in stacks:
        s_.close()
    for cm in comms:
        moe.moe_loopback_comm_destroy(cm)
    moe.moe_loopback_comm_destroy(grp)
    assert not errs, errs
    for r in range(1, G):
        for l in range(L):
            assert torch.equal(res[r][0][l].view(torch.int16), res[0][0][l].view(torch.int16)), (r, l)
            assert torch.equal(res[r][1][l]["out_f32"], res[0][1][l]["out_f32"]), (r, l)
    print("tp stack", G, T, _check_stack_layers(layers, x, res[0][0], res[0][1], k, literal_bf16=T <= 128))


# ---------------------------------------------------------------- hybrid EP x TP
def _run_hybrid(moe, inp, ep, tp, shards, flags=0, max_tokens=None):
    """G = ep*tp ranks (threads) on one GPU; rank (e, t) = e*tp + t; EP groups =
    ranks with the same t, TP groups = ranks with the same e; rank (e, t) gets the
    token shard e."""
    import threading
    G = ep * tp
    ep_groups = [moe.moe_loopback_comm_create(ep) for _ in range(tp)]
    tp_groups = [moe.moe_loopback_comm_create(tp) for _ in range(ep)]
    handles = []
    blocks = []
    mt = max_tokens or max(1, max(s.shape[0] for s in shards))
    for e in range(ep):
        for t in range(tp):
            ce = moe.moe_loopback_comm_rank(ep_groups[t], e)
            ct = moe.moe_loopback_comm_rank(tp_groups[e], t)
            handles += [ce, ct]
            blocks.append(moe.MoEBlock(inp["wg"], inp["w1"], inp["w3"], inp["w2"], top_k=2, max_tokens=mt,
                                       par=moe.MOE_PAR_HYBRID, world_size=G, rank=e * tp + t, nccl_comm=ce,
                                       tp_size=tp, tp_comm=ct, flags=flags))
    torch.cuda.synchronize()
    d = inp["wg"].shape[1]
    res = [None] * G
    errs = []

    def work(r):
        try:
            st = torch.cuda.Stream()
            x = shards[r // tp]
            T = x.shape[0]
            aux = {"topk_idx": torch.empty(max(T, 1), 2, dtype=torch.int32, device="cuda"),
                   "out_f32": torch.empty(max(T, 1), d, dtype=torch.float32, device="cuda")}
            out = torch.empty(max(T, 1), d, dtype=torch.bfloat16, device="cuda")
            with torch.cuda.stream(st):
                moe.moe_forward(blocks[r].ctx, x if T else out, T, blocks[r].router_w, blocks[r].w13, blocks[r].w2,
                                out, aux, st)
            st.synchronize()
            res[r] = (out[:T].clone(), {n: v[:T].clone() for n, v in aux.items()})
        except Exception as ex:  # pragma: no cover
            errs.append((r, ex))

    ths = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    for b in blocks:
        b.close()
    for h in handles:
        moe.moe_loopback_comm_destroy(h)
    for g in ep_groups + tp_groups:
        moe.moe_loopback_comm_destroy(g)
    assert not errs, errs
    return res


@pytest.mark.parametrize("ep,tp", [(2, 2), (2, 4), (4, 2), (1, 2), (2, 1)])
@pytest.mark.parametrize("mode", ["capacity", "exact"])
def test_hybrid_loopback(moe, ep, tp, mode):
    shape = synth.MoEShape(T=72, d=256, f=1024, E=8, k=2)
    inp = _inputs(shape, 70 + ep * 10 + tp)
    host = to_host_inputs(inp)
    cuts = np.linspace(0, shape.T, ep + 1).astype(int)
    shards = [inp["x"][cuts[e]:cuts[e + 1]] for e in range(ep)]
    res = _run_hybrid(moe, inp, ep, tp, shards, flags=moe.MOE_FLAG_EP_EXACT if mode == "exact" else 0,
                      max_tokens=shape.T)
    for e in range(ep):
        for t in range(1, tp):
            assert torch.equal(res[e * tp + t][0].view(torch.int16), res[e * tp][0].view(torch.int16))
    outs = [res[e * tp][0] for e in range(ep)]
    auxs = [res[e * tp][1] for e in range(ep)]
    _check_group_outputs(host, 2, host["x"], outs, auxs)


@pytest.mark.parametrize("ep,tp", [(2, 4), (4, 2)])
def test_mixtral_decode_hybrid(moe, mixtral_weights, ep, tp):
    """The paper's Exp4 hybrids (EP2xTP4, EP4xTP2) at Mixtral size, 64-token decode."""
    w, host = mixtral_weights
    x = synth.make_tokens(64, 4096, seed=301, device="cuda")
    per = 64 // ep
    shards = [x[per * e:per * (e + 1)] for e in range(ep)]
    res = _run_hybrid(moe, w, ep, tp, shards, max_tokens=per)
    outs = [res[e * tp][0] for e in range(ep)]
    auxs = [res[e * tp][1] for e in range(ep)]
    e32, e16 = _check_group_outputs(host, 2, synth.bf16_bits(x), outs, auxs)
    print(f"EP{ep}xTP{tp}", e32, e16)


# ---------------------------------------------------------------- FP8 weights
def _fp8_inputs(shape, seed):
    inp = _inputs(shape, seed)
    qs = {n: synth.quantize_fp8_rows(inp[n]) for n in ("w1", "w3", "w2")}
    # oracle inputs: the exact dequantised weights (fp32) and the bf16 tokens / router (exact in fp32)
    host = {n: synth.dequantize_fp8_rows(*qs[n]).cpu().numpy() for n in qs}
    host["x"] = inp["x"].float().cpu().numpy()
    host["wg"] = inp["wg"].float().cpu().numpy()
    return inp, qs, host


@pytest.mark.parametrize("T,d,f,E", [(16, 128, 128, 4), (64, 512, 1024, 8), (300, 256, 512, 8), (7, 128, 256, 2),
                                     (200, 384, 640, 6)])
def test_fp8_weights(moe, T, d, f, E):
    """FP8 E4M3 weights with per-row power-of-two scales: the GPU must match the oracle
    evaluated on the exact dequantised weights (same tolerance as bf16)."""
    inp, qs, host = _fp8_inputs(synth.MoEShape(T=T, d=d, f=f, E=E, k=2), 800 + T)
    blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T,
                       flags=moe.MOE_FLAG_FP8_WEIGHTS)
    run = GpuRun(blk, inp["x"])
    st = check_forward(run, host, 2)
    print("fp8", T, d, f, E, st)
    blk.close()


@pytest.mark.parametrize("T", [16, 64, 128])
def test_fp8_skewed(moe, T):
    """FP8 decode under skewed routing (expert 0 ~4x as popular, synth.make_tokens_skewed):
    uneven token tiles per expert on the 8-bit GEMMs, parity against the exact-dequant
    oracle."""
    shape = synth.MoEShape(T=T, d=512, f=1024, E=8, k=2)
    inp, qs, host = _fp8_inputs(shape, 900 + T)
    x = synth.make_tokens_skewed(T, shape.d, inp["wg"], seed=901 + T, device="cuda")
    host["x"] = x.float().cpu().numpy()
    blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T,
                       flags=moe.MOE_FLAG_FP8_WEIGHTS)
    run = GpuRun(blk, x)
    check_forward(run, host, 2)
    blk.close()


@pytest.mark.parametrize("T", [64, 300])
def test_fp8_two_term_tokens(moe, T):
    """FP8 weights, both GEMMs on 8-bit MMAs: tokens split into two E4M3 terms with a
    per-row power-of-two scale. Rows scaled by 2^3 and 2^-10 (exact in bf16) and a zero row
    exercise the token scale, the h block scales (an all-zero block) and their ranges;
    every row against the oracle, the zero row exactly zero."""
    shape = synth.MoEShape(T=T, d=512, f=1024, E=8, k=2)
    inp, qs, host = _fp8_inputs(shape, 900 + T)
    x = inp["x"].float()
    x[1] *= 8.0
    x[2] *= 2.0 ** -10
    x[3] = 0
    inp["x"] = x.to(torch.bfloat16)
    host["x"] = inp["x"].float().cpu().numpy()
    blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T,
                       flags=moe.MOE_FLAG_FP8_WEIGHTS)
    run = GpuRun(blk, inp["x"])
    print("fp8", T, check_forward(run, host, 2))
    assert np.all(run.np("out_f32")[3] == 0)
    blk.close()


@pytest.mark.parametrize("nb_cap", [0, 32, 64])
def test_fp8_block_scales(moe, nb_cap):
    """The UE8M0 block scales of h (one per token row and 32 ffn columns) must reach the
    block-scaled w2 MMA at the right (row, K block): w1 rows scaled per 32-column block by
    2^(b mod 7 - 3) and token rows by 2^(t mod 5 - 2), so neighbouring blocks and rows get
    different scales -- a scale applied to the wrong row or block is off by powers of two.
    Token tiles capped at 32 / 64 rows put B tiles at every 32-row group of the 128-row
    scale atom."""
    shape = synth.MoEShape(T=200, d=256, f=512, E=8, k=2)
    inp = _inputs(shape, 1300 + nb_cap)
    w1 = inp["w1"].float()
    blk_scale = torch.tensor([2.0 ** (b % 7 - 3) for b in range(shape.f // 32)], device=w1.device)
    w1 = w1 * blk_scale.repeat_interleave(32).view(1, -1, 1)
    inp["w1"] = w1.to(torch.bfloat16)
    x = inp["x"].float() * torch.tensor([2.0 ** (t % 5 - 2) for t in range(shape.T)], device=w1.device).view(-1, 1)
    inp["x"] = x.to(torch.bfloat16)
    qs = {n: synth.quantize_fp8_rows(inp[n]) for n in ("w1", "w3", "w2")}
    host = {n: synth.dequantize_fp8_rows(*qs[n]).cpu().numpy() for n in qs}
    host["x"] = inp["x"].float().cpu().numpy()
    host["wg"] = inp["wg"].float().cpu().numpy()
    blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=shape.T,
                       flags=moe.MOE_FLAG_FP8_WEIGHTS, tuning={"swap_nb_cap": nb_cap} if nb_cap else None)
    print("fp8 block scales", nb_cap, check_forward(GpuRun(blk, inp["x"]), host, 2))
    blk.close()


def test_fp8_mixtral_decode(moe):
    """64-token decode at Mixtral size with FP8 weights, all tokens vs the oracle."""
    w = synth.make_weights(4096, 14336, 8, seed=43, device="cuda")
    qs = {n: synth.quantize_fp8_rows(w[n]) for n in ("w1", "w3", "w2")}
    host = {n: synth.dequantize_fp8_rows(*qs[n]).cpu().numpy() for n in qs}
    x = synth.make_tokens(64, 4096, seed=44, device="cuda")
    host["x"] = x.float().cpu().numpy()
    host["wg"] = w["wg"].float().cpu().numpy()
    blk = moe.MoEBlock(w["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=64,
                       flags=moe.MOE_FLAG_FP8_WEIGHTS)
    run = GpuRun(blk, x)
    st = check_forward(run, host, 2)
    print("fp8 C2", st)
    blk.close()


def test_cuda_graph_capture(moe):
    """The single-GPU forward has no host synchronisation: it can be captured into a
    CUDA graph (PDL edges included) and replayed with bit-identical results."""
    for shape, flags in ((synth.MoEShape(T=64, d=256, f=512, E=8, k=2), 0),
                         (synth.MoEShape(T=600, d=256, f=512, E=8, k=2), moe.MOE_FLAG_FORCE_TILED)):
        inp = _inputs(shape, 900 + shape.T)
        blk = _block(moe, inp, 2, shape.T, flags)
        ref = blk.forward(inp["x"]).clone()
        out = torch.empty_like(ref)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            moe.moe_forward(blk.ctx, inp["x"], shape.T, blk.router_w, blk.w13, blk.w2, out, None,
                            torch.cuda.current_stream())
        for _ in range(3):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
        blk.close()


def test_cuda_graph_capture_fp8(moe):
    """FP8-weight forward (bench.py --fp8 replays it as a CUDA graph): capturable, and
    replays bit-identical to the eager call."""
    T = 64
    inp, qs, _ = _fp8_inputs(synth.MoEShape(T=T, d=256, f=512, E=8, k=2), 950)
    blk = moe.MoEBlock(inp["wg"], qs["w1"], qs["w3"], qs["w2"], top_k=2, max_tokens=T,
                       flags=moe.MOE_FLAG_FP8_WEIGHTS)
    ref = blk.forward(inp["x"]).clone()
    out = torch.empty_like(ref)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        moe.moe_forward(blk.ctx, inp["x"], T, blk.router_w, blk.w13, blk.w2, out, None,
                        torch.cuda.current_stream(), blk.s13, blk.s2)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
    blk.close()


def test_large_token_counts(moe):
    """T > 65535 (1-D grids everywhere; no gridDim.y limit), tiny hidden size."""
    shape = synth.MoEShape(T=70000, d=64, f=128, E=4, k=2)
    inp = _inputs(shape, 1234)
    blk = _block(moe, inp, 2, shape.T)
    run = GpuRun(blk, inp["x"])
    rng = np.random.default_rng(1)
    toks = np.unique(np.concatenate([[0, 65535, 65536, shape.T - 1], rng.choice(shape.T, 60, replace=False)]))
    check_forward(run, to_host_inputs(inp), 2, tokens=toks)
    blk.close()


def test_ep_exact_many_slots(moe):
    """EP exact-count exchange with more than 65535 receive slots (G * max_tokens * k)."""
    shape = synth.MoEShape(T=40000, d=64, f=128, E=4, k=2)
    inp = _inputs(shape, 4321)
    host = to_host_inputs(inp)
    shards = [inp["x"][:20000], inp["x"][20000:]]
    res = _run_group(moe, inp, moe.MOE_PAR_EP, 2, shards, flags=moe.MOE_FLAG_EP_EXACT, max_tokens=20000)
    outs = [r[0] for r in res]
    auxs = [r[1] for r in res]
    _check_group_outputs(host, 2, host["x"], outs, auxs)
