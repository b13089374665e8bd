"""Stress of the fused decode FFN's cross-CTA protocol (csrc/ffn_fused.cuh: tile claims on
sched[0], h-tile readiness counters, the last CTA's counter reset) without a race detector
(compute-sanitizer is closed on this GPU pool): many back-to-back forwards of one context
with a different token count and routing every time, each compared bit for bit with the
two-kernel swap path at the same K splits (tests/test_fused.py shows the two are
bit-identical where the split boundaries coincide), so a stale counter, a tile read before
its h was published or a lost claim shows up as a mismatch or a hang.

Routing alternates between the router (natural, near-uniform) and forced routing through
moe_forward_routed with a skewed expert popularity (SURVEY 8(d) skew variant, up to every
token on the same two experts -- several token tiles per expert, some experts empty).
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

E, K, TMAX = 8, 2, 128
ITERS = 96


@pytest.fixture(scope="module")
def moe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2408_00008_b200 as m
    return m


def _routing(rng, T):
    """Forced top-2 routing with a random Zipf-like expert popularity: distinct experts per
    token, gates renormalised (sum 1)."""
    skew = rng.choice([0.0, 1.0, 2.5, 8.0])
    p = 1.0 / np.arange(1, E + 1) ** skew
    p = p[rng.permutation(E)]
    p /= p.sum()
    idx = np.stack([rng.choice(E, 2, replace=False, p=p) for _ in range(T)]).astype(np.int32)
    g = rng.random((T, 1)).astype(np.float32) * 0.8 + 0.1
    w = np.concatenate([g, 1.0 - g], axis=1).astype(np.float32)
    return torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()


def _run(moe, blk, x, routed):
    T, D = x.shape
    out = torch.empty(T, D, dtype=torch.bfloat16, device="cuda")
    aux = {"out_f32": torch.empty(T, D, dtype=torch.float32, device="cuda")}
    n0 = moe.moe_launch_count(blk.ctx)
    if routed is None:
        blk.forward(x, out, aux)
    else:
        blk.forward_routed(x, routed[0], routed[1], out, aux)
    torch.cuda.synchronize()
    return out, aux["out_f32"], moe.moe_launch_count(blk.ctx) - n0


@pytest.mark.parametrize("D,F", [(512, 2048), (2048, 4096)])  # 16 / 32 ffn tiles: ~1 / ~2 tiles per CTA and phase
@pytest.mark.parametrize("variant", ["bf16", "half", "fp8"])
def test_fused_stress_bit_identical(moe, variant, D, F):
    rng = np.random.default_rng({"bf16": 11, "half": 12, "fp8": 13}[variant])
    w = synth.make_weights(D, F, E, seed=31, device="cuda")
    flags, tmax = moe.MOE_FLAG_FORCE_SWAP, TMAX
    w13 = {n: w[n] for n in ("w1", "w3", "w2")}
    if variant == "fp8":  # the FP8 fused kernel takes 32-row token tiles (T <= 32 keeps every expert in one)
        flags, tmax = moe.MOE_FLAG_FP8_WEIGHTS, 32
        w13 = {n: synth.quantize_fp8_rows(w[n]) for n in ("w1", "w3", "w2")}
    fused_tu = {"fused": 2, "fused_uniform": 1, "fused_splits": 4}
    if variant == "half":
        fused_tu["fused_half"] = 2
    blocks = [moe.MoEBlock(w["wg"], w13["w1"], w13["w3"], w13["w2"], top_k=K, max_tokens=tmax, flags=flags,
                           split_k=4, tuning=tu) for tu in (fused_tu, {"fused": 1})]
    try:
        n_fused = 0
        for it in range(ITERS):
            T = int(rng.integers(1, tmax + 1))
            x = synth.make_tokens(T, D, seed=1000 + it, device="cuda")
            routed = _routing(rng, T) if it % 2 else None
            (o_f, y_f, l_f), (o_2, y_2, l_2) = (_run(moe, b, x, routed) for b in blocks)
            assert l_2 == l_f + 1, (it, T, l_f, l_2)  # the fused launch replaced both GEMM kernels
            n_fused += 1
            assert torch.equal(y_f.view(torch.int32), y_2.view(torch.int32)), (it, T, routed is not None)
            assert torch.equal(o_f.view(torch.int16), o_2.view(torch.int16)), (it, T)
            if it % 8 == 0:  # the same forward again on the fused context: counters were reset
                o_r, y_r, _ = _run(moe, blocks[0], x, routed)
                assert torch.equal(y_r.view(torch.int32), y_f.view(torch.int32)), (it, T)
        assert n_fused == ITERS
    finally:
        for b in blocks:
            b.close()
