"""Seeded synthetic inputs for the MoE block -- shared by tests/ and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
numbers and rounds them to the storage dtype. Both the CUDA path and the
oracle consume the exact bytes it returns (the oracle decodes bf16 itself).

Recipe (PAPER.md is silent, Sec. 5 used real
Mixtral weights and OpenOrca prompts, which are out of scope):
  x   ~ N(0, 1)          [T, d]
  W_g ~ N(0, 1/d)        [E, d]
  W1  ~ N(0, 1/d)        [E, f, d]   (HF nn.Linear [out, in])
  W3  ~ N(0, 1/d)        [E, f, d]
  W2  ~ N(0, 1/f)        [E, d, f]
all rounded to bf16 with round-to-nearest-even (torch's `.to(torch.bfloat16)`),
or kept fp32 for the tiny config's fp32 self-tests (BASELINE.json configs[0]).
This gives router logits with std ~1, i.e. real top-2 competition, and an
expert output rms ~0.6.

Seeds: tensor i of layer L draws from torch.Generator(device).manual_seed(
seed * 1000 + 100 * L + i) with i = 0 (x), 1 (W_g), 2 (W1), 3 (W3), 4 (W2).
Large configs may be drawn on a CUDA generator (fast); the bytes are then
copied to the host for the oracle, which is allowed because torch's RNG is
plumbing, not the CUDA path under test.
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass(frozen=True)
class MoEShape:
    T: int
    d: int
    f: int
    E: int
    k: int


# BASELINE.json configs (numbered from 0 here): 0 tiny, 1 decode, 2 prefill.
TINY = MoEShape(T=16, d=64, f=128, E=4, k=2)
DECODE = MoEShape(T=64, d=4096, f=14336, E=8, k=2)
PREFILL = MoEShape(T=64 * 512, d=4096, f=14336, E=8, k=2)


def _randn(shape, std, seed, device, dtype):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    t = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t.to(dtype)


def make_tokens(T, d, seed, layer=0, device="cpu", dtype=torch.bfloat16):
    return _randn((T, d), 1.0, seed * 1000 + 100 * layer + 0, device, dtype)


# C5 stack recipe (R12): x_{l+1} = x_l + MoE_l(x_l) with the single-layer recipe
# diverges -- the SwiGLU block's output grows with the square of its input (rms 0.44 at
# input rms 1), so the residual stream reaches rms 1e5 by layer 8 and NaN by layer 16 at
# T = 64, and the NaN rows all route to experts 0 and 1 (scripts/exp/stack_counts.py).
# The stack therefore draws W2 with std STACK_W2_SCALE / sqrt(f): the block's gain drops to
# ~0.11 at rms 1 and the stream stays near rms 1-2 over 32 layers with every expert used.
STACK_W2_SCALE = 0.25


def make_weights(d, f, E, seed, layer=0, device="cpu", dtype=torch.bfloat16, w2_scale=1.0):
    """Return dict wg [E,d], w1 [E,f,d], w3 [E,f,d], w2 [E,d,f] (HF layout). w2_scale scales
    the std of W2 (STACK_W2_SCALE for the C5 stack)."""
    base = seed * 1000 + 100 * layer
    return {
        "wg": _randn((E, d), 1.0 / math.sqrt(d), base + 1, device, dtype),
        "w1": _randn((E, f, d), 1.0 / math.sqrt(d), base + 2, device, dtype),
        "w3": _randn((E, f, d), 1.0 / math.sqrt(d), base + 3, device, dtype),
        "w2": _randn((E, d, f), w2_scale / math.sqrt(f), base + 4, device, dtype),
    }


# SURVEY 8(d) optional skew variant: x = z + mu with mu along router row 0, so expert 0's
# logit gains SKEW_ALPHA (the other logits move by ~cos(W_g rows) ~ 1/64) and expert 0 is
# picked ~4x as often as each other expert. SKEW_ALPHA from a Monte-Carlo of top-2 over 8
# iid N(0,1) logits (the recipe's logit distribution): P(expert 0 in the top 2) = 8/11
# <=> a 4:1 popularity ratio at alpha ~ 1.43 (1.4 -> 3.91, 1.5 -> 4.18).
SKEW_ALPHA = 1.43


def make_tokens_skewed(T, d, wg, seed, layer=0, device="cpu", dtype=torch.bfloat16, alpha=SKEW_ALPHA):
    """Tokens of the 4:1 expert-popularity workload (expert 0 popular): N(0,1) tokens plus
    alpha * g / |g|^2, g = router row 0 (bf16 router weights as given)."""
    z = _randn((T, d), 1.0, seed * 1000 + 100 * layer + 0, device, torch.float32)
    g = wg[0].to(device=device, dtype=torch.float32)
    return (z + alpha * g / g.dot(g)).to(dtype)


def make_inputs(shape: MoEShape, seed, layer=0, device="cpu", dtype=torch.bfloat16):
    w = make_weights(shape.d, shape.f, shape.E, seed, layer, device, dtype)
    w["x"] = make_tokens(shape.T, shape.d, seed, layer, device, dtype)
    return w


def bf16_bits(t: torch.Tensor):
    """bf16 tensor -> numpy uint16 view of the same bytes (host)."""
    assert t.dtype == torch.bfloat16
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view("uint16")


def quantize_fp8_rows(w: torch.Tensor):
    """Input preparation for the FP8-weight variant: for every output row
    of the HF [out, in] matrix a power-of-two scale s = 2^ceil(log2(max|w| / 448))
    (448 = largest E4M3 value) and q = E4M3(w / s) with torch's RNE conversion.
    Returns (q as uint8 bytes, s fp32 [..., out]); the exact weight is q * s."""
    wf = w.float()
    amax = wf.abs().amax(dim=-1).clamp_min(1e-30)
    s = torch.exp2(torch.ceil(torch.log2(amax / 448.0)))
    q = (wf / s.unsqueeze(-1)).to(torch.float8_e4m3fn)
    return q.view(torch.uint8), s.contiguous()


def dequantize_fp8_rows(q: torch.Tensor, s: torch.Tensor):
    """Exact fp32 value of q * s (E4M3 -> fp32 is exact; s is a power of two)."""
    return q.view(torch.float8_e4m3fn).float() * s.unsqueeze(-1)
