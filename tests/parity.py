"""Parity helpers shared by the GPU tests, smoke() and bench.py's checks.

The comparison rules are DESIGN.md readings R4 (routing margin rule) and R8
(tolerance), from BASELINE.json north_star: "Routing indices must match the
oracle bit-exactly, except for tokens whose 2nd/3rd logit margin is below 1e-3;
those tokens are logged and excluded. Outputs must match within max relative
error 2e-2 (bf16) per element, normalised by the row RMS."
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

MARGIN = 1e-3      # north_star: 2nd/3rd logit margin
TOL = 2e-2         # north_star: max relative error per element, normalised by the row RMS


def to_host_inputs(inp):
    """torch bf16 tensors (any device) -> dict of numpy uint16 bit patterns for the oracle."""
    return {k: synth.bf16_bits(v) for k, v in inp.items()}


def row_rms(y):
    r = np.sqrt(np.mean(np.asarray(y, np.float64) ** 2, axis=1))
    small = r < 1e-30
    if small.any():
        r = r.copy()
        r[small] = max(r[~small].mean() if (~small).any() else 1.0, 1e-30)
    return r


def rel_err(y_gpu, y_ref):
    """max_c |y_gpu - y_ref| / rms(y_ref row), per row."""
    y_gpu = np.asarray(y_gpu, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    return np.max(np.abs(y_gpu - y_ref), axis=1) / row_rms(y_ref)


def routing_check(gpu_idx, ref):
    """Margin rule (R4). Returns (excluded token mask, list of mismatching tokens)."""
    gpu_idx = np.asarray(gpu_idx)
    excl = ref["m23"] < MARGIN
    bad = []
    for t in np.nonzero(~excl)[0]:
        g, o = gpu_idx[t], ref["idx"][t]
        if sorted(g.tolist()) != sorted(o.tolist()):
            bad.append(int(t))
        elif ref["m12"][t] >= MARGIN and g.tolist() != o.tolist():
            bad.append(int(t))
    return excl, bad


class GpuRun:
    """Runs the CUDA path once through the C ABI with every aux output attached."""

    def __init__(self, block, x, routed=None):
        import paper_2408_00008_b200 as moe  # noqa: F401  (CUDA path)
        T, d = x.shape
        dev = x.device
        E, k = block.E, block.k
        self.aux = {
            "logits": torch.empty(T, E, dtype=torch.float32, device=dev),
            "topk_idx": torch.empty(T, k, dtype=torch.int32, device=dev),
            "topk_w": torch.empty(T, k, dtype=torch.float32, device=dev),
            "expert_counts": torch.empty(E, dtype=torch.int32, device=dev),
            "expert_offsets": torch.empty(E + 1, dtype=torch.int32, device=dev),
            "pos": torch.empty(T, k, dtype=torch.int32, device=dev),
            "out_f32": torch.empty(T, d, dtype=torch.float32, device=dev),
        }
        self.out = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        if routed is None:
            block.forward(x, self.out, self.aux)
        else:
            block.forward_routed(x, routed[0], routed[1], self.out, self.aux)
        torch.cuda.synchronize()

    def np(self, name):
        if name == "out":
            return self.out.float().cpu().numpy().astype(np.float64)
        return self.aux[name].cpu().numpy()


def check_forward(run: GpuRun, host, k, tokens=None, literal_bf16=True, tol=TOL, routed=False):
    """Full parity of one GPU run against the oracle. host = numpy uint16 inputs.
    tokens: optional subset of token indices for the output comparison.
    Returns a dict of statistics; raises AssertionError on any violation."""
    x, wg, w1, w3, w2 = (host[n] for n in ("x", "wg", "w1", "w3", "w2"))
    T = x.shape[0]
    E = wg.shape[0]
    stats = {}
    gidx = run.np("topk_idx")
    ref = oracle.router(x, wg, k)
    if not routed:
        # router logits: fp32 accumulation of exact products vs fp64
        lg = run.np("logits")
        stats["logit_max_abs_err"] = float(np.max(np.abs(lg - ref["logits"]))) if T else 0.0
        assert stats["logit_max_abs_err"] < 1e-3 * 0.1, stats
        excl, bad = routing_check(gidx, ref)
        stats["excluded"] = int(excl.sum())
        assert not bad, f"routing mismatch outside the margin band at tokens {bad[:10]}"
        # gates: fp32 closed form vs fp64 (for the GPU's own selection)
        gw = run.np("topk_w")
        if k == 2:
            l = ref["logits"]
            l1 = np.take_along_axis(l, gidx[:, :1].astype(np.int64), 1)[:, 0]
            l2 = np.take_along_axis(l, gidx[:, 1:2].astype(np.int64), 1)[:, 0]
            w0 = 1.0 / (1.0 + np.exp(l2 - l1))
            stats["gate_max_abs_err"] = float(np.max(np.abs(gw[:, 0] - w0))) if T else 0.0
            assert stats["gate_max_abs_err"] < 1e-5, stats
        assert np.all(np.abs(gw.sum(1) - 1.0) < 1e-6)
    # permutation: exact integers against the oracle's permutation of the GPU's routing
    perm = oracle.permutation(gidx, E, 128)
    np.testing.assert_array_equal(run.np("expert_counts"), perm["counts"])
    np.testing.assert_array_equal(run.np("expert_offsets"), perm["offsets"])
    np.testing.assert_array_equal(run.np("pos"), perm["pos"])
    # outputs
    toks = np.arange(T) if tokens is None else np.asarray(tokens)
    y_ref = oracle.moe_forward(x, wg, w1, w3, w2, k, forced_idx=gidx, tokens=toks)
    of32 = run.np("out_f32")[toks]
    ob16 = run.np("out")[toks]
    e32 = rel_err(of32, y_ref)
    stats["max_rel_err_f32"] = float(e32.max()) if len(toks) else 0.0
    assert stats["max_rel_err_f32"] <= tol, stats
    # the stored bf16 output is exactly RNE(out_f32) (torch's conversion as the library reference)
    rne = torch.from_numpy(run.np("out_f32")[toks]).to(torch.bfloat16).float().numpy().astype(np.float64)
    np.testing.assert_array_equal(ob16, rne)
    e16 = rel_err(ob16, y_ref)
    stats["max_rel_err_bf16"] = float(e16.max()) if len(toks) else 0.0
    stats["bf16_floor"] = float(rel_err(oracle.bf16_round(y_ref), y_ref).max()) if len(toks) else 0.0
    if literal_bf16:
        assert stats["max_rel_err_bf16"] <= tol, stats
    return stats
