"""Pins for the fp64 oracle (CPU only, -m "not gpu").

The oracle (oracle/moe_oracle.cpp) is trusted for GPU parity only because it
is pinned here to things other than itself:
  * the hand-derived worked example (tests/golden/worked_example.json),
  * textbook / library routines (numpy float64 matmul, einsum, Python math),
  * brute force on tiny inputs (all k-subsets, all experts evaluated densely),
  * closed forms (sigma(l1-l2) gates, silu(1) = sigma(1), identical experts),
  * invariances (token permutation, batch independence, expert relabelling),
  * the EP / TP partition identities.
Each test names the step of the definition (moe_oracle.cpp header / DESIGN.md)
it pins.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _np(t):
    return t.detach().cpu().numpy()


def _tiny(seed, dtype="f32", shape=synth.TINY):
    """C1 inputs (BASELINE.json configs[0]: fp32 random weights) as numpy arrays."""
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    inp = synth.make_inputs(shape, seed, dtype=tdt)
    if dtype == "f32":
        return {k: _np(v) for k, v in inp.items()}
    return {k: synth.bf16_bits(v) for k, v in inp.items()}


def _dec(a):
    return oracle.bf16_to_f64(a) if a.dtype == np.uint16 else a.astype(np.float64)


def _np_silu(z):
    return z / (1.0 + np.exp(-z))


def _np_dense_block(inp, k):
    """Independent numpy reference: evaluate ALL experts densely (brute force),
    then select by (logit desc, index asc) via np.lexsort, softmax-renormalise."""
    x, wg, w1, w3, w2 = (_dec(inp[n]) for n in ("x", "wg", "w1", "w3", "w2"))
    logits = x @ wg.T                                   # [T,E]
    a = np.einsum("td,efd->tef", x, w1)
    b = np.einsum("td,efd->tef", x, w3)
    o = np.einsum("tef,edf->ted", _np_silu(a) * b, w2)  # [T,E,d]
    T, E = logits.shape
    y = np.zeros((T, x.shape[1]))
    for t in range(T):
        order = np.lexsort((np.arange(E), -logits[t]))   # primary: -logit, then index
        S = order[:k]
        p = np.exp(logits[t] - logits[t].max())
        p /= p.sum()
        w = p[S] / p[S].sum()
        y[t] = (w[:, None] * o[t, S]).sum(0)
    return y, logits


# ---------------------------------------------------------------- worked example
def test_worked_example_golden():
    """Pins steps 2-6 incl. the tie-break (reading R3) on the hand-derived example."""
    g = json.load(open(os.path.join(GOLDEN, "worked_example.json")))
    x = np.array(g["x"], np.float64)
    wg = np.array(g["wg"], np.float64)
    w1 = np.array(g["w1"], np.float64)
    w3 = np.array(g["w3"], np.float64)
    w2 = np.array(g["w2"], np.float64)
    r = oracle.router(x, wg, g["k"])
    np.testing.assert_array_equal(r["logits"][0], g["expect_logits"])
    assert list(r["idx"][0]) == g["expect_idx"]
    np.testing.assert_allclose(r["w"][0], g["expect_w"], rtol=0, atol=1e-15)
    y = oracle.moe_forward(x, wg, w1, w3, w2, g["k"])
    np.testing.assert_allclose(y[0], g["expect_y"], rtol=0, atol=1e-15)
    # closed form, independent of both: y0 = sigma(1) * (sigma(.5)*1 + (1-sigma(.5))*2)
    s = lambda z: 1.0 / (1.0 + math.exp(-z))
    assert abs(y[0, 0] - s(1.0) * (s(0.5) + 2 * (1 - s(0.5)))) < 1e-15
    assert r["m23"][0] == 0.0  # the tie is a true tie (exempt from the margin rule)


def test_silu_one():
    """Pins silu (reading R11): E=1, k=1, d=f=1, all weights 1 -> y = silu(1) = sigma(1)."""
    one = np.ones((1, 1))
    y = oracle.moe_forward(one, one, one[None], one[None], one[None], k=1)
    assert abs(y[0, 0] - 0.7310585786300049) < 1e-16
    x0 = np.zeros((1, 1))
    assert oracle.moe_forward(x0, one, one[None], one[None], one[None], k=1)[0, 0] == 0.0


# ---------------------------------------------------------------- router (steps 2-4)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_logits_match_numpy_matmul(dtype, seed):
    """Step 2 vs numpy float64 matmul (library routine) on the decoded bytes."""
    inp = _tiny(seed, dtype)
    r = oracle.router(inp["x"], inp["wg"], 2)
    ref = _dec(inp["x"]) @ _dec(inp["wg"]).T
    np.testing.assert_allclose(r["logits"], ref, rtol=1e-12, atol=1e-13)


def _brute_topk(l, k):
    """All k-subsets; keep the max-sum ones; lexicographically smallest index tuple;
    slots ordered by (logit desc, index asc)."""
    best, best_set = None, None
    for S in itertools.combinations(range(len(l)), k):
        s = sum(l[i] for i in S)
        if best is None or s > best:
            best, best_set = s, S
    return sorted(best_set, key=lambda i: (-l[i], i))


@pytest.mark.parametrize("E,k", [(2, 1), (2, 2), (4, 2), (8, 2), (8, 1), (5, 3)])
def test_topk_bruteforce(E, k):
    """Step 3 vs brute-force subset enumeration, with many exact ties (integer logits)."""
    rng = np.random.default_rng(E * 10 + k)
    T = 300
    L = rng.integers(-3, 4, size=(T, E)).astype(np.float64)  # ties everywhere
    L[: T // 3] = rng.permutation(np.tile(np.arange(E, dtype=np.float64), (T // 3, 1)).T).T
    r = oracle.router(L, np.eye(E), k)  # x = logits, W_g = I -> l = x exactly
    np.testing.assert_array_equal(r["logits"], L)
    for t in range(T):
        assert list(r["idx"][t]) == _brute_topk(list(L[t]), k), (t, L[t])


def test_gates_closed_form():
    """Step 4: top-2 renormalised softmax == sigma(l1 - l2); sums to 1; ties -> 0.5."""
    rng = np.random.default_rng(7)
    E = 8
    L = rng.normal(size=(200, E)) * 3
    L[0] = 0.25
    r = oracle.router(L, np.eye(E), 2)
    for t in range(len(L)):
        l1, l2 = L[t, r["idx"][t, 0]], L[t, r["idx"][t, 1]]
        w0 = 1.0 / (1.0 + math.exp(l2 - l1))
        assert abs(r["w"][t, 0] - w0) < 1e-14
        assert abs(r["w"][t].sum() - 1.0) < 1e-15
        assert r["w"][t, 0] >= r["w"][t, 1]
    assert tuple(r["w"][0]) == (0.5, 0.5) and list(r["idx"][0]) == [0, 1]
    # E=2, k=2: both experts always picked
    r2 = oracle.router(L[:, :2], np.eye(2), 2)
    assert all(sorted(i) == [0, 1] for i in r2["idx"])
    # k=1: gate is exactly 1
    r1 = oracle.router(L, np.eye(E), 1)
    assert np.all(r1["w"] == 1.0)
    # general k: w_j = exp(l_j) / sum_selected exp(l)
    r3 = oracle.router(L, np.eye(E), 3)
    for t in range(5):
        S = r3["idx"][t]
        ex = [math.exp(L[t, i]) for i in S]
        np.testing.assert_allclose(r3["w"][t], [v / sum(ex) for v in ex], rtol=1e-13)


def test_margins():
    """Reading R4: m12 = l(1)-l(2), m23 = l(2)-l(3) from the fp64 logits."""
    L = np.array([[3.0, 1.0, 2.0, 0.5], [1.0, 1.0, 1.0, 0.0]])
    r = oracle.router(L, np.eye(4), 2)
    assert list(r["m12"]) == [1.0, 0.0] and list(r["m23"]) == [1.0, 0.0]


# ---------------------------------------------------------------- experts (step 5)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_single_expert_is_dense_swiglu(dtype):
    """E=1, k=1 => the block is a dense SwiGLU FFN: compare with numpy float64."""
    shape = synth.MoEShape(T=9, d=64, f=128, E=1, k=1)
    inp = _tiny(3, dtype, shape)
    y = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=1)
    x, w1, w3, w2 = (_dec(inp[n]) for n in ("x", "w1", "w3", "w2"))
    ref = (_np_silu(x @ w1[0].T) * (x @ w3[0].T)) @ w2[0].T
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-13)


def test_identical_experts_routing_independent():
    """W_e = W for all e => y = SwiGLU_W(x) for ANY routing (gates sum to 1)."""
    inp = _tiny(4, "f32")
    E = inp["w1"].shape[0]
    for n in ("w1", "w3", "w2"):
        inp[n] = np.repeat(inp[n][:1], E, axis=0)
    y = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=2)
    x, w1, w3, w2 = (_dec(inp[n]) for n in ("x", "w1", "w3", "w2"))
    ref = (_np_silu(x @ w1[0].T) * (x @ w3[0].T)) @ w2[0].T
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-13)
    forced = np.array([[3, 1]] * x.shape[0], np.int32)
    yf = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=2,
                            forced_idx=forced)
    np.testing.assert_allclose(yf, ref, rtol=1e-11, atol=1e-13)


# ---------------------------------------------------------------- whole block
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("seed", list(range(5)))
def test_block_vs_dense_bruteforce(dtype, seed):
    """Steps 2-6 vs a numpy brute force that evaluates every expert densely (C1)."""
    inp = _tiny(seed, dtype)
    y = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=2)
    ref, _ = _np_dense_block(inp, 2)
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-13)


def test_block_k1_and_k3():
    for k in (1, 3):
        inp = _tiny(11, "f32")
        y = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=k)
        ref, _ = _np_dense_block(inp, k)
        np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-13)


def test_forced_routing():
    """Step 8: forced S -> y = sum_j w_j(S) o_{S_j}, gates renormalised over S."""
    inp = _tiny(5, "f32")
    x, wg, w1, w3, w2 = (_dec(inp[n]) for n in ("x", "wg", "w1", "w3", "w2"))
    T = x.shape[0]
    rng = np.random.default_rng(0)
    forced = np.stack([rng.choice(4, 2, replace=False) for _ in range(T)]).astype(np.int32)
    y = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=2,
                           forced_idx=forced)
    l = x @ wg.T
    for t in range(T):
        S = forced[t]
        p = np.exp(l[t, S] - l[t].max())
        w = p / p.sum()
        o = [(_np_silu(w1[e] @ x[t]) * (w3[e] @ x[t])) @ w2[e].T for e in S]
        np.testing.assert_allclose(y[t], w[0] * o[0] + w[1] * o[1], rtol=1e-11, atol=1e-13)


def test_residual_flag():
    """Reading R12 (C5 stack): residual adds x exactly."""
    inp = _tiny(6, "f32")
    args = (inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"])
    y = oracle.moe_forward(*args, k=2)
    yr = oracle.moe_forward(*args, k=2, residual=True)
    np.testing.assert_allclose(yr, y + inp["x"].astype(np.float64), rtol=0, atol=1e-15)


# ---------------------------------------------------------------- invariances
def test_token_permutation_equivariance_and_batch_independence():
    inp = _tiny(8, "bf16")
    args = lambda x: (x, inp["wg"], inp["w1"], inp["w3"], inp["w2"])
    y = oracle.moe_forward(*args(inp["x"]), k=2)
    perm = np.random.default_rng(1).permutation(inp["x"].shape[0])
    yp = oracle.moe_forward(*args(inp["x"][perm]), k=2)
    np.testing.assert_array_equal(yp, y[perm])          # exact: same per-token arithmetic
    y1 = oracle.moe_forward(*args(inp["x"][5:6]), k=2)  # T=1 batch
    np.testing.assert_array_equal(y1[0], y[5])
    ysub = oracle.moe_forward(*args(inp["x"]), k=2, tokens=[7, 2, 7])
    np.testing.assert_array_equal(ysub, y[[7, 2, 7]])


def test_expert_relabelling_invariance():
    inp = _tiny(9, "f32")
    y = oracle.moe_forward(inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"], k=2)
    pi = np.array([2, 0, 3, 1])
    y2 = oracle.moe_forward(inp["x"], inp["wg"][pi], inp["w1"][pi], inp["w3"][pi], inp["w2"][pi], k=2)
    np.testing.assert_allclose(y2, y, rtol=1e-13, atol=1e-15)


# ---------------------------------------------------------------- partitions (step 9)
@pytest.mark.parametrize("mode,G", [("ep", 2), ("ep", 4), ("tp", 2), ("tp", 4), ("tp", 8)])
def test_partition_sums_to_full(mode, G):
    inp = _tiny(10, "bf16")
    args = (inp["x"], inp["wg"], inp["w1"], inp["w3"], inp["w2"])
    y = oracle.moe_forward(*args, k=2)
    P = oracle.partition(*args, k=2, G=G, mode=mode)
    np.testing.assert_allclose(P.sum(0), y, rtol=1e-12, atol=1e-14)
    if mode == "ep":  # each token's output lives on at most k ranks
        nz = (np.abs(P).sum(2) > 0).sum(0)
        assert np.all(nz <= 2)


@pytest.mark.parametrize("G,dead", [(2, [2, 3]), (2, [0, 1]), (4, [1, 3])])
def test_partition_ep_ownership(G, dead):
    """EP rank r owns experts [r*E/G, (r+1)*E/G): with x > 0 and the router rows of the
    `dead` experts negated (their logits < 0 < the others', so top-2 never picks them),
    the ranks owning only dead experts hold exactly zero and the rest sum to y."""
    inp = _tiny(11, "f32")
    x = np.abs(inp["x"])
    wg = np.abs(inp["wg"])
    wg[dead] *= -1
    args = (x, wg, inp["w1"], inp["w3"], inp["w2"])
    P = oracle.partition(*args, k=2, G=G, mode="ep")
    E = wg.shape[0]
    for r in range(G):
        owned = set(range(r * E // G, (r + 1) * E // G))
        if owned <= set(dead):
            assert np.all(P[r] == 0), r
        else:
            assert np.abs(P[r]).max() > 0, r
    np.testing.assert_allclose(P.sum(0), oracle.moe_forward(*args, k=2), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("G,dead_rank", [(2, 1), (2, 0), (4, 2)])
def test_partition_tp_ownership(G, dead_rank):
    """TP rank r owns ffn columns [r*f/G, (r+1)*f/G): with those W2 columns zeroed for
    dead_rank, its partial is exactly zero and the others still sum to y."""
    inp = _tiny(12, "f32")
    f = inp["w1"].shape[1]
    w2 = inp["w2"].copy()
    w2[:, :, dead_rank * f // G:(dead_rank + 1) * f // G] = 0
    args = (inp["x"], inp["wg"], inp["w1"], inp["w3"], w2)
    P = oracle.partition(*args, k=2, G=G, mode="tp")
    for r in range(G):
        assert (np.all(P[r] == 0)) == (r == dead_rank), r
    np.testing.assert_allclose(P.sum(0), oracle.moe_forward(*args, k=2), rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- permutation (step 7)
def _brute_perm(idx, E, align):
    T, k = idx.shape
    counts = [int(sum(1 for t in range(T) for j in range(k) if idx[t, j] == e)) for e in range(E)]
    offs = [0]
    for e in range(E):
        offs.append(offs[-1] + -(-counts[e] // align) * align)
    pos = np.zeros((T, k), np.int64)
    for t in range(T):
        for j in range(k):
            e = idx[t, j]
            earlier = sum(1 for t2 in range(t) if e in idx[t2])
            pos[t, j] = offs[e] + earlier
    return counts, offs, pos


@pytest.mark.parametrize("T,E,k,align", [(16, 4, 2, 128), (64, 8, 2, 16), (333, 8, 2, 128),
                                         (50, 8, 1, 128), (200, 4, 2, 1), (0, 8, 2, 128)])
def test_permutation_bruteforce_and_inverse(T, E, k, align):
    rng = np.random.default_rng(T + E)
    idx = np.array([rng.choice(E, k, replace=False) for _ in range(T)], np.int32).reshape(T, k)
    r = oracle.permutation(idx, E, align)
    counts, offs, pos = _brute_perm(idx, E, align)
    assert list(r["counts"]) == counts and list(r["offsets"]) == offs
    np.testing.assert_array_equal(r["pos"], pos)
    assert r["counts"].sum() == T * k
    # permute then un-permute is the identity (bit-exact), positions are unique
    x = rng.integers(0, 2**16, size=(T, 8), dtype=np.uint16)
    buf = np.zeros((max(int(r["offsets"][-1]), 1), 8), np.uint16)
    flat = r["pos"].reshape(-1)
    assert len(set(flat.tolist())) == T * k
    for t in range(T):
        for j in range(k):
            buf[r["pos"][t, j]] = x[t]
    for j in range(k):
        np.testing.assert_array_equal(buf[r["pos"][:, j]], x)
    # each segment is stable (increasing token index) and inside its expert's range
    for e in range(E):
        lo, hi = r["offsets"][e], r["offsets"][e] + r["counts"][e]
        toks = [t for p in range(lo, hi) for t in range(T) for j in range(k) if r["pos"][t, j] == p]
        assert toks == sorted(toks) and all(idx[t].tolist().count(e) == 1 for t in toks)


def test_permutation_pathological():
    """All tokens to one expert pair; 127/128/129-row segments."""
    for n in (127, 128, 129):
        idx = np.array([[0, 1]] * n, np.int32)
        r = oracle.permutation(idx, 4, 128)
        assert list(r["counts"]) == [n, n, 0, 0]
        seg = -(-n // 128) * 128
        assert list(r["offsets"]) == [0, seg, 2 * seg, 2 * seg, 2 * seg]
        np.testing.assert_array_equal(r["pos"][:, 0], np.arange(n))
        np.testing.assert_array_equal(r["pos"][:, 1], seg + np.arange(n))
    with pytest.raises(ValueError):
        oracle.permutation(np.array([[1, 1]], np.int32), 4, 128)   # duplicate expert
    with pytest.raises(ValueError):
        oracle.permutation(np.array([[0, 4]], np.int32), 4, 128)   # out of range


def test_bf16_helpers():
    """The oracle's bf16 decode / RNE helpers vs torch's conversion (library routine)."""
    v = torch.randn(10000, dtype=torch.float32) * 3
    v[:4] = torch.tensor([1.0, 1.00390625, 1.01171875, -2.5])  # exact halfway cases
    bits = synth.bf16_bits(v.to(torch.bfloat16))
    np.testing.assert_array_equal(oracle.bf16_to_f64(bits), v.to(torch.bfloat16).double().numpy())
    np.testing.assert_array_equal(oracle.bf16_round(v.numpy()), v.to(torch.bfloat16).double().numpy())


def test_bf16_round_fp64_single_rounding():
    """bf16_round on fp64 inputs rounds ONCE (no fp64 -> fp32 -> bf16 double rounding).
    Pins: hand-derived cases where double rounding is wrong, and brute-force RNE in
    exact rational arithmetic (fractions.Fraction) over random fp64 values incl.
    subnormal-range and overflow edges."""
    from fractions import Fraction
    # 1 + 2^-8 is the midpoint of the bf16 neighbours 1 and 1 + 2^-7; a hair above it must
    # round UP, although fp32(1 + 2^-8 + 2^-30) is the midpoint itself (which rounds to even = 1)
    cases = {1 + 2.0 ** -8 + 2.0 ** -30: 1 + 2.0 ** -7, 1 + 2.0 ** -8 - 2.0 ** -30: 1.0,
             1 + 2.0 ** -8: 1.0, 1 + 3 * 2.0 ** -8: 1 + 2.0 ** -6, -(1 + 2.0 ** -8 + 2.0 ** -40): -(1 + 2.0 ** -7),
             2.0 ** 128: np.inf, 3.3895313892515355e38: 3.3895313892515355e38, 0.0: 0.0}
    got = oracle.bf16_round(np.array(list(cases)))
    np.testing.assert_array_equal(got, np.array(list(cases.values())))

    def rne_exact(x):
        if x == 0:
            return 0.0
        fx = Fraction(x)
        s = -1 if fx < 0 else 1
        fx = abs(fx)
        e = 0
        while fx >= 2 ** (e + 1):
            e += 1
        while fx < 2 ** e:
            e -= 1
        e = max(e, -126)                      # bf16 subnormals share the spacing 2^-133
        ulp = Fraction(2) ** (e - 7)
        q, rem = divmod(fx, ulp)
        if rem * 2 > ulp or (rem * 2 == ulp and q % 2 == 1):
            q += 1
        v = q * ulp
        return s * (np.inf if v >= 2 ** 128 else float(v))

    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.standard_normal(300) * 10.0 ** rng.integers(-5, 5, 300),
                         rng.standard_normal(50) * 2.0 ** -130, rng.standard_normal(20) * 3e38])
    np.testing.assert_array_equal(oracle.bf16_round(xs), np.array([rne_exact(float(x)) for x in xs]))
