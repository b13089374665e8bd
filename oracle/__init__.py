"""fp64 CPU oracle for the MoE block -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path never does; it
shares no code with it (see moe_oracle.cpp's header for the definition and
the PAPER.md / BASELINE.json passages it follows).

Thin ctypes marshalling over liboracle.so (built from moe_oracle.cpp by
`build()`): numpy arrays in, numpy arrays out. Inputs may be bf16 bit patterns
(numpy uint16), float32 or float64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "moe_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (portable flags: the .so travels to the GPU box)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call([
            "g++", "-O3", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
            "-ffp-contract=off", "-fno-fast-math", "-Wall", "-o", tmp, _SRC,
        ])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        override = os.environ.get("ORACLE_LIB")  # tests/test_oracle_mutations.py: a mutated build
        if not override:
            build()
        lib = ctypes.CDLL(override or _LIB_PATH)
        P = ctypes.c_void_p
        I, L = ctypes.c_int, ctypes.c_int64
        lib.oracle_router.argtypes = [I, P, P, L, I, I, I, P, P, P, P, P]
        lib.oracle_moe_forward.argtypes = [I, P, P, P, P, P, L, I, I, I, I, P, P, L, I, P]
        lib.oracle_partition.argtypes = [I, P, P, P, P, P, L, I, I, I, I, I, I, P, L, P]
        lib.oracle_permutation.argtypes = [P, L, I, I, I, P, P, P]
        lib.oracle_set_threads.argtypes = [I]
        for fn in (lib.oracle_router, lib.oracle_moe_forward, lib.oracle_partition,
                   lib.oracle_permutation, lib.oracle_set_threads):
            fn.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dtype_code(*arrs):
    dts = {a.dtype for a in arrs}
    if len(dts) != 1:
        raise TypeError(f"mixed input dtypes {dts}")
    dt = dts.pop()
    if dt == np.uint16:
        return 0
    if dt == np.float32:
        return 1
    if dt == np.float64:
        return 2
    raise TypeError(f"unsupported dtype {dt}")


def _c(a):
    return np.ascontiguousarray(a)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def router(x, wg, k):
    """Steps 2-4: fp64 logits [T,E], top-k idx [T,k] int32, gates [T,k] fp64,
    margins m12 = l(1)-l(2), m23 = l(2)-l(3) [T]."""
    x, wg = _c(x), _c(wg)
    T, d = x.shape
    E = wg.shape[0]
    logits = np.empty((T, E), np.float64)
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float64)
    m12 = np.empty(T, np.float64)
    m23 = np.empty(T, np.float64)
    rc = _load().oracle_router(_dtype_code(x, wg), _ptr(x), _ptr(wg), T, d, E, k,
                               _ptr(logits), _ptr(idx), _ptr(w), _ptr(m12), _ptr(m23))
    if rc:
        raise ValueError(f"oracle_router rc={rc}")
    return {"logits": logits, "idx": idx, "w": w, "m12": m12, "m23": m23}


def moe_forward(x, wg, w1, w3, w2, k, forced_idx=None, tokens=None, residual=False):
    """Steps 2-6 (step 8 with forced_idx): y [n, d] fp64 for the listed tokens (all by default)."""
    x, wg, w1, w3, w2 = map(_c, (x, wg, w1, w3, w2))
    T, d = x.shape
    E, f, _ = w1.shape
    fi = None if forced_idx is None else _c(np.asarray(forced_idx, np.int32))
    if fi is not None and fi.shape != (T, k):
        raise ValueError("forced_idx must be [T,k]")
    tl = None if tokens is None else _c(np.asarray(tokens, np.int64))
    n = T if tl is None else len(tl)
    y = np.empty((n, d), np.float64)
    rc = _load().oracle_moe_forward(_dtype_code(x, wg, w1, w3, w2), _ptr(x), _ptr(wg), _ptr(w1),
                                    _ptr(w3), _ptr(w2), T, d, f, E, k, _ptr(fi), _ptr(tl), n,
                                    int(bool(residual)), _ptr(y))
    if rc:
        raise ValueError(f"oracle_moe_forward rc={rc}")
    return y


def partition(x, wg, w1, w3, w2, k, G, mode, tokens=None):
    """Step 9: per-rank partial outputs [G, n, d] for mode 'ep' or 'tp'."""
    x, wg, w1, w3, w2 = map(_c, (x, wg, w1, w3, w2))
    T, d = x.shape
    E, f, _ = w1.shape
    tl = None if tokens is None else _c(np.asarray(tokens, np.int64))
    n = T if tl is None else len(tl)
    out = np.empty((G, n, d), np.float64)
    m = {"ep": 1, "tp": 2}[mode]
    rc = _load().oracle_partition(_dtype_code(x, wg, w1, w3, w2), _ptr(x), _ptr(wg), _ptr(w1),
                                  _ptr(w3), _ptr(w2), T, d, f, E, k, G, m, _ptr(tl), n, _ptr(out))
    if rc:
        raise ValueError(f"oracle_partition rc={rc}")
    return out


def permutation(idx, E, align):
    """Step 7: counts [E] int32, offsets [E+1] int64, pos [T,k] int64 (stable by token)."""
    idx = _c(np.asarray(idx, np.int32))
    T, k = idx.shape
    counts = np.empty(E, np.int32)
    offsets = np.empty(E + 1, np.int64)
    pos = np.empty((T, k), np.int64)
    rc = _load().oracle_permutation(_ptr(idx), T, k, E, align, _ptr(counts), _ptr(offsets), _ptr(pos))
    if rc:
        raise ValueError(f"oracle_permutation rc={rc}")
    return {"counts": counts, "offsets": offsets, "pos": pos}


def set_threads(n):
    """OpenMP threads of the oracle's parallel loops (n <= 0: unchanged); returns the
    previous maximum. Timing only (bench.py cpu_baseline): results do not depend on it."""
    return int(_load().oracle_set_threads(int(n)))


def bf16_round(a):
    """Round fp32/fp64 values to bf16 (RNE, one rounding straight from the input's own
    precision -- no intermediate fp32 step) and return fp64 -- used to form the bf16
    rounding floor of the expected output (reading R8). bf16 keeps 8
    significant bits and the fp32 exponent range: a = q * 2^(e-8) with q in [128, 256)
    for normals (e from frexp, clamped at the subnormal exponent -125), q rounded to an
    integer half-to-even (np.rint), magnitudes >= 2^128 -> inf."""
    a = np.asarray(a, np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        _, e = np.frexp(a)
        e = np.maximum(e, -125)
        q = np.ldexp(a, 8 - e)                  # exact: a power-of-two scaling
        r = np.ldexp(np.rint(q), e - 8)
        r = np.where(np.abs(r) >= 2.0 ** 128, np.copysign(np.inf, a), r)
        r = np.where(np.isfinite(a), r, a)      # inf / nan pass through
    return r


def bf16_to_f64(bits):
    """Decode bf16 bit patterns (uint16) to fp64."""
    b = np.asarray(bits, np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)
