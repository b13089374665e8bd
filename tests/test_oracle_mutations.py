"""Mutation check of the oracle's pins (CPU, -m "not gpu").

A pin is only worth something if a plausible mistake in the oracle breaks it.
This test recompiles oracle/moe_oracle.cpp with one deliberate mistake at a time
(a flipped sign, a dropped term, a transposed operand, a wrong tie-break, an
off-by-one index) into a temporary library, runs the oracle's pin tests
(tests/test_oracle.py) against it in a subprocess, and requires every mutant
to be killed (at least one pin fails).
"""
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "moe_oracle.cpp")

# (name, original snippet, mutated snippet)
MUTANTS = [
    ("silu sign", "return z / (1.0 + std::exp(-z));", "return z / (1.0 + std::exp(z));"),
    ("no renormalisation", "w[j] = p[S[j]] / s;", "w[j] = p[S[j]];"),
    ("W2 transposed", "dec(w2, ((size_t)e * d + r) * f + i)", "dec(w2, ((size_t)e * f + i) * d + r)"),
    ("tie-break reversed", "return a < b;", "return a > b;"),
    ("position off by one", "offsets[e] + seen[e]", "offsets[e] + seen[e] + (t > 0)"),
    ("w1/w3 swapped", "h[i] = silu(a) * b;", "h[i] = silu(b) * a;"),
    ("router drops last column", "for (int c = 0; c < d; ++c)\n            s += dec(x", "for (int c = 0; c < d - 1; ++c)\n            s += dec(x"),
    ("softmax without max shift", "p[e] = std::exp(l[e] - lmax);", "p[e] = std::exp(l[e] - lmax) + 1e-3;"),
    ("residual dropped", "acc[r] += dec(x, (size_t)t * d + r);", "acc[r] += 0.0;"),
    ("segment not padded", "offsets[e + 1] = offsets[e] + ((int64_t)(counts[e] + align - 1) / align) * align;",
     "offsets[e + 1] = offsets[e] + counts[e];"),
    ("logits sorted ascending", "if (l[a] != l[b]) return l[a] > l[b];", "if (l[a] != l[b]) return l[a] < l[b];"),
    ("gates paired with the wrong expert", "acc[r] += wt[j] * o[r];", "acc[r] += wt[k - 1 - j] * o[r];"),
    ("w3 read as w1", "b += dec(w3, ((size_t)e * f + i) * d + c) * xc;",
     "b += dec(w1, ((size_t)e * f + i) * d + c) * xc;"),
    ("EP experts owned round-robin", "if (e / (E / G) != r) continue;", "if (e % G != r) continue;"),
    ("TP ffn slices reversed", "r * (f / G), (r + 1) * (f / G)", "(G - 1 - r) * (f / G), (G - r) * (f / G)"),
]


@pytest.mark.parametrize("name,orig,mut", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_mutant_is_killed(name, orig, mut, tmp_path):
    src = open(SRC).read()
    assert orig in src, f"mutation anchor for '{name}' not found: the oracle changed, update the mutant"
    msrc = tmp_path / "moe_oracle_mut.cpp"
    msrc.write_text(src.replace(orig, mut, 1))
    lib = tmp_path / "liboracle_mut.so"
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-o", str(lib), str(msrc)])
    env = dict(os.environ, ORACLE_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant '{name}' survived every pin:\n{r.stdout[-2000:]}"
