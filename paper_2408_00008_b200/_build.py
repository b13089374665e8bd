"""Build libmoe.so in-tree with nvcc for sm_100a (the .so travels to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmoe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-shared",
]


def nccl_include():
    """NCCL 2.28's headers (device API: symmetric windows, LSA barriers, multimem) shipped
    with the nvidia-nccl wheel torch uses; None if absent (nvls.cu then builds a stub)."""
    try:
        import nvidia
        for base in nvidia.__path__:
            inc = os.path.join(base, "nccl", "include")
            if os.path.exists(os.path.join(inc, "nccl_device.h")):
                return inc
    except ImportError:
        pass
    return None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(ROOT, "include", "moe.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libmoe.so; `out` / `defines` build experiment variants (A/B timing)."""
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    inc = nccl_include()
    nccl_flags = ["-I", inc, "-DMOE_HAVE_NCCL_DEVICE"] if inc else []
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), *nccl_flags,
           "-o", tmp, os.path.join(CSRC, "moe.cu"), os.path.join(CSRC, "nvls.cu"), "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python _build.py [--force] [--out PATH] [-DNAME=VAL ...]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv or out is not None, verbose=out is None, out=out, defines=defs))
