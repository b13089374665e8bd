"""CPU-side checks of the C-ABI boundary (no compute calls, no GPU needed):
libmoe.so loads, exports every symbol include/moe.h declares, validates
configurations, and fails loudly (no CPU fallback) without an sm_100 device."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "moe.h")).read()
    return sorted(set(re.findall(r"MOE_API\s+[\w\s\*]+?\b(moe_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2408_00008_b200 as moe
    syms = _header_symbols()
    assert len(syms) >= 16, syms
    lib = ctypes.CDLL(moe.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"libmoe.so does not export {s}"
    assert sorted(moe.EXPORTED) == syms


def test_no_torch_or_oracle_in_boundary():
    """The ABI header has no torch types; the product tree never references oracle/."""
    hdr = open(os.path.join(ROOT, "include", "moe.h")).read()
    assert "torch" not in hdr and "at::" not in hdr
    pkg = os.path.join(ROOT, "paper_2408_00008_b200")
    for dp, _, fns in os.walk(pkg):
        for fn in fns:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, fn)).read()
                assert "import oracle" not in txt and "moe_oracle" not in txt and "liboracle" not in txt, fn


def test_packed_sizes_and_validation():
    import paper_2408_00008_b200 as moe
    cfg = moe.make_config(4096, 14336, 8, 2, 64)
    a, b = moe.moe_packed_sizes(cfg)
    assert a == 8 * 2 * 14336 * 4096 * 2 and b == 8 * 4096 * 14336 * 2
    odd = moe.make_config(320, 1024, 4, 2, 64)  # W2 rows padded to a multiple of 256 (tiled layout)
    assert moe.moe_packed_sizes(odd) == (4 * 2 * 1024 * 320 * 2, 4 * 512 * 1024 * 2)
    tp = moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=8, rank=3, nccl_comm=1)
    a, b = moe.moe_packed_sizes(tp)
    assert a == 8 * 2 * 1792 * 4096 * 2 and b == 8 * 4096 * 1792 * 2
    ep = moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_EP, world_size=8, rank=3, nccl_comm=1)
    a, b = moe.moe_packed_sizes(ep)
    assert a == 1 * 2 * 14336 * 4096 * 2
    bad = [
        moe.make_config(100, 14336, 8, 2, 64),            # hidden % 64
        moe.make_config(4096, 1000, 8, 2, 64),            # ffn % 128
        moe.make_config(4096, 14336, 8, 3, 64),           # top_k
        moe.make_config(4096, 14336, 33, 2, 64),          # E > 32
        moe.make_config(4096, 14336, 8, 2, 0),            # max_tokens
        moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_EP, world_size=3, nccl_comm=1),  # E % G
        moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=8, nccl_comm=1, rank=8),
        moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=2),  # no comm
        moe.make_config(4096, 14336, 8, 2, 64, flags=moe.MOE_FLAG_FORCE_SWAP | moe.MOE_FLAG_FORCE_TILED),
    ]
    for c in bad:
        with pytest.raises(moe.MoEError) as ei:
            moe.moe_packed_sizes(c)
        assert ei.value.status == moe.MOE_ERR_INVALID


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_init_fails_loudly_without_gpu():
    import paper_2408_00008_b200 as moe
    with pytest.raises(moe.MoEError) as ei:
        moe.moe_init(moe.make_config(64, 128, 4, 2, 16))
    assert ei.value.status == moe.MOE_ERR_UNSUPPORTED


def test_tuning_validation():
    """moe_config.tuning (include/moe.h moe_tuning): out-of-range overrides and nonzero
    reserved fields are rejected before anything runs; valid ones pass validation."""
    import paper_2408_00008_b200 as moe
    ok = moe.make_config(4096, 14336, 8, 2, 64, tuning={"g1_grid": 112, "spec_l2": -1, "pair_nblk": 1,
                                                        "swap_nb_cap": 32, "weight_hint": 3})
    moe.moe_packed_sizes(ok)
    for bad in ({"pair_nblk": 3}, {"swap_pair": 3}, {"weight_hint": 4}, {"swap_nb_cap": 48}, {"g1_grid": -1}, {"g2_swap_rows": -5},
                {"fused": 3}, {"fused_splits": 9}, {"fused_stages": -1}, {"fused_combine": 3}, {"fused_chain": 2},
                {"fused_uniform": 5}):
        with pytest.raises(moe.MoEError) as ei:
            moe.moe_packed_sizes(moe.make_config(4096, 14336, 8, 2, 64, tuning=bad))
        assert ei.value.status == moe.MOE_ERR_INVALID, bad
    t = moe.make_tuning({"g1_grid": 1})
    t.reserved[len(t.reserved) - 1] = 1
    with pytest.raises(moe.MoEError):
        moe.moe_packed_sizes(moe.make_config(4096, 14336, 8, 2, 64, tuning=t))
    with pytest.raises(KeyError):
        moe.make_tuning({"no_such_knob": 1})
    # P2P groups are bounded by the one-warp signal kernel
    with pytest.raises(moe.MoEError) as ei:
        moe.moe_packed_sizes(moe.make_config(4096, 16384, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=64,
                                             flags=moe.MOE_FLAG_P2P))
    assert ei.value.status == moe.MOE_ERR_UNSUPPORTED


def test_struct_layout_matches_header(tmp_path):
    """The ctypes mirrors of moe_config / moe_tuning / moe_aux / moe_expert_weights have
    the size and field offsets a C compiler gives the header's structs."""
    import subprocess
    import paper_2408_00008_b200 as moe
    structs = {"moe_config": moe.moe_config, "moe_tuning": moe.moe_tuning, "moe_aux": moe.moe_aux,
               "moe_expert_weights": moe.moe_expert_weights}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "moe.h"', "int main(void) {"]
    for name, py in structs.items():
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{name} {fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-pedantic", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        n, f, v = ln.split()
        got[(n, f)] = int(v)
    for name, py in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(py), name
        for fname, _ in py._fields_:
            assert got[(name, fname)] == getattr(py, fname).offset, (name, fname)


def test_nvls_flag_validation():
    """MOE_FLAG_NVLS (TP all-reduce over NVLink SHARP) is a TP + NCCL-communicator option."""
    import paper_2408_00008_b200 as moe
    for bad in (moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_EP, world_size=2, nccl_comm=1,
                                flags=moe.MOE_FLAG_NVLS),
                moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=2, flags=moe.MOE_FLAG_NVLS),
                moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=2,
                                flags=moe.MOE_FLAG_NVLS | moe.MOE_FLAG_P2P),
                moe.make_config(4096, 14336, 8, 2, 64, flags=moe.MOE_FLAG_NVLS)):
        with pytest.raises(moe.MoEError) as ei:
            moe.moe_packed_sizes(bad)
        assert ei.value.status == moe.MOE_ERR_INVALID
    moe.moe_packed_sizes(moe.make_config(4096, 14336, 8, 2, 64, par=moe.MOE_PAR_TP, world_size=2, nccl_comm=1,
                                         flags=moe.MOE_FLAG_NVLS))
