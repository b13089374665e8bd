#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, on .ncu-rep files
brought back in gpurun_out/).

  python scripts/ncu_summary.py full <report.ncu-rep> [...]   -> key counters per kernel
  python scripts/ncu_summary.py launches <launches.csv>       -> per-launch device times + shares
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%active"),
    ("sm__inst_executed_pipe_tc.sum", "inst_tc"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__cycles_active.avg", "smsp_cycles_active"),
]


def full(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(p, "no data")
            continue
        hdr, units = rows[0], rows[1]
        print(f"## {p}")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            print(f"- kernel: `{name[:110]}`")
            for k, short in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    print(f"  - {short} ({k}): {r[i]} {units[i]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    ks = [(int(r[ii]), r[ki], float(r[vi])) for r in rows[hi + 1:] if len(r) > vi]
    mine = [k for k in ks if "moe::" in k[1] or "moe_" in k[1]]
    print(f"# {path}: {len(ks)} launches, {len(mine)} libmoe launches (ns, cold-cache, serialised)")
    agg = {}
    for _, n, v in mine:
        short = n.split("(")[0].replace("void ", "")
        agg.setdefault(short, []).append(v)
    # medians: the list also holds bench.py's e2e pass, whose combine stores into pinned
    # HOST memory (over PCIe) -- an outlier for the device-resident forward
    med = {k: sorted(v)[len(v) // 2] for k, v in agg.items() if "pack" not in k}
    tot = sum(med.values())
    print("| kernel | launches | median us | share of forward (medians) |")
    print("|---|---|---|---|")
    for k, m in sorted(med.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {len(agg[k])} | {m / 1000:.2f} | {m / tot:.3f} |")
    print()
    print("| ID | kernel | ns |")
    print("|---|---|---|")
    for i, n, v in mine:
        print(f"| {i} | `{n.split('(')[0]}` | {v:.0f} |")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2:])
    else:
        launches(sys.argv[2])
