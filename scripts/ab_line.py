"""One-line summary of a bench.py JSON line (A/B sweeps): ms_per_step, kernel_ms, parity."""
import json
import sys

lines = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not lines:
    print("NO JSON:", open(sys.argv[1]).read()[-300:].replace("\n", " | "))
    sys.exit(0)
d = json.loads(lines[-1])
km = d.get("kernel_ms") or {}
kern = d.get("kernels")
if kern:  # bench.py --shard line
    print(f"ms={d['ms_per_step']:.4f} step_frac={d.get('step_frac_hbm', d.get('step_frac_sustained')):.3f} kernels="
          + str({k: (round(v['ms'] * 1e3, 1), round(v.get('frac_hbm', v.get('frac_sustained', 0)), 3))
                 for k, v in kern.items()}))
else:
    print(f"ms={d.get('ms_per_step'):.4f} value={d.get('value'):.0f} parity={d.get('parity', {}).get('ok')} "
          f"kernels={ {k: round(v * 1e3, 1) for k, v in km.items()} } sm={d.get('clocks', {}).get('sm_mhz')}")
