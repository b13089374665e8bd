# Per-rank shard shapes on one GPU (bench.py --shard), decode and prefill.
# usage: bash scripts/shard_sweep.sh <tag> [configs] [extra bench args]
TAG=${1:-run}; CONFS=${2:-"decode prefill"}; shift 2
for c in $CONFS; do for s in ${SHARDS:-ep2 ep4 ep8 tp2 tp4 tp8}; do
  st=20; [ $c = prefill ] && st=5
  timeout -s KILL 300 python bench.py --shard $s --config $c --steps $st --warmup 3 "$@" 2>&1 | grep "^{" >> gpurun_out/shard_${c}_$TAG.jsonl
done; done
python - "$TAG" <<'PY'
import json, sys, glob
for f in sorted(glob.glob(f"gpurun_out/shard_*_{sys.argv[1]}.jsonl")):
    for l in open(f):
        j = json.loads(l); k = j["kernels"]
        key = "frac_hbm" if j["config"] == "decode" else "frac_sustained"
        print(j["config"], j["shard"], round(j["ms_per_step"], 4), {n: round(v[key], 3) for n, v in k.items()},
              j.get("step_frac_hbm", j.get("step_frac_sustained")))
PY
