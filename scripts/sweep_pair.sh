# sweep raster / L2-hint settings of the CTA-pair prefill GEMMs (moe_tuning.pair_order bits, include/moe.h)
for t in "$@"; do
  timeout -s KILL 300 python bench.py --tuning pair_order=$t --config prefill --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$t.log 2>&1
  python - "$t" <<'PY'
import json,sys
t=sys.argv[1]
l=[x for x in open(f"gpurun_out/sweep_{t}.log") if x.startswith("{")]
if not l: print(t, "FAILED"); sys.exit()
j=json.loads(l[-1]); print("tune", t, "ms", round(j["ms_per_step"],3), "g1", j["kernel_ms"]["gemm1_w13_swiglu"], "g2", j["kernel_ms"]["gemm2_w2"], "clk", j["clocks"]["sm_mhz"])
PY
done
