# prefill L2 policy sweep (tuning.pair_hints): DRAM bytes per launch (ncu) and step time (interleaved)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
HINTS="0 2 6 32 128 130 16"
for o in $HINTS; do
  timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:moe_gemm_pair -s 2 -c 2 --csv python bench.py --tuning pair_hints=$o --config prefill --steps 1 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | grep -E '"(dram|gpu__time)' | awk -F'","' -v o=$o '{print o, $5, $(NF-2), $NF}'
done > gpurun_out/prefill_hint_ncu.log
for r in 1 2 3; do for o in $HINTS; do
  timeout -s KILL 300 python bench.py --tuning pair_hints=$o --config prefill --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$o', $r, round(j['ms_per_step'],3), j['kernel_ms'], j['clocks']['sm_mhz'])"
done; done > gpurun_out/prefill_hint_time.log
cat gpurun_out/prefill_hint_ncu.log gpurun_out/prefill_hint_time.log
