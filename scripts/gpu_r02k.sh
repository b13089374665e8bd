# prefill tile-order sweep: DRAM bytes per launch (ncu) and step time (interleaved), K3 and K4 bands
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
# pair_order = r1 | r2<<2 | b1<<4 | b2<<10 (include/moe.h); default r1=2 b1=16 r2=3 b2=4 (wide)
ORDERS="4366 4622 5118 4878 2318 6414 8462 4364 8458"
for o in $ORDERS; do
  timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:moe_gemm_pair -s 2 -c 2 --csv python bench.py --tuning pair_order=$o --config prefill --steps 1 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | grep -E '"(dram|gpu__time)' | awk -F'","' -v o=$o '{print o, $5, $(NF-2), $NF}'
done > gpurun_out/prefill_order_ncu.log
for r in 1 2; do for o in $ORDERS; do
  timeout -s KILL 300 python bench.py --tuning pair_order=$o --config prefill --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$o', $r, round(j['ms_per_step'],3), j['kernel_ms'], j['clocks']['sm_mhz'])"
done; done > gpurun_out/prefill_order_time.log
cat gpurun_out/prefill_order_ncu.log gpurun_out/prefill_order_time.log
