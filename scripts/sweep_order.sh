# DRAM traffic + time of the prefill pair GEMMs per tile order (moe_tuning.pair_order, include/moe.h)
for t in "$@"; do
  timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:moe_gemm_pair -s 2 -c 2 --csv python bench.py --tuning pair_order=$t --config prefill --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E '"(dram|gpu__time|sm__pipe)' | awk -F'","' -v t=$t '{print t, $5, $(NF-2), $NF}'
done
