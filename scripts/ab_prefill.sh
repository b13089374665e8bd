# A/B of libmoe build variants (build_ab/libmoe_<v>.so) on the prefill bench, interleaved,
# with the SM clock (prefill runs under sw_power_cap, so clock is part of the result).
# usage: bash scripts/ab_prefill.sh "<v1> <v2> ..." [rounds] [extra bench args]
VARS=$1; R=${2:-3}; shift 2
for r in $(seq 1 $R); do for v in $VARS; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python bench.py --config prefill --steps 20 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/abp_${v}_${r}.log 2>&1
  grep -h "^{" gpurun_out/abp_${v}_${r}.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); km=j['kernel_ms']
    print('$v', $r, round(j['ms_per_step'],3), round(j['value']), 'sm_mhz', j['clocks']['sm_mhz'], 'g1', round(km['gemm1_w13_swiglu'],3), 'g2', round(km['gemm2_w2'],3), 'frac', round(j['roofline']['frac'],4))
" || tail -3 gpurun_out/abp_${v}_${r}.log
done; done
