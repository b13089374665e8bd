# A/B of environment settings on the prefill bench, interleaved, with the SM clock.
# usage: bash scripts/ab_env_prefill.sh "<VAR=a> <VAR=b> ..." [rounds] [extra bench args]
SETS=$1; R=${2:-3}; shift 2
for r in $(seq 1 $R); do for v in $SETS; do
  env $v timeout -s KILL 300 python bench.py --config prefill --steps 20 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/abpe.log 2>&1
  grep -h "^{" gpurun_out/abpe.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); km=j['kernel_ms']
    print('$v', $r, round(j['ms_per_step'],3), round(j['value']), 'sm_mhz', j['clocks']['sm_mhz'], 'g1', round(km['gemm1_w13_swiglu'],3), 'g2', round(km['gemm2_w2'],3), 'frac', round(j['roofline']['frac'],4))
" || tail -5 gpurun_out/abpe.log
done; done
