# A/B timing of environment-variable sets (several variables per set, joined by ','), interleaved.
# usage: bash scripts/ab_env2.sh "A=1,B=2 A=3" [rounds] [extra bench args]
SETS=$1; R=${2:-3}; shift 2
for r in $(seq 1 $R); do for v in $SETS; do
  env ${v//,/ } timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/abenv.log 2>&1
  grep -h "^{" gpurun_out/abenv.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$v', $r, round(j['ms_per_step'],4), round(j['value']), round(j['roofline']['frac'],4), round(j['e2e']['value']), j['kernel_ms'])
" || tail -5 gpurun_out/abenv.log
done; done
