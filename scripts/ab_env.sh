# A/B timing of moe_tuning settings (bench.py --tuning) on one bench config, interleaved.
# usage: bash scripts/ab_env.sh "<field=a> <field=b,field2=c> ..." [rounds] [extra bench args]
SETS=$1; R=${2:-3}; shift 2
for r in $(seq 1 $R); do for v in $SETS; do
  timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --tuning "$v" "$@" > gpurun_out/abenv.log 2>&1
  grep -h "^{" gpurun_out/abenv.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$v', $r, round(j['ms_per_step'],4), round(j['value']), j['roofline']['frac'], j['e2e']['value'])
" || tail -5 gpurun_out/abenv.log
done; done
