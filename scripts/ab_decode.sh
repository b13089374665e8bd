# A/B timing of libmoe build variants (build_ab/libmoe_<v>.so) on the decode bench, interleaved.
# usage: bash scripts/ab_decode.sh "<v1> <v2> ..." [rounds] [extra bench args]
VARS=$1; R=${2:-3}; shift 2
for r in $(seq 1 $R); do for v in $VARS; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/ab_${v}_${r}.log 2>&1
  grep -h "^{" gpurun_out/ab_${v}_${r}.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$v', $r, round(j['ms_per_step'],4), round(j['value']), round(j['step_roofline_frac'],4))
"
done; done
