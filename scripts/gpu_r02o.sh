python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2 3; do for t in "" "g2_nb=32" "g1_nb=32" "g1_nb=32,g2_nb=32"; do
  timeout -s KILL 200 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-parity ${t:+--tuning $t} 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('[$t]', $r, round(j['ms_per_step']*1000,2), {k: round(v*1000,1) for k,v in j['kernel_ms'].items()}, j['clocks']['sm_mhz'])"
done; done
