# honest C5 stack (W2 x0.25): M1 path / tile variants, interleaved
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2 3; do for t in "" "--tuning g1_grid=148" "--tuning g2_grid=148" "--tuning g1_grid=148,g2_grid=148" "--tuning g1_grid=128"; do
  timeout -s KILL 600 python bench.py --config stack --stack-batch M1 --steps 5 --warmup 3 --no-cpu-baseline $t 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('[$t]', $r, round(j['ms_per_step'],3), round(j['value']), 'hbm', round(j['step_roofline_frac'],3), {k: round(v*1000,1) for k,v in j['kernel_ms_per_launch'].items()}, j['clocks']['sm_mhz'])"
done; done
