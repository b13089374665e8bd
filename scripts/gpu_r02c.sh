# stack-shape token tiles: NB 192 (new auto) vs the old 128 / 256, splits
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { timeout -s KILL 200 python bench.py --steps 50 --warmup 5 "$@" 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); k=j['kernels']; key='frac_hbm' if j['config']!='prefill' else 'frac_sustained'
    print('$*', round(j['ms_per_step']*1000,1), 'us', {n:(round(v[key],3), round(v['ms']*1000,1)) for n,v in k.items()}, 'step', round(j.get('step_frac_hbm', j.get('step_frac_sustained')),3))
"; }
for r in 1 2; do
for s in tp1 tp8; do
  run --shard $s --config stack
  run --shard $s --config stack --split-k 1
  run --shard $s --config stack --tuning g1_nb=128,g2_nb=256
  run --shard $s --config stack --tuning g1_nb=128
  run --shard $s --config stack --tuning g2_nb=256
  run --shard $s --config stack --tuning g1_grid=148
done; done
for s in tp1 ep8 tp8; do run --shard $s --config decode; done
timeout -s KILL 600 python bench.py --config stack --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_stack_c.log 2>&1
timeout -s KILL 600 python bench.py --config stack --steps 10 --warmup 3 --no-cpu-baseline --no-parity --split-k 1 > gpurun_out/bench_stack_c1.log 2>&1
grep -h "^{" gpurun_out/bench_stack_c*.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('stack32', j['ms_per_step'], j['value'], j['step_roofline_frac'], j['kernel_ms_per_launch'], j['clocks'])"
