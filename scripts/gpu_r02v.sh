# pair swap w1/w3 with smem-staged h (bulk row copies, early TMEM release): parity + timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "swap_pair" > gpurun_out/pytest_spair.log 2>&1
tail -3 gpurun_out/pytest_spair.log
for r in 1 2; do
  timeout -s KILL 300 python bench.py --shard tp1 --config stack --steps 50 --warmup 5 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('shard', $r, round(j['ms_per_step']*1000,1), {k: round(v*1000,1) for k,v in j['kernel_ms'].items()})"
done
for r in 1 2 3; do for t in "--tuning swap_pair=1" ""; do
  timeout -s KILL 600 python bench.py --config stack --stack-batch M1 --steps 5 --warmup 3 --no-cpu-baseline $t 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('[$t]', $r, round(j['ms_per_step'],3), round(j['value']), 'hbm', round(j['step_roofline_frac'],3), {k: round(v*1000,1) for k,v in j['kernel_ms_per_launch'].items()}, j['clocks']['sm_mhz'])"
done; done
