python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { timeout -s KILL 200 python bench.py --steps 50 --warmup 5 "$@" 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); k=j['kernels']; key='frac_hbm' if j['config']!='prefill' else 'frac_sustained'
    print('$*', round(j['ms_per_step']*1000,1), 'us', {n:(round(v[key],3), round(v['ms']*1000,1)) for n,v in k.items()}, 'step', round(j.get('step_frac_hbm', j.get('step_frac_sustained')),3))
"; }
for r in 1 2; do
for s in ep8 tp8 ep4 tp4 ep2 tp2; do run --shard $s --config decode; run --shard $s --config decode --tuning xpf_mb=-1; done
run --shard tp8 --config stack; run --shard tp8 --config stack --tuning xpf_mb=-1
run --shard tp4 --config stack; run --shard tp4 --config stack --tuning xpf_mb=-1
done
for mb in 16 32 128; do run --shard ep8 --config decode --tuning xpf_mb=$mb; run --shard tp8 --config decode --tuning xpf_mb=$mb; done
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -rs -k "ep or tp or swap or decode or stack or nvls or c2" -s > gpurun_out/pytest_i.log 2>&1; echo rc=$? >> gpurun_out/pytest_i.log
grep -E "NVLS at world|passed|failed|rc=" gpurun_out/pytest_i.log | tail -5
