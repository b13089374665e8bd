# shard sweeps: small per-rank decode shapes and the T=575 stack layer
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { timeout -s KILL 200 python bench.py --steps 50 --warmup 5 "$@" 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); k=j['kernels']; key='frac_hbm' if j['config']!='prefill' else 'frac_sustained'
    print('$*', round(j['ms_per_step']*1000,1), 'us', {n:(round(v[key],3), round(v['ms']*1000,1)) for n,v in k.items()}, 'step', round(j.get('step_frac_hbm', j.get('step_frac_sustained')),3))
"; }
for s in tp1 ep2 tp2 ep4 tp4 ep8 tp8; do run --shard $s --config decode; done
for s in tp1 tp2 tp4 tp8; do run --shard $s --config stack; done
for sk in 1 2 4; do run --shard ep8 --config decode --split-k $sk; run --shard tp8 --config decode --split-k $sk; run --shard tp4 --config decode --split-k $sk; run --shard ep4 --config decode --split-k $sk; done
for g in 56 74 96 112 128 148; do run --shard ep8 --config decode --tuning g2_grid=$g; run --shard tp8 --config decode --tuning g2_grid=$g; done
for g in 74 96 112 128 148; do run --shard ep8 --config decode --tuning g1_grid=$g; run --shard tp8 --config decode --tuning g1_grid=$g; done
for sk in 1 2 4; do run --shard tp1 --config stack --split-k $sk; run --shard tp8 --config stack --split-k $sk; done
