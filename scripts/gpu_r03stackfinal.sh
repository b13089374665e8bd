# stack lines + decode shard lines on the final build (the M0 layers and the TP2 / EP2 ranks run the fused decode FFN)
O=gpurun_out/r03stackfinal; mkdir -p $O
timeout -s KILL 900 python bench.py --config stack --steps 10 --warmup 3 > $O/bench_stack.json 2> $O/bench_stack.err; echo "M1 $?"
for b in M0 cycle; do timeout -s KILL 900 python bench.py --config stack --stack-batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_stack_$b.json 2> $O/bench_stack_$b.err; echo "$b $?"; done
for s in ep2 ep4 ep8 tp2 tp4 tp8; do
  timeout -s KILL 300 python bench.py --shard $s --config decode --steps 30 --warmup 3 2>&1 | grep "^{" >> $O/shards.jsonl
done
for f in bench_stack bench_stack_M0 bench_stack_cycle; do python -c "
import json; j=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', round(j['value']), j['ms_per_step'], j.get('roofline',{}).get('frac'), j['clocks']['sm_mhz'])"; done
python -c "
import json
for l in open('$O/shards.jsonl'):
    j=json.loads(l); print(j['shard'], round(j['ms_per_step']*1000,1), {k:(round(v['ms']*1000,1), round(v['frac_hbm'],3)) for k,v in j['kernels'].items()}, round(j['step_frac_hbm'],3))"
