# pair swap kernel timing probes (wrong results by design) on one T=575 stack layer:
# p0 = product, p1 = no MMAs, p2 = no token loads, p3 = no h/y stores
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2 3; do for v in p0 p1 p2 p3; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python bench.py --shard tp1 --config stack --steps 50 --warmup 5 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$v', $r, round(j['ms_per_step']*1000,1), {k: round(v*1000,1) for k,v in j['kernel_ms'].items()})"
done; done
