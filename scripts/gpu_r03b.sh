# fused FFN kernel: parity tests, then A/B bench fused vs two kernels (decode)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03b.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x -s > gpurun_out/pytest_fused_b.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_b.log
tail -5 gpurun_out/pytest_fused_b.log
if grep -q 'rc=0' gpurun_out/pytest_fused_b.log; then
for i in 1 2; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --tuning fused=1 > gpurun_out/bench_b_off_$i.log 2>&1
timeout -s KILL 300 python bench.py --no-cpu-baseline --tuning fused=2 > gpurun_out/bench_b_on_$i.log 2>&1
for s in 1 2 4; do timeout -s KILL 300 python bench.py --no-cpu-baseline --tuning fused=2,fused_splits=$s > gpurun_out/bench_b_on_s${s}_$i.log 2>&1; done
done
for f in gpurun_out/bench_b_*.log; do echo $f $(python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print(d.get('ms_per_step'), d.get('kernel_ms'), d.get('parity',{}).get('ok'))
"); done
fi
