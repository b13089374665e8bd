python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for b in M0 M1 M2 cycle; do
  timeout -s KILL 900 python bench.py --config stack --stack-batch $b --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/stack_$b.log 2>&1
  grep "^{" gpurun_out/stack_$b.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$b', round(j['ms_per_step'],3), round(j['value']), 'hbm', round(j['step_roofline_frac'],3), 'tensor', round(j['step_tensor_frac'],3), j['forwards_per_step'], j['kernel_ms_per_launch'])" || tail -5 gpurun_out/stack_$b.log
done
