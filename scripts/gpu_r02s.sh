# pair swap kernels: stage-depth sensitivity on the C5 stack M1 + one ncu --set full capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do for v in s3 s4 s8; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 600 python bench.py --config stack --stack-batch M1 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$v', $r, round(j['ms_per_step'],3), round(j['value']), 'hbm', round(j['step_roofline_frac'],3), {k: round(v*1000,1) for k,v in j['kernel_ms_per_launch'].items()}, j['clocks']['sm_mhz'])"
done; done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_swap_pair" -s 4 -c 2 -o gpurun_out/prof_stack_spair python bench.py --shard tp1 --config stack --steps 1 --warmup 3 > gpurun_out/ncu_spair.log 2>&1
tail -3 gpurun_out/ncu_spair.log
