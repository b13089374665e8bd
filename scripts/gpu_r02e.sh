python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "fp8" -s > gpurun_out/pytest_fp8e.log 2>&1; echo rc=$? >> gpurun_out/pytest_fp8e.log
tail -3 gpurun_out/pytest_fp8e.log
timeout -s KILL 300 python bench.py --fp8 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fp8_e.log 2>&1
grep "^{" gpurun_out/bench_fp8_e.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('fp8', j['ms_per_step'], j['value'], j['roofline']['frac'], j['kernel_ms'], j['step_roofline_frac'])"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_fp8x" -s 4 -c 2 -o gpurun_out/prof_fp8_e python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/ncu_fp8_e.log 2>&1
tail -3 gpurun_out/ncu_fp8_e.log
