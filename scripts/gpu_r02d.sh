# FP8 block-scaled path: parity first, then the FP8 decode bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "fp8" -s > gpurun_out/pytest_fp8.log 2>&1; echo rc=$? >> gpurun_out/pytest_fp8.log
tail -40 gpurun_out/pytest_fp8.log
timeout -s KILL 300 python bench.py --fp8 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fp8_d.log 2>&1
grep "^{" gpurun_out/bench_fp8_d.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('fp8', j['ms_per_step'], j['value'], j['roofline']['frac'], j['kernel_ms'], j['step_roofline_frac'])"
tail -3 gpurun_out/bench_fp8_d.log
