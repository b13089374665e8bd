python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
(cd scripts/exp && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o small_stream small_stream.cu && ./small_stream) > gpurun_out/small_stream.log 2>&1
fp8() { timeout -s KILL 200 python bench.py --fp8 --steps 50 --warmup 5 --no-cpu-baseline "$@" 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('fp8 $*', round(j['ms_per_step']*1000,1), {k: round(v*1000,1) for k,v in j['kernel_ms'].items()}, round(j['step_roofline_frac'],3))
"; }
for sk in 0 1 2 4 8; do for g in 0 128 112; do fp8 --split-k $sk --tuning g2_grid=$g; done; done
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_g.log 2>&1; echo rc=$? >> gpurun_out/pytest_g.log
tail -3 gpurun_out/pytest_g.log
