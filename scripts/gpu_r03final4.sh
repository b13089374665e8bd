# final evidence after the host-output in-kernel combine: GPU suite, smoke, decode / FP8 lines
O=gpurun_out/r03final4; mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest $?"; tail -n 1 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke $?"
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > $O/bench_decode.json 2> $O/bench_decode.err; echo "bench $?"
timeout -s KILL 400 python bench.py --fp8 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_decode_fp8.json 2> $O/bench_decode_fp8.err; echo "fp8 $?"
for f in bench_decode bench_decode_fp8; do python -c "
import json; j=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', round(j['value']), round(j['ms_per_step'],4), round(j['roofline']['frac'],3), round(j['e2e']['value']), j['clocks']['sm_mhz'], j['clocks']['reasons'])"; done
