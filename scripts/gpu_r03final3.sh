# final evidence refresh after the geometric taper: GPU suite, smoke, decode / FP8 lines, decode launch list
O=gpurun_out/r03final3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build $?"
timeout -s KILL 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest $?"; tail -n 1 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke $?"
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > $O/bench_decode.json 2> $O/bench_decode.err; echo "bench $?"
timeout -s KILL 400 python bench.py --fp8 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_decode_fp8.json 2> $O/bench_decode_fp8.err; echo "fp8 $?"
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_decode_b.json 2> $O/bench_decode_b.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_decode.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1; echo "ncu $?"
for f in bench_decode bench_decode_fp8 bench_decode_b; do python -c "
import json; j=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', round(j['value']), j['ms_per_step'], j['roofline']['frac'], j['e2e']['value'], j['clocks']['sm_mhz'], j['clocks']['reasons'])"; done
