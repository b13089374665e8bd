# final-HEAD check: full GPU suite, smoke, default decode bench line
O=gpurun_out/r03final2; mkdir -p $O
timeout -s KILL 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest $?"
tail -n 3 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke $?"
timeout -s KILL 600 python bench.py > $O/bench_decode.json 2> $O/bench_decode.err; echo "bench $?"
cat $O/bench_decode.json | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['roofline']['frac'], j['e2e']['value'], j['clocks'])"
