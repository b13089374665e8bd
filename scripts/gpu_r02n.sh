python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x -rs -s > gpurun_out/pytest_n.log 2>&1; echo rc=$? >> gpurun_out/pytest_n.log
grep -E "^C2|^C3|^stack|^tp stack|skewed|^EP|^ep |^tp |fp8 |NVLS|passed|failed|rc=" gpurun_out/pytest_n.log | tail -40
b() { timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline "$@" 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('$*', round(j['ms_per_step'],4), round(j['value']), j.get('graph_replay'), j.get('parity',{}).get('ok'), j.get('expert_rows'), j['config'].get('routing'))
" || echo "FAILED $*"; }
b --skew
b --config stack --skew --steps 5
b --par ep
b --par tp
b --par ep --p2p
b --par tp --p2p
b --par ep --flags 0x20
