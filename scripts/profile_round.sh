# Evidence for profiles/<tag>: bench JSON lines (decode, prefill, 32-layer stack, FP8, the
# reference arm), ncu launch lists (gpu__time_duration, clock-control none), one
# `ncu --set full` capture per GEMM family, per-rank shard sweeps and compute-sanitizer.
# usage (under gpurun, repo root): bash scripts/profile_round.sh <tag>
TAG=${1:-r02}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -rs -k "p2p or nvls or graph" > $O/pytest_p2p.log 2>&1; echo rc=$? >> $O/pytest_p2p.log
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > $O/bench_decode.log 2>&1
timeout -s KILL 400 python bench.py --config prefill --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_prefill.log 2>&1
timeout -s KILL 900 python bench.py --config stack --steps 10 --warmup 3 > $O/bench_stack.log 2>&1
timeout -s KILL 400 python bench.py --fp8 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_decode_fp8.log 2>&1
timeout -s KILL 400 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_decode.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_prefill.csv python bench.py --config prefill --steps 2 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_decode_fp8.csv python bench.py --fp8 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_" -s 2 -c 5 -o $O/prof_decode python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_pair" -s 2 -c 2 -o $O/prof_prefill python bench.py --config prefill --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_fp8x" -s 2 -c 2 -o $O/prof_decode_fp8 python bench.py --fp8 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_kernel" -s 4 -c 2 -o $O/prof_stack_layer python bench.py --shard tp1 --config stack --steps 1 --warmup 3 > /dev/null 2>&1
for c in decode prefill stack; do for s in ep2 ep4 ep8 tp2 tp4 tp8; do
  st=30; [ $c = prefill ] && st=5
  timeout -s KILL 300 python bench.py --shard $s --config $c --steps $st --warmup 3 2>&1 | grep "^{" >> $O/shards.jsonl
done; done
bash scripts/sanitize.sh $O/sanitizer
ls -la $O
