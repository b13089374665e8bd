# Evidence for profiles/r03 (final build of round 3): bench lines, launch lists, ncu full capture
# of the fused decode FFN, per-rank shard sweep, compute-sanitizer incl. the fused kernel.
# usage (under gpurun, repo root): bash scripts/profile_round3.sh <tag>
TAG=${1:-r03}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > $O/bench_decode.log 2>&1
timeout -s KILL 400 python bench.py --config prefill --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_prefill.log 2>&1
timeout -s KILL 900 python bench.py --config stack --steps 10 --warmup 3 > $O/bench_stack.log 2>&1
for b in M0 cycle; do timeout -s KILL 900 python bench.py --config stack --stack-batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_stack_$b.log 2>&1; done
timeout -s KILL 400 python bench.py --fp8 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_decode_fp8.log 2>&1
timeout -s KILL 400 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_decode.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_ffn_fused" -s 2 -c 2 -o $O/prof_decode_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_combine" -s 2 -c 2 -o $O/prof_decode_combine python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
for c in decode stack; do for s in ep2 ep4 ep8 tp2 tp4 tp8; do
  timeout -s KILL 300 python bench.py --shard $s --config $c --steps 30 --warmup 3 2>&1 | grep "^{" >> $O/shards.jsonl
done; done
bash scripts/sanitize.sh $O/sanitizer
ls -la $O
