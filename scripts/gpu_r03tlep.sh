O=gpurun_out/r03tlep; mkdir -p $O
for s in ep8 tp8 ep4; do
  MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 300 python scripts/exp/timeline.py 64 - --shard $s >> $O/timeline_$s.log 2>&1
  MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 300 python scripts/exp/timeline.py 64 - --shard $s >> $O/timeline_$s.log 2>&1
done
timeout -s KILL 300 python bench.py --shard ep8 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_ep8.json 2>&1
cat $O/timeline_*.log; tail -c 1500 $O/bench_ep8.json
