O=gpurun_out/r03m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_comb_on.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_comb_off.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --tuning fused_combine=1 > /dev/null 2>&1
for s in 4 2; do timeout -s KILL 300 python bench.py --no-cpu-baseline --tuning fused_splits=$s > $O/bench_s$s.log 2>&1; python scripts/ab_line.py $O/bench_s$s.log; done
