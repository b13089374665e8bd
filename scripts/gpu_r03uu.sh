O=gpurun_out/r03uu; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 400 python bench.py --fp8 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_decode_fp8.log 2>&1
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > $O/bench_decode.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_ffn_fused" -s 2 -c 1 -o $O/prof_fp8_fused python bench.py --fp8 --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_decode_fp8.csv python bench.py --fp8 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
ls $O
