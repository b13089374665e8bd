# fused FFN default: full GPU suite, default bench line, launch list, ncu full of the fused kernel
O=gpurun_out/r03j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > $O/bench_decode.log 2>&1
tail -c 400 $O/bench_decode.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_decode.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_ffn_fused" -s 2 -c 2 -o $O/prof_decode_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
ls $O
