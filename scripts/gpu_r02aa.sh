# r02 evidence refresh for the CTA-pair swap build: stack M1 / cycle lines, ncu full of the pair
# kernels on one stack layer, launch list of one stack layer
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/r02b; mkdir -p $O
timeout -s KILL 900 python bench.py --config stack --stack-batch M1 --steps 10 --warmup 3 > $O/bench_stack_M1.log 2>&1
timeout -s KILL 900 python bench.py --config stack --stack-batch cycle --steps 3 --warmup 3 > $O/bench_stack_cycle.log 2>&1
grep "^{" $O/bench_stack_M1.log | head -c 600; echo
grep "^{" $O/bench_stack_cycle.log | head -c 400; echo
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_swap_pair" -s 4 -c 2 -o $O/prof_stack_layer_pair python bench.py --shard tp1 --config stack --steps 1 --warmup 3 > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_stack_layer.csv python bench.py --shard tp1 --config stack --steps 3 --warmup 3 > /dev/null 2>&1
ls $O
