set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_a.log 2>&1; echo rc=$? >> gpurun_out/pytest_a.log
tail -5 gpurun_out/pytest_a.log
timeout -s KILL 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_decode_a.log 2>&1
tail -c 3000 gpurun_out/bench_decode_a.log
bash scripts/shard_sweep.sh a "decode prefill"
