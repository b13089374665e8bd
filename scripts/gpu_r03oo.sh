# next-layer weight prefetch in the fused FFN's tail (MoEStack): stack tests, M0 / cycle A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_oo.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_fused.py -q -x -k "stack or graph" > gpurun_out/pytest_oo.log 2>&1; echo rc=$? >> gpurun_out/pytest_oo.log
tail -2 gpurun_out/pytest_oo.log
bash scripts/ab_tunings.sh oo_M0 3 "--config stack --stack-batch M0 --steps 10 --warmup 3 --no-cpu-baseline" - next_prefetch=-1 next_prefetch=32
bash scripts/ab_tunings.sh oo_cyc 2 "--config stack --stack-batch cycle --steps 5 --warmup 3 --no-cpu-baseline" - next_prefetch=-1
