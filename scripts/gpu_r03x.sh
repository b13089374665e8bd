python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03x.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py -q -x -k "fp8" > gpurun_out/pytest_x.log 2>&1; echo rc=$? >> gpurun_out/pytest_x.log
tail -2 gpurun_out/pytest_x.log
bash scripts/ab_tunings.sh x_fp8 2 "--fp8" - fused=1 g1_grid=128 fused_stages=4 fused_stages=3
