python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03aa.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py -q -x -k "fp8 or parity" > gpurun_out/pytest_aa.log 2>&1; echo rc=$? >> gpurun_out/pytest_aa.log
tail -2 gpurun_out/pytest_aa.log
bash scripts/ab_tunings.sh aa_fp8 2 "--fp8" fused=2 -
