python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_rr.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py tests/test_gpu_parity.py -q -x -k "fp8" > gpurun_out/pytest_rr.log 2>&1; echo rc=$? >> gpurun_out/pytest_rr.log
tail -2 gpurun_out/pytest_rr.log
if grep -q 'rc=0' gpurun_out/pytest_rr.log; then
bash scripts/ab_tunings.sh rr_fp8 3 "--fp8 --no-parity" fused=2 - fused=2,fused_uniform=1
fi
