# speculative L2 prefetch for the FP8 decode (fused kernel; the two-kernel FP8 G1 waits before reading counts)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_tt.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py tests/test_gpu_parity.py -q -x -k "fp8 or spec" > gpurun_out/pytest_tt.log 2>&1; echo rc=$? >> gpurun_out/pytest_tt.log
tail -2 gpurun_out/pytest_tt.log
if grep -q 'rc=0' gpurun_out/pytest_tt.log; then
bash scripts/ab_tunings.sh tt_fp8 3 "--fp8 --no-parity" - spec_l2=-1 spec_l2=32 fused=1
fi
