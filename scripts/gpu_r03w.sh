# FP8 fused FFN: tests (fused + FP8 parity), FP8 decode A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03w.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py tests/test_gpu_parity.py -q -x -k "fp8" > gpurun_out/pytest_w.log 2>&1; echo rc=$? >> gpurun_out/pytest_w.log
tail -3 gpurun_out/pytest_w.log
if grep -q 'rc=0' gpurun_out/pytest_w.log; then
bash scripts/ab_tunings.sh w_fp8 3 "--fp8" - fused=1 fused_splits=8 fused_stages=4
fi
