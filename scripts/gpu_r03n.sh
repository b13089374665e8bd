# in-kernel combine: fused tests, timeline, decode A/B (combine in kernel vs separate vs two-kernel)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03n.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_n.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_n.log
tail -3 gpurun_out/pytest_fused_n.log
if grep -q 'rc=0' gpurun_out/pytest_fused_n.log; then
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2 >> gpurun_out/timeline_n.log 2>&1
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2,fused_combine=1 >> gpurun_out/timeline_n.log 2>&1
bash scripts/ab_tunings.sh n_dec 3 "" - fused_combine=1 fused=1
fi
