# split chaining in the fused FFN: tests, timeline, decode A/B over splits
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03r.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_r.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_r.log
tail -3 gpurun_out/pytest_fused_r.log
if grep -q 'rc=0' gpurun_out/pytest_fused_r.log; then
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2 >> gpurun_out/timeline_r.log 2>&1
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2,fused_splits=8 >> gpurun_out/timeline_r.log 2>&1
bash scripts/ab_tunings.sh r_dec 3 "" - fused_chain=1 fused_splits=8 fused_splits=6 fused=1
fi
