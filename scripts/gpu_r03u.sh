# fused -> combine epoch hand-off: fused tests + parity subset, timeline, decode A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03u.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py tests/test_gpu_parity.py -q -x -k "fused or c2 or c1_parity or graph or spec" > gpurun_out/pytest_u.log 2>&1; echo rc=$? >> gpurun_out/pytest_u.log
tail -3 gpurun_out/pytest_u.log
if grep -q 'rc=0' gpurun_out/pytest_u.log; then
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 - >> gpurun_out/timeline_u.log 2>&1
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused_handoff=1 >> gpurun_out/timeline_u.log 2>&1
bash scripts/ab_tunings.sh u_dec 3 "" - fused_handoff=1
fi
