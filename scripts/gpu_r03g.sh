# fused FFN v3 (tail tiles, all-ready fast path, no claim-ahead): parity, timelines, shard A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03g.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_g.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_g.log
tail -3 gpurun_out/pytest_fused_g.log
if grep -q 'rc=0' gpurun_out/pytest_fused_g.log; then
for sh in "" "--shard tp8" "--shard ep8"; do
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2 $sh >> gpurun_out/timeline_g.log 2>&1
done
bash scripts/ab_tunings.sh g_dec 2 "" - fused=2 fused=2,fused_splits=8
for s in ep8 tp8; do
bash scripts/ab_tunings.sh g_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2 fused=2,fused_splits=8
done
fi
