# fused FFN v4 (tapered split-major w2 tiles): parity, timelines, shard A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03h.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_h.log
tail -3 gpurun_out/pytest_fused_h.log
if grep -q 'rc=0' gpurun_out/pytest_fused_h.log; then
for sh in "" "--shard tp8" "--shard ep8"; do
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2 $sh >> gpurun_out/timeline_h.log 2>&1
done
bash scripts/ab_tunings.sh h_dec 2 "" - fused=2 fused=2,fused_splits=8 fused=2,fused_uniform=1
for s in ep8 tp8; do
bash scripts/ab_tunings.sh h_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2 fused=2,fused_splits=8 fused=2,fused_uniform=1
done
fi
