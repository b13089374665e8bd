# fused FFN v2 (tail tiles, claim-ahead, all-ready fast path): parity, timelines, shard A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03f.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_f.log
tail -3 gpurun_out/pytest_fused_f.log
if grep -q 'rc=0' gpurun_out/pytest_fused_f.log; then
for sh in "" "--shard tp8" "--shard ep8"; do
for tu in - fused=2 fused=2,fused_splits=8; do
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 $tu $sh >> gpurun_out/timeline_f.log 2>&1
done; done
bash scripts/ab_tunings.sh f_dec 2 "" - fused=2 fused=2,fused_splits=8 fused=2,fused_splits=2
for s in ep8 tp8 ep4 tp4; do
bash scripts/ab_tunings.sh f_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2 fused=2,fused_splits=8 fused=2,fused_splits=2
done
fi
