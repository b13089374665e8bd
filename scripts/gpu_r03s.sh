# fused FFN with 128-row w1/w3 tiles (fused_half): tests, timelines, shard A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03s.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_s.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_s.log
tail -3 gpurun_out/pytest_fused_s.log
if grep -q 'rc=0' gpurun_out/pytest_fused_s.log; then
for sh in "--shard ep8" "--shard tp8"; do
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2,fused_half=2 $sh >> gpurun_out/timeline_s.log 2>&1
done
for s in ep8 tp8; do
bash scripts/ab_tunings.sh s_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2,fused_half=2 fused=2,fused_half=2,fused_uniform=1 fused=2,fused_half=2,fused_splits=8
done
for s in ep4 tp4; do
bash scripts/ab_tunings.sh s_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2,fused_half=2 fused=2,fused_half=1
done
bash scripts/ab_tunings.sh s_dec 2 "" - fused_half=2
fi
