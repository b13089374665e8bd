# fused FFN v5 (spec prefetch off the producer lane): parity, timeline, decode A/B x3, shards
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03i.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_i.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_i.log
tail -3 gpurun_out/pytest_fused_i.log
if grep -q 'rc=0' gpurun_out/pytest_fused_i.log; then
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 200 python scripts/exp/timeline.py 64 fused=2 >> gpurun_out/timeline_i.log 2>&1
bash scripts/ab_tunings.sh i_dec 3 "" - fused=2
for s in ep2 ep4 tp2 tp4 tp8 ep8; do
bash scripts/ab_tunings.sh i_$s 1 "--shard $s --config decode --steps 20 --warmup 3" - fused=2 fused=2,fused_uniform=1
done
fi
