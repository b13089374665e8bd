# fused FFN at the per-rank shard shapes (decode + stack layer) vs two kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03d.log 2>&1
for s in ep8 tp8 ep4 tp4 ep2 tp2; do
bash scripts/ab_tunings.sh d_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2 fused=2,fused_stages=4 fused=2,fused_splits=4
done
for s in ep8 tp8; do
bash scripts/ab_tunings.sh st_$s 1 "--shard $s --config stack --steps 20 --warmup 3" - fused=2 fused=2,fused_splits=4
done
