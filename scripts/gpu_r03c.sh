# fused FFN sweep: grid / stages / splits at decode; EP8 / TP8 per-rank shapes
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03c.log 2>&1
bash scripts/ab_tunings.sh dec 2 "" - fused=2,fused_splits=4 fused=2,fused_splits=4,fused_stages=4 fused=2,fused_splits=4,fused_stages=3 fused=2,fused_splits=4,g1_grid=112 fused=2,fused_splits=4,g1_grid=128 fused=2,fused_splits=4,g1_grid=128,fused_stages=4
for s in ep8 tp8 ep4 tp4; do
bash scripts/ab_tunings.sh sh_$s 2 "--shard $s --config decode --steps 20 --warmup 3" - fused=2 fused=2,fused_stages=4 fused=2,fused_stages=3
done
