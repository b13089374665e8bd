# EP / TP rank shapes: two kernels (default) vs the fused FFN with 128-row w1/w3 tiles, now with the geometric taper
for s in ep8 tp8 ep4 tp4; do
  bash scripts/ab_tunings.sh shf_$s 2 "--shard $s --steps 50 --warmup 3" - fused=2,fused_half=2 fused=2,fused_half=2,fused_splits=8 > /dev/null 2>&1
done
cat gpurun_out/ab_shf_*.txt | cut -c1-120
