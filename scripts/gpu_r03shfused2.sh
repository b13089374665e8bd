# taper rule: geometric only where one split's w2 tiles cover half the grid (EP4 / EP8 ranks back on linear)
for s in ep8 ep4 ep2 tp8; do
  bash scripts/ab_tunings.sh shg_$s 2 "--shard $s --steps 50 --warmup 3" fused=2,fused_half=2 fused=2,fused_half=2,fused_uniform=2 > /dev/null 2>&1
done
bash scripts/ab_tunings.sh shg_dec 3 "--steps 100 --warmup 5" - fused_uniform=2 > /dev/null 2>&1
cat gpurun_out/ab_shg_*.txt | cut -c1-110
