# fused w2 split taper: linear S-i (default) vs geometric 2^(S-1-i) (fused_uniform=2) vs quadratic (=3)
O=gpurun_out/r03taper; mkdir -p $O
bash scripts/ab_tunings.sh taper 4 "--steps 100 --warmup 5" - fused_uniform=2 fused_uniform=3 fused_uniform=2,fused_splits=5 fused_uniform=3,fused_splits=3 > /dev/null 2>&1
cat gpurun_out/ab_taper.txt
