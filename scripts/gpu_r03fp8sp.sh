# FP8 fused decode: w2 split count / taper re-swept on the final build
bash scripts/ab_tunings.sh f8s 3 "--fp8 --steps 100 --warmup 5" - fused_splits=3 fused_splits=5 fused_splits=6 fused_uniform=3 fused_uniform=0 > /dev/null 2>&1
cut -c1-70 gpurun_out/ab_f8s.txt
