# decode knobs re-swept on the geometric-taper build: speculative prefetch depth, ring depth
bash scripts/ab_tunings.sh sp 3 "--steps 100 --warmup 5" - spec_l2=32 spec_l2=64 fused_stages=4 > /dev/null 2>&1
cut -c1-60 gpurun_out/ab_sp.txt
