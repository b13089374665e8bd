# bf16 fused decode with a 32-row token tile (swap_nb_cap=32: 6 ring stages instead of 5) vs the 64-row default
bash scripts/ab_tunings.sh nb32 3 "--steps 100 --warmup 5" - swap_nb_cap=32 swap_nb_cap=32,fused_stages=5 > /dev/null 2>&1
cut -c1-200 gpurun_out/ab_nb32.txt
