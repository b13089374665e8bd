# M0 stack (32 fused decode layers): geometric (default) vs linear split taper, interleaved on one box
bash scripts/ab_tunings.sh m0 3 "--config stack --stack-batch M0 --steps 10 --warmup 3" - fused_uniform=2 > /dev/null 2>&1
cut -c1-80 gpurun_out/ab_m0.txt
