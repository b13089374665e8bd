# T=575: fused FFN with 128-row token tiles (2 per expert) vs the CTA-pair swap kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03z.log 2>&1
bash scripts/ab_tunings.sh z_tp1 2 "--shard tp1 --config stack --steps 20 --warmup 3" - fused=2,swap_nb_cap=128 swap_nb_cap=128
bash scripts/ab_tunings.sh z_M1 2 "--config stack --stack-batch M1 --steps 10 --warmup 3 --no-cpu-baseline" - fused=2,swap_nb_cap=128
