# M2 (T=4152) stack batch: tokens-as-M pair tiles (default) vs swap-AB tiles (N = valid tokens, no padded tail)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03ff.log 2>&1
bash scripts/ab_tunings.sh ff_M2 2 "--config stack --stack-batch M2 --steps 5 --warmup 3 --no-cpu-baseline" - g1_swap_rows=2048,g2_swap_rows=2048 g1_swap_rows=2048,g2_swap_rows=2048,swap_pair=1 g1_swap_rows=2048
