python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03gg.log 2>&1
bash scripts/ab_tunings.sh gg_fp8 3 "--fp8" fused=2 -
bash scripts/ab_tunings.sh gg_bf16 2 "" - weight_hint=2
