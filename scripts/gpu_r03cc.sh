python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03cc.log 2>&1
bash scripts/ab_tunings.sh cc_dec 3 "" - fused_splits=3 fused_splits=5 fused_splits=6
