python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_mm.log 2>&1
bash scripts/ab_tunings.sh mm_fp8 2 "--fp8 --no-parity" fused=2 fused=2,fused_uniform=1 fused=2,fused_splits=2 fused=2,fused_uniform=1,fused_splits=2 fused=2,fused_splits=1 -
