# stack batches with the fused FFN (M0 layers take it) vs two kernels; fused tests re-run
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03o.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused.py -q -x > gpurun_out/pytest_fused_o.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused_o.log
tail -2 gpurun_out/pytest_fused_o.log
for b in M0 cycle; do
bash scripts/ab_tunings.sh o_$b 2 "--config stack --stack-batch $b --steps 10 --warmup 3" - fused=1
done
