python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03ee.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stack or swap_pair or skew" > gpurun_out/pytest_ee.log 2>&1; echo rc=$? >> gpurun_out/pytest_ee.log
tail -2 gpurun_out/pytest_ee.log
for r in 1 2; do for s in tp8 ep8 tp4 ep4; do
timeout -s KILL 300 python bench.py --shard $s --config stack --steps 30 --warmup 3 > gpurun_out/ee_${s}_$r.log 2>&1
echo "$s r$r $(python scripts/ab_line.py gpurun_out/ee_${s}_$r.log)" | tee -a gpurun_out/ab_ee.txt
done; done
