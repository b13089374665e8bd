# FP8 decode: w2 split-K and grid variants of the block-scaled K4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_pp.log 2>&1
for r in 1 2; do
for v in "" "--split-k 8" "--split-k 6" "--split-k 2" "--tuning g2_grid=128" "--tuning g1_grid=148"; do
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity $v > gpurun_out/pp.log 2>&1
echo "[$v] r$r $(python scripts/ab_line.py gpurun_out/pp.log)" | tee -a gpurun_out/ab_pp.txt
done; done
