# two-kernel w2 split-K at the per-rank shapes (decode): auto vs 8 vs 2
for r in 1 2; do
for s in ep8 tp8 ep4 tp4; do
for sk in 0 8 2; do
timeout -s KILL 300 python bench.py --shard $s --config decode --steps 30 --warmup 3 --split-k $sk > gpurun_out/v_${s}_${sk}_$r.log 2>&1
echo "$s split_k=$sk r$r $(python scripts/ab_line.py gpurun_out/v_${s}_${sk}_$r.log)" | tee -a gpurun_out/ab_v.txt
done; done; done
