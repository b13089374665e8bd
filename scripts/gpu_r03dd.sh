# TP8 rank of the T=575 stack layer (BASELINE configs[4] per-rank shape): w2 split-K x pair/single
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03dd.log 2>&1
for r in 1 2; do
for sk in 0 2 3; do
for tu in "-" "swap_pair=1"; do
if [ "$tu" = "-" ]; then T=""; else T="--tuning $tu"; fi
timeout -s KILL 300 python bench.py --shard tp8 --config stack --steps 30 --warmup 3 --split-k $sk $T > gpurun_out/dd_${sk}_${tu}_$r.log 2>&1
echo "tp8st split_k=$sk [$tu] r$r $(python scripts/ab_line.py gpurun_out/dd_${sk}_${tu}_$r.log)" | tee -a gpurun_out/ab_dd.txt
done; done; done
