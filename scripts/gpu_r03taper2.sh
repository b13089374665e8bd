# geometric split taper as the default: fused tests, decode / FP8 / TP2-rank A/B against the linear taper
O=gpurun_out/r03taper2; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_fused.py tests/test_fused_stress.py -m gpu -x -q > $O/pytest_fused.txt 2>&1; echo "pytest $?"; tail -n 1 $O/pytest_fused.txt
bash scripts/ab_tunings.sh tg 3 "--steps 100 --warmup 5" - fused_uniform=2 fused_splits=3 fused_splits=5 fused_splits=6 > /dev/null 2>&1
bash scripts/ab_tunings.sh tg8 3 "--fp8 --steps 100 --warmup 5" - fused_uniform=2 > /dev/null 2>&1
bash scripts/ab_tunings.sh tgtp2 3 "--shard tp2 --steps 100 --warmup 5" - fused_uniform=2 > /dev/null 2>&1
cat gpurun_out/ab_tg.txt gpurun_out/ab_tg8.txt gpurun_out/ab_tgtp2.txt | cut -c1-90
