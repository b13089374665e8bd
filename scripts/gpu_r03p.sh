# spec L2 prefetch for T <= 1024 incl. the CTA-pair w1/w3 kernel: full suite, stack M1 A/B, tp8 stack shard
O=gpurun_out/r03p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
if grep -q 'rc=0' $O/pytest.log; then
bash scripts/ab_tunings.sh p_M1 2 "--config stack --stack-batch M1 --steps 10 --warmup 3" - spec_l2=-1
bash scripts/ab_tunings.sh p_tp8st 2 "--shard tp8 --config stack --steps 20 --warmup 3" - spec_l2=-1
bash scripts/ab_tunings.sh p_tp1st 2 "--shard tp1 --config stack --steps 20 --warmup 3" - spec_l2=-1
fi
