# combine with 4x the blocks at small T: full GPU suite + decode A/B
O=gpurun_out/r03t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
bash scripts/ab_tunings.sh t_dec 3 "" - combine_vec=4 fused=1 fused=1,combine_vec=4
