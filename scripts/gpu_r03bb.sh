O=gpurun_out/r03bb; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
tail -4 $O/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
