O=gpurun_out/r03k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -5 $O/pytest.log
