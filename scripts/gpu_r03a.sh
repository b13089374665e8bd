# re-entry sanity: rebuild on the box, full GPU suite, default bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03a.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r03a.log 2>&1; echo rc=$? >> gpurun_out/pytest_r03a.log
timeout -s KILL 400 python bench.py > gpurun_out/bench_r03a.log 2>&1
tail -3 gpurun_out/pytest_r03a.log; tail -c 600 gpurun_out/bench_r03a.log
