python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/pytest_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_h.log
tail -12 gpurun_out/pytest_h.log
