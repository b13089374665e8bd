# EP dispatch folded into the router: P2P / EP tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03hh.log 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "p2p or router_dispatch or ep_ or mixtral_decode_8" > gpurun_out/pytest_hh.log 2>&1; echo rc=$? >> gpurun_out/pytest_hh.log
tail -3 gpurun_out/pytest_hh.log
