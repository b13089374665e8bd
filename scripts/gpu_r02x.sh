python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python scripts/exp/stack_graph.py 575 2>&1 | tail -8
MOE_LIB=build_ab/libmoe_tl.so timeout -s KILL 600 python scripts/exp/stack_graph.py 575 2>&1 | tail -20
