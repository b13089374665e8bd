python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export MOE_LIB=build_ab/libmoe_tl.so
for a in "64 - --fp8" "64 -"; do timeout -s KILL 300 python scripts/exp/timeline.py $a 2>&1 | tail -12; done
