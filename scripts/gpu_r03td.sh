O=gpurun_out/r03td; mkdir -p $O
for i in 1 2 3; do MOE_LIB=build_ab/libmoe_tld.so timeout -s KILL 300 python scripts/exp/timeline.py 64 - --teardown >> $O/timeline_td.log 2>&1; done
cat $O/timeline_td.log
