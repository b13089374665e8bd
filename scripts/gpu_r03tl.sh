# decode timeline: exit stamps before (tl) and after (tlx) the router's scan hand-off and the fused FFN's counter reset
O=gpurun_out/r03tl; mkdir -p $O
for v in tl tlx tl tlx; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python scripts/exp/timeline.py 64 >> $O/timeline_$v.log 2>&1
done
tail -n 30 $O/timeline_tl.log $O/timeline_tlx.log
