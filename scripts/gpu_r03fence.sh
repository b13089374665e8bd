# fused FFN fences: __threadfence (fence.sc.gpu, f0) vs fence.acq_rel.gpu at the exit hand-off (f1) and at the tile publishes too (f2)
O=gpurun_out/r03fence; mkdir -p $O
for v in f1 f2; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 900 python -m pytest tests/test_fused.py -m gpu -x -q > $O/pytest_$v.txt 2>&1; echo "pytest $v $?"; tail -n 1 $O/pytest_$v.txt
done
for v in tlx0 tlx2; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python scripts/exp/timeline.py 64 >> $O/timeline_$v.log 2>&1
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python scripts/exp/timeline.py 64 >> $O/timeline_$v.log 2>&1
done
tail -n 9 $O/timeline_tlx0.log $O/timeline_tlx2.log
bash scripts/ab_decode.sh "f0 f1 f2" 4 > $O/ab.txt 2>&1
cat $O/ab.txt
