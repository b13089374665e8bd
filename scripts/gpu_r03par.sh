# fused FFN exit hand-off: two counter sets + parity flip (new) vs the last CTA's fenced reset (old, HEAD build)
O=gpurun_out/r03par; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_fused.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_new.txt 2>&1; echo "pytest $?"; tail -n 2 $O/pytest_new.txt
for i in 1 2; do MOE_LIB=build_ab/libmoe_tldn.so timeout -s KILL 300 python scripts/exp/timeline.py 64 - --teardown >> $O/timeline_td.log 2>&1; done
cat $O/timeline_td.log
bash scripts/ab_decode.sh "old new" 5 > $O/ab.txt 2>&1
cat $O/ab.txt
