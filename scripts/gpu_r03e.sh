# timelines: fused vs two kernels at decode and at EP8 / TP8 rank shapes
export MOE_LIB=build_ab/libmoe_tl.so
for sh in "" "--shard tp8" "--shard ep8"; do
for tu in - fused=2 fused=2,fused_splits=4; do
timeout -s KILL 200 python scripts/exp/timeline.py 64 $tu $sh >> gpurun_out/timeline_e.log 2>&1
done; done
cat gpurun_out/timeline_e.log
