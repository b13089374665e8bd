# Interleaved A/B of libmoe build variants on bench.py lines: bash scripts/ab_lib_shard.sh <tag> "<v1 v2 ..>" <rounds> "<bench args>"
TAG=$1; VARS=$2; R=$3; ARGS=$4
for r in $(seq 1 $R); do for v in $VARS; do
  MOE_LIB=build_ab/libmoe_$v.so timeout -s KILL 300 python bench.py --no-cpu-baseline $ARGS > gpurun_out/abl_${TAG}_${v}_$r.log 2>&1
  echo "$TAG r$r [$v] $(python scripts/ab_line.py gpurun_out/abl_${TAG}_${v}_$r.log)" | tee -a gpurun_out/abl_${TAG}.txt
done; done
