# Interleaved A/B over tuning strings: bash scripts/ab_tunings.sh <tag> <rounds> "<bench args>" tuning1 tuning2 ...
# ("-" = no tuning). Prints ms_per_step per run and kernel_ms.
TAG=$1; ROUNDS=$2; ARGS=$3; shift 3
for i in $(seq 1 $ROUNDS); do
  j=0
  for t in "$@"; do
    j=$((j+1))
    if [ "$t" = "-" ]; then TU=""; else TU="--tuning $t"; fi
    timeout -s KILL 300 python bench.py --no-cpu-baseline $ARGS $TU > gpurun_out/ab_${TAG}_${j}_$i.log 2>&1
    echo "$TAG r$i [$t] $(python scripts/ab_line.py gpurun_out/ab_${TAG}_${j}_$i.log)" | tee -a gpurun_out/ab_${TAG}.txt
  done
done
