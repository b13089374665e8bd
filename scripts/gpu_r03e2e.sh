# e2e (host buffers, zero-copy output) with the in-kernel combine: output slices stream to the host as they complete
for i in 1 2 3; do for t in - fused_combine=1; do
  if [ "$t" = "-" ]; then TU=""; else TU="--tuning $t"; fi
  timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 $TU 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('r$i', '$t', 'ms', round(j['ms_per_step'],4), 'e2e_ms', round(j['e2e']['ms_per_step'],4), 'e2e', round(j['e2e']['value']))" | tee -a gpurun_out/ab_e2e.txt
done; done
