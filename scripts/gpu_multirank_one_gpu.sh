# The multi-rank bench flow on a ONE-GPU box (BENCH_ONE_DEVICE=1: every rank on cuda:0,
# gloo host group, P2P transport over CUDA IPC between the processes): sharding, the
# exchange, graph replay, max-over-ranks timing and the parity reduction of
# `bench.py --gpus 2`. Timings are not results (two ranks share one GPU).
export BENCH_ONE_DEVICE=1 CUDA_DEVICE_MAX_CONNECTIONS=32
for par in ep tp; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --p2p --par $par --steps 20 --warmup 3 --no-cpu-baseline \
    > gpurun_out/multirank_$par.log 2>&1
  echo "$par rc=$?"
  grep "^{" gpurun_out/multirank_$par.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print(j['n_gpus'], j['config']['parallelism'], j['config']['transport'], round(j['ms_per_step'],4), j.get('graph_replay'), j.get('parity'))" || tail -20 gpurun_out/multirank_$par.log
done
