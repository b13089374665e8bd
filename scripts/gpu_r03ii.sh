# multi-rank EP flow on one GPU (2 processes, P2P over CUDA IPC): router-folded dispatch vs permute dispatch
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r03ii.log 2>&1
export BENCH_ONE_DEVICE=1 CUDA_DEVICE_MAX_CONNECTIONS=32
for r in 1 2; do for tu in "" "--tuning ep_fold=1"; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --p2p --par ep --steps 50 --warmup 5 --no-cpu-baseline $tu \
    > gpurun_out/ii_$r.log 2>&1
  echo "[$tu] r$r rc=$? $(grep '^{' gpurun_out/ii_$r.log | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print(round(j['ms_per_step'],4), j.get('graph_replay'), j.get('parity',{}).get('ok'), j.get('gpu_launches'))")" | tee -a gpurun_out/ab_ii.txt
done; done
