# One GPU round: parity tests, benches, ncu launch lists and full captures.
# usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-run}
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
timeout -s KILL 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_decode_$TAG.log 2>&1
timeout -s KILL 400 python bench.py --config prefill --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_prefill_$TAG.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_decode_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_prefill_$TAG.csv python bench.py --config prefill --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_" -s 4 -c 5 -o gpurun_out/prof_decode_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_decode_$TAG.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"moe_" -s 2 -c 5 -o gpurun_out/prof_prefill_$TAG python bench.py --config prefill --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_prefill_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log
