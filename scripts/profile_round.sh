# Evidence for profiles/<tag>: bench JSON lines, ncu launch lists (gpu__time_duration, clock-control none)
# and one `ncu --set full` capture of every libmoe kernel of one forward, decode and prefill.
# usage (under gpurun, repo root): bash scripts/profile_round.sh <tag>
TAG=${1:-r01}
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_decode_$TAG.log 2>&1
timeout -s KILL 400 python bench.py --config prefill --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_prefill_$TAG.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_decode_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_prefill_$TAG.csv python bench.py --config prefill --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_" -s 2 -c 5 -o gpurun_out/prof_decode_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"moe_" -s 2 -c 5 -o gpurun_out/prof_prefill_$TAG python bench.py --config prefill --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
# FP8-weight decode variant
timeout -s KILL 400 python bench.py --steps 100 --warmup 5 --fp8 --no-cpu-baseline > gpurun_out/bench_decode_fp8_$TAG.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_fp8" -s 2 -c 2 -o gpurun_out/prof_decode_fp8_$TAG python bench.py --steps 1 --warmup 3 --fp8 --no-cpu-baseline > /dev/null 2>&1
# 32-layer stack (configs[4] shape on one GPU)
timeout -s KILL 600 python bench.py --config stack --steps 5 --warmup 3 > gpurun_out/bench_stack_$TAG.log 2>&1
