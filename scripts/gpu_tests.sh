# GPU parity tests only (fast iteration): bash scripts/gpu_tests.sh <tag> [pytest -k expr]
TAG=${1:-run}
K=${2:-}
if [ -n "$K" ]; then
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -k "$K" -s > gpurun_out/pytest_$TAG.log 2>&1
else
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -s > gpurun_out/pytest_$TAG.log 2>&1
fi
echo rc=$? >> gpurun_out/pytest_$TAG.log
tail -30 gpurun_out/pytest_$TAG.log
