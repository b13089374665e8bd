O=gpurun_out/r03fp8grp; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_fused.py -m gpu -q -x > $O/pytest_fused.txt 2>&1; echo "fused $?"; tail -n 3 $O/pytest_fused.txt
