O=gpurun_out/r03stress; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_fused_stress.py -m gpu -q -x > $O/pytest_stress.txt 2>&1; echo "stress $?"; tail -n 15 $O/pytest_stress.txt
