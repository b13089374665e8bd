# FP8 decode with the speculative L2 prefetch: parity + A/B of its depth, timeline
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fp8 or speculative" > gpurun_out/pytest_fp8spec.log 2>&1
tail -3 gpurun_out/pytest_fp8spec.log
bash scripts/ab_env.sh "spec_l2=-1 spec_l2=8 spec_l2=16 spec_l2=32" 3 --fp8 --no-parity
