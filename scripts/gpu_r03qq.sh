python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_qq.log 2>&1
MOE_LIB=build_ab/libmoe_g2r128.so timeout -s KILL 900 python -m pytest tests/test_fused.py -q -x -k "fp8" > gpurun_out/pytest_qq.log 2>&1; echo rc=$? >> gpurun_out/pytest_qq.log
tail -2 gpurun_out/pytest_qq.log
for r in 1 2 3; do
MOE_LIB=build_ab/libmoe_g2r128.so timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity --tuning fused=2 > gpurun_out/qq.log 2>&1
echo "g2rows128 fused r$r $(python scripts/ab_line.py gpurun_out/qq.log)" | tee -a gpurun_out/ab_qq.txt
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity --tuning fused=2 > gpurun_out/qq.log 2>&1
echo "g2rows256 fused r$r $(python scripts/ab_line.py gpurun_out/qq.log)" | tee -a gpurun_out/ab_qq.txt
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity > gpurun_out/qq.log 2>&1
echo "two kernels r$r $(python scripts/ab_line.py gpurun_out/qq.log)" | tee -a gpurun_out/ab_qq.txt
done
