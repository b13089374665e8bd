# FP8 w2: double-buffered B-scale TMEM columns (default build) vs single set (libmoe_sfb0.so)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_nn.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_fused.py -q -x -k "fp8" > gpurun_out/pytest_nn.log 2>&1; echo rc=$? >> gpurun_out/pytest_nn.log
tail -2 gpurun_out/pytest_nn.log
for r in 1 2 3; do
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity > gpurun_out/nn_db_$r.log 2>&1
echo "sfb double r$r $(python scripts/ab_line.py gpurun_out/nn_db_$r.log)" | tee -a gpurun_out/ab_nn.txt
MOE_LIB=build_ab/libmoe_sfb0.so timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity > gpurun_out/nn_s_$r.log 2>&1
echo "sfb single r$r $(python scripts/ab_line.py gpurun_out/nn_s_$r.log)" | tee -a gpurun_out/ab_nn.txt
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity --tuning fused=2 > gpurun_out/nn_f_$r.log 2>&1
echo "sfb double fused r$r $(python scripts/ab_line.py gpurun_out/nn_f_$r.log)" | tee -a gpurun_out/ab_nn.txt
done
