# probe: fused kernel with w1/w3 tiles only (timing; wrong outputs), FP8 and bf16, vs the two-kernel K3
for r in 1 2; do
MOE_LIB=build_ab/libmoe_g1only.so timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity --tuning fused=2 > gpurun_out/ll_f8_$r.log 2>&1
echo "g1only fp8 fused r$r $(python scripts/ab_line.py gpurun_out/ll_f8_$r.log)" | tee -a gpurun_out/ab_ll.txt
MOE_LIB=build_ab/libmoe_g1only.so timeout -s KILL 300 python bench.py --no-cpu-baseline --no-parity > gpurun_out/ll_bf_$r.log 2>&1
echo "g1only bf16 fused r$r $(python scripts/ab_line.py gpurun_out/ll_bf_$r.log)" | tee -a gpurun_out/ab_ll.txt
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity > gpurun_out/ll_two_$r.log 2>&1
echo "two-kernel fp8 r$r $(python scripts/ab_line.py gpurun_out/ll_two_$r.log)" | tee -a gpurun_out/ab_ll.txt
done
