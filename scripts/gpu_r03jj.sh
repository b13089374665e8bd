# probe: FP8 fused without the G1 publish fences (timing only)
for r in 1 2; do
MOE_LIB=build_ab/libmoe_nofence.so timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity --tuning fused=2 > gpurun_out/jj_nf_$r.log 2>&1
echo "nofence fused r$r $(python scripts/ab_line.py gpurun_out/jj_nf_$r.log)" | tee -a gpurun_out/ab_jj.txt
timeout -s KILL 300 python bench.py --fp8 --no-cpu-baseline --no-parity --tuning fused=2 > gpurun_out/jj_f_$r.log 2>&1
echo "fenced fused r$r $(python scripts/ab_line.py gpurun_out/jj_f_$r.log)" | tee -a gpurun_out/ab_jj.txt
MOE_LIB=build_ab/libmoe_nofence.so timeout -s KILL 300 python bench.py --no-cpu-baseline --no-parity > gpurun_out/jj_nfb_$r.log 2>&1
echo "nofence bf16 r$r $(python scripts/ab_line.py gpurun_out/jj_nfb_$r.log)" | tee -a gpurun_out/ab_jj.txt
done
