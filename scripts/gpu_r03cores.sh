# w2 CTAs co-resident with the w1/w3 GEMM at the rank shapes: early pre-wait stages (e88) + smaller rings (e35: 3 / 5, e43: 4 / 3 stages)
O=gpurun_out/r03cores; mkdir -p $O
MOE_LIB=build_ab/libmoe_e35.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ep or tp or decode" > $O/pytest_e35.txt 2>&1; echo "pytest e35 $?"; tail -n 1 $O/pytest_e35.txt
for s in ep8 tp8 ep4 tp4; do bash scripts/ab_lib_shard.sh cr_$s "base e88 e35 e43" 2 "--shard $s --steps 50 --warmup 3" > /dev/null 2>&1; done
bash scripts/ab_lib_shard.sh cr_dec2k "base e35" 2 "--steps 100 --warmup 5 --tuning fused=1" > /dev/null 2>&1
cat gpurun_out/abl_cr_*.txt | cut -c1-130
