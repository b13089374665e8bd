O=gpurun_out/r03ncufinal; mkdir -p $O
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_ffn_fused" -s 2 -c 1 -o $O/prof_decode_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > $O/ncu.log 2>&1; echo "ncu $?"
ls -la $O
