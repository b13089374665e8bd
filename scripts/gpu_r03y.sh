O=gpurun_out/r03y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_ffn_fused" -s 2 -c 1 -o $O/prof_fp8_fused python bench.py --fp8 --steps 1 --warmup 3 --no-cpu-baseline --no-parity > $O/ncu1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_fp8x" -s 4 -c 2 -o $O/prof_fp8_two python bench.py --fp8 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --tuning fused=1 > $O/ncu2.log 2>&1
ls $O
