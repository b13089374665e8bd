# bf16 fused FFN with 128-row w2 tiles x two K blocks per stage (MOE_FUSED_BF16_G2_128, build_ab/libmoe_g2p.so)
# vs the default 256-row w2 tiles; plus the FP8 in-kernel combine fix on the default build
O=gpurun_out/r03g2p; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_fused.py -m gpu -x -q > $O/pytest_default.txt 2>&1; echo "default $?"
MOE_LIB=build_ab/libmoe_g2p.so timeout -s KILL 900 python -m pytest tests/test_fused.py -m gpu -x -q -k "not fp8" > $O/pytest_g2p.txt 2>&1; echo "g2p $?"
tail -3 $O/pytest_default.txt $O/pytest_g2p.txt
cp paper_2408_00008_b200/libmoe.so build_ab/libmoe_def.so
bash scripts/ab_decode.sh "def g2p" 4 > $O/ab.txt 2>&1
cat $O/ab.txt
