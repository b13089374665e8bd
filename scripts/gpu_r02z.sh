# full GPU suite + compute-sanitizer (incl. the CTA-pair swap kernels) + stack shard sweep (pair auto vs off)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/gpu_tests.sh z
bash scripts/sanitize.sh gpurun_out/sanitizer_z
SHARDS="tp1 ep2 ep4 ep8 tp2 tp4 tp8" bash scripts/shard_sweep.sh zpair stack
SHARDS="tp1 ep2 ep4 ep8 tp2 tp4 tp8" bash scripts/shard_sweep.sh zsingle stack --tuning swap_pair=1
