# pre-wait L2 prefetch depth of the decode GEMMs (tuning g1_pf_l2 / g2_pf_l2): decode + stack M1, interleaved
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/ab_env.sh "g2_pf_l2=0 g2_pf_l2=32 g2_pf_l2=96 g2_pf_l2=224 g1_pf_l2=0" 3 --no-parity
for r in 1 2; do for t in "" "--tuning g2_pf_l2=96" "--tuning g2_pf_l2=224" "--tuning g1_pf_l2=16,g2_pf_l2=96"; do
  timeout -s KILL 600 python bench.py --config stack --stack-batch M1 --steps 5 --warmup 3 --no-cpu-baseline --no-parity $t 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('[$t]', $r, round(j['ms_per_step'],3), round(j['value']), 'hbm', round(j['step_roofline_frac'],3), {k: round(v*1000,1) for k,v in j['kernel_ms_per_launch'].items()}, j['clocks']['sm_mhz'])"
done; done
