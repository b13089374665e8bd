python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/ab_env.sh "spec_l2=-1 spec_l2=0 spec_l2=8 spec_l2=16" 4 --fp8 --no-parity --steps 400
