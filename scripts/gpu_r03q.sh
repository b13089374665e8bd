# spec L2 prefetch depth sweep: decode, T=575 single layer, tp8 stack rank, 32-layer M1
bash scripts/ab_tunings.sh q_dec 2 "" - spec_l2=-1 spec_l2=8 spec_l2=16
bash scripts/ab_tunings.sh q_tp1st 2 "--shard tp1 --config stack --steps 20 --warmup 3" - spec_l2=-1 spec_l2=8 spec_l2=16
bash scripts/ab_tunings.sh q_tp8st 2 "--shard tp8 --config stack --steps 20 --warmup 3" - spec_l2=-1 spec_l2=8 spec_l2=16
bash scripts/ab_tunings.sh q_M1 2 "--config stack --stack-batch M1 --steps 10 --warmup 3" - spec_l2=-1 spec_l2=8 spec_l2=16
