"""Six small-ffn decode forwards (T from argv) for an ncu capture of the router / permute /
combine kernels: ncu ... -k regex:"router|permute|combine" python scripts/exp/rl1.py 64"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2408_00008_b200 as moe
T = int(sys.argv[1])
w = synth.make_weights(4096, 1024, 8, seed=0, device="cuda")
x = synth.make_tokens(T, 4096, seed=1, device="cuda")
blk = moe.MoEBlock(w["wg"], w["w1"], w["w3"], w["w2"], max_tokens=64)
for _ in range(6):
    blk.forward(x)
torch.cuda.synchronize()
