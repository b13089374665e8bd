"""Experiment: does tcgen05 kind::f16 accept A = fp16 with B = bf16? Swap-AB decode path with
fp16 weight bytes (build_ab/libmoe_af16.so reads the swap GEMMs' A operand as fp16)."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
os.environ["MOE_LIB"] = "build_ab/libmoe_af16.so"
import numpy as np, torch
import synth, oracle
import paper_2408_00008_b200 as moe
from parity import rel_err
shape = synth.MoEShape(T=64, d=512, f=1024, E=8, k=2)
inp = synth.make_inputs(shape, 3, device="cuda", dtype=torch.float32)
x = inp["x"].to(torch.bfloat16); wg = inp["wg"].to(torch.bfloat16)
w16 = {n: inp[n].to(torch.float16) for n in ("w1", "w3", "w2")}
fake = {n: v.view(torch.bfloat16) for n, v in w16.items()}  # fp16 bytes through the bf16 packer
blk = moe.MoEBlock(wg, fake["w1"], fake["w3"], fake["w2"], top_k=2, max_tokens=64, flags=moe.MOE_FLAG_FORCE_SWAP)
aux = {"out_f32": torch.empty(64, 512, device="cuda"), "topk_idx": torch.empty(64, 2, dtype=torch.int32, device="cuda")}
out = blk.forward(x, aux=aux); torch.cuda.synchronize()
h = {"x": x.float().cpu().numpy().astype(np.float64), "wg": wg.float().cpu().numpy().astype(np.float64)}
for n in w16: h[n] = w16[n].float().cpu().numpy().astype(np.float64)
y = oracle.moe_forward(h["x"], h["wg"], h["w1"], h["w3"], h["w2"], 2, forced_idx=aux["topk_idx"].cpu().numpy())
print("mixed A=f16 B=bf16 max rel err:", rel_err(aux["out_f32"].cpu().numpy(), y).max())
