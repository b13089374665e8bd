"""Routing and residual-stream rms per layer of the 32-layer C5 stack (one GPU): expert
counts and output rms at layers 0..31 for the single-layer weight recipe (W2 std 1/sqrt(f))
and the stack recipe (synth.STACK_W2_SCALE). python scripts/exp/stack_counts.py"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2408_00008_b200 as moe  # noqa: E402

d, f, E, L = 4096, 14336, 8, 32
for scale in (1.0, synth.STACK_W2_SCALE):
    st = None
    for l in range(L):
        lw = synth.make_weights(d, f, E, seed=0, layer=l, device="cuda", w2_scale=scale)
        if st is None:
            st = moe.MoEStack([lw], top_k=2, max_tokens=575)
        else:
            st.add_layer(lw)
        del lw
    torch.cuda.empty_cache()
    for T in (64, 575):
        x = synth.make_tokens(T, d, seed=1, device="cuda")
        aux = [{"expert_counts": torch.empty(E, dtype=torch.int32, device="cuda")} for _ in range(L)]
        outs = []
        st.forward(x, layer_aux=aux, layer_outputs=outs)
        torch.cuda.synchronize()
        for l in (0, 1, 2, 4, 8, 16, 24, 31):
            print(f"w2_scale={scale} T={T} layer {l}: counts {aux[l]['expert_counts'].tolist()} "
                  f"rms {float(outs[l].float().pow(2).mean().sqrt()):.4g}", flush=True)
        del outs
    st.close()
    del st
    torch.cuda.empty_cache()
