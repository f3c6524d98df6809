"""T = 1 step chain (10 distinct layers, one CUDA graph) for profiling the
latency-bound one-token step: `ncu -k moe_step_kernel ... python tools/debug/t1_chain.py`."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import build_layer
T = int(os.environ.get("T", 1))
dic = q.generate_dictionary()
layers = [build_layer(128, 768, 3072, seed=s, dic=dic, max_tokens=max(8, T)) for s in range(10)]
x = torch.from_numpy(q.bf16_round(np.random.default_rng(0).normal(size=(T, 768)).astype(np.float32))).cuda().to(torch.bfloat16)
a = torch.from_numpy(q.RouterSim(128, rule="argmax", seed=0).assign(x.float().cpu().numpy())).cuda()
outs = [torch.empty((T, 768), device="cuda") for _ in layers]
def chain():
    for i, l in enumerate(layers):
        l.forward_device(x, a, out=outs[i])
chain(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    chain()
for _ in range(int(os.environ.get("REPS", 5))): g.replay()
torch.cuda.synchronize()
print("done")
