"""Fixed cost of the fused step by token count: all tokens dropped (ids -1)
-> only the plan and empty phases run; chains of 10 steps in a CUDA graph."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import build_layer
dic = q.generate_dictionary()
layers = [build_layer(128, 768, 3072, seed=s, dic=dic, max_tokens=256) for s in range(10)]
for T in (1, 8, 32, 64, 128, 256):
    x = torch.zeros((T, 768), device="cuda", dtype=torch.bfloat16)
    a = torch.full((T,), -1, dtype=torch.int32, device="cuda")
    a[T - 1] = 3  # one valid token: the phases run one expert
    outs = [torch.empty((T, 768), device="cuda") for _ in layers]
    def chain():
        for i, l in enumerate(layers):
            l.forward_device(x, a, out=outs[i])
    chain(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        chain()
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(T, "one valid token among T: us per step", round(e0.elapsed_time(e1) * 1e3 / 500, 2))
