"""Fixed cost of one fused step: all tokens dropped (ids -1) vs a real T=1
step, both as chains of 10 steps in a CUDA graph; plus empty-kernel launch floor."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200 import _lib
from paper_2310_16795_b200.synth import build_layer
dic = q.generate_dictionary()
layers = [build_layer(128, 768, 3072, seed=s, dic=dic, max_tokens=8) for s in range(10)]
x = torch.from_numpy(q.bf16_round(np.random.default_rng(0).normal(size=(1, 768)).astype(np.float32))).cuda().to(torch.bfloat16)
for name, ids in (("dropped", [-1]), ("T=1", [5])):
    a = torch.tensor(ids, dtype=torch.int32, device="cuda")
    outs = [torch.empty((1, 768), device="cuda") for _ in layers]
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
    print(name, "us per step", e0.elapsed_time(e1) * 1e3 / 500)
# empty kernel floor with the step's launch shape (cooperative, 768 threads, ~200 KB smem)
def empty_chain():
    for _ in range(10):
        _lib.check(_lib.lib.qmoe_debug_empty_launch(200 * 1024, 768 | (1 << 16), _lib.stream_ptr()))
empty_chain(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    empty_chain()
for _ in range(5): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): g.replay()
e1.record(); torch.cuda.synchronize()
print("empty cooperative 768x200KB us per launch", e0.elapsed_time(e1) * 1e3 / 500)
