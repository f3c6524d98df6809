"""Host API timing: blocking forward() per step vs forward_stream at depth
1-3 (cold pool of layers, Switch-base-128, T = 64)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import build_layer
dic = q.generate_dictionary()
L = 10
layers = [build_layer(128, 768, 3072, seed=s, dic=dic, max_tokens=64) for s in range(L)]
rng = np.random.default_rng(0)
xs = [q.bf16_round(rng.normal(size=(64, 768)).astype(np.float32)) for _ in range(4)]
router = q.RouterSim(128, rule="argmax", seed=0)
asg = [router.assign(x) for x in xs]
items = lambda n: ((layers[i % L], xs[i % 4], asg[i % 4]) for i in range(n))
N = 200
for depth in (1, 2, 3):
    for _ in q.forward_stream(items(3 * L), depth=depth):
        pass
for rep in range(2):
    t0 = time.perf_counter()
    for lay, x, a in items(N):
        lay.forward(x, a)
    print("forward", round((time.perf_counter() - t0) / N * 1e6, 1), "us/step")
    for depth in (1, 2, 3):
        t0 = time.perf_counter()
        for _ in q.forward_stream(items(N), depth=depth):
            pass
        print("stream depth", depth, round((time.perf_counter() - t0) / N * 1e6, 1), "us/step")
g = torch.cuda.CUDAGraph()
# device-only reference: the graphs back to back without host work
sts = [lay._stages[(64, False, 0)] for lay in layers]
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    sts[i % L]["graphs"][True].replay()
torch.cuda.synchronize()
print("graphs back to back (no host staging)", round((time.perf_counter() - t0) / N * 1e6, 1), "us/step")
