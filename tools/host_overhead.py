import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer
dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
E, dm, dff = WORKLOADS["switch-base-128"]
lay = build_layer(E, dm, dff, seed=0, dic=dic, device=dev, max_tokens=64)
x = q.bf16_round(np.random.default_rng(0).normal(size=(64, dm)).astype(np.float32))
a = q.RouterSim(E, rule="argmax", seed=0).assign(x)
for _ in range(20): lay.forward(x, a)
st = next(iter(lay._stages.values())); g = st["graphs"][False]; s = torch.cuda.current_stream()
N = 500
def tm(fn):
    for _ in range(20): fn()
    t0 = time.perf_counter()
    for _ in range(N): fn()
    return (time.perf_counter() - t0) / N * 1e6
print("forward", tm(lambda: lay.forward(x, a)))
print("replay+event sync", tm(lambda: (g.replay(), st["done"].record(), st["done"].synchronize())))
print("replay+stream sync", tm(lambda: (g.replay(), s.synchronize())))
print("replay+cuda sync", tm(lambda: (g.replay(), torch.cuda.synchronize())))
print("replay only (no sync)", tm(lambda: g.replay())); torch.cuda.synchronize()
print("event record+sync alone", tm(lambda: (st["done"].record(), st["done"].synchronize())))
print("copyto x", tm(lambda: np.copyto(st["xv"], x)))
print("copy out", tm(lambda: st["yv"].copy()))
print("use_dense", tm(lambda: lay.use_dense(64)))
