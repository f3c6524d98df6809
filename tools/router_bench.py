"""Device router (qmoe_route) latency: CUDA-graph replay of router alone, and
of router + fused step (Switch-base-128), for several token counts."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)


def replay_us(fn, n=200):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for E, d in ((128, 768), (2048, 2080)):
    for rule in ("argmax", "hash"):
        r = q.DeviceRouter(q.RouterSim(E, rule=rule, seed=0), d, dev)
        for T in (1, 64, 256):
            x = torch.randn(T, d, device=dev).to(torch.bfloat16)
            print(f"router {rule} E={E} d={d} T={T}: {replay_us(lambda: r(x, gated=True)):.1f} us per step (graph)")
dic = q.generate_dictionary()
E, dm, dff = WORKLOADS["switch-base-128"]
lay = build_layer(E, dm, dff, seed=0, dic=dic, device=dev, max_tokens=256)
r = q.DeviceRouter(q.RouterSim(E, rule="argmax", seed=0), dm, dev)
for T in (1, 64):
    x = torch.randn(T, dm, device=dev).to(torch.bfloat16)
    out = torch.empty(T, dm, device=dev)
    a = r(x)[0]
    print(f"step alone T={T}: {replay_us(lambda: lay.forward_device(x, a, out=out)):.1f} us; "
          f"router + gated step: {replay_us(lambda: lay.forward_routed(x, r, gated=True, out=out)):.1f} us (one layer, warm L2)")
