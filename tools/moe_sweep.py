"""MoE-step timing sweep (experiment harness): a pool of distinct layers
(> 4x L2, cold), T tokens per step, graphs of 10 consecutive layer steps (a
forward's launch pattern), CUDA events. Prints one line per T:
  T step_us GB/s
Usage: [QMOE_LIB_PATH=variants/x/libqmoe.so] python tools/moe_sweep.py [T ...]
Env: WORKLOAD (default switch-base-128), HOT (per-step hot-table cap),
LG="wi,wo" (lanes per row override)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q  # noqa: E402
from paper_2310_16795_b200.synth import WORKLOADS, build_layer  # noqa: E402

Ts = [int(t) for t in sys.argv[1:]] or [1, 8, 64]
wl = os.environ.get("WORKLOAD", "switch-base-128")
E, d_model, d_ff = WORKLOADS[wl]
dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
L2 = 126 << 20
layers, pool = [], 0
while pool < 4 * L2:
    lay = build_layer(E, d_model, d_ff, seed=len(layers), dic=dic, device=dev, max_tokens=max(Ts))
    if "HOT" in os.environ:  # hot-table entries staged per step (overrides the size rule)
        lay.STEP_HOT_MAX = int(os.environ["HOT"])
        lay.hot_entries = lambda T, wi, h=int(os.environ["HOT"]): h
    if "LG" in os.environ:  # "wi,wo": lanes per row (log2) for every T (bounded by the checkpoints)
        lgs = tuple(min(int(v), c) for v, c in zip(os.environ["LG"].split(","), lay.max_lg))
        for T in Ts:
            lay._lanes[T] = lgs
    layers.append(lay)
    pool += int(lay.expert_bytes.sum())
L = len(layers)
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
lib = os.environ.get("QMOE_LIB_PATH", "product")
for T in Ts:
    nb = 4
    xs = [q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32)) for _ in range(nb)]
    asg = [router.assign(x) for x in xs]
    xd = [torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in xs]
    ad = [torch.from_numpy(a).to(dev) for a in asg]
    outs = [torch.empty((T, d_model), device=dev) for _ in layers]
    C = 10
    nch = max(1, L * nb // C)

    def chain(j):
        for u in range(C):
            i = j * C + u
            layers[i % L].forward_device(xd[i % nb], ad[i % nb], out=outs[i % L])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        chain(0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graphs = []
    for j in range(nch):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            chain(j)
        graphs.append(g)
    for g in graphs:
        g.replay()
    torch.cuda.synchronize()
    reps = max(2, 40 // nch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for g in graphs:
            g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * nch * C)
    nbytes = np.mean([layers[i % L].touched_bytes(asg[i % nb]) for i in range(nch * C)])
    print(f"{lib} {wl} lg={layers[0].lanes_per_row(T)} T={T} step {us:.2f} us  {nbytes / us / 1e3:.1f} GB/s", flush=True)
    del graphs
