"""MoE-step timing sweep (experiment harness): Switch-base-128 layer pool,
T tokens, CUDA-graph replay of one step, for a given hot-table size
(QMOE_HOT_ENTRIES, read once per process). Prints one line per run:
  H T step_us wi_us wo_us plan_us GB/s
Usage: python tools/moe_sweep.py [H] [T ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q  # noqa: E402
from paper_2310_16795_b200.synth import WORKLOADS, build_layer  # noqa: E402

H = sys.argv[1] if len(sys.argv) > 1 else "-1"
if H != "-1":
    os.environ["QMOE_HOT_ENTRIES"] = H
Ts = [int(t) for t in sys.argv[2:]] or [64]
wl = os.environ.get("WORKLOAD", "switch-base-128")
E, d_model, d_ff = WORKLOADS[wl]
dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
L2 = 126 << 20
layers, pool = [], 0
while pool < 4 * L2:
    lay = build_layer(E, d_model, d_ff, seed=len(layers), dic=dic, device=dev, max_tokens=max(Ts))
    layers.append(lay)
    pool += int(lay.expert_bytes.sum())
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
for T in Ts:
    xs = [q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32)) for _ in range(4)]
    asg = [router.assign(x) for x in xs]
    xd = [torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in xs]
    ad = [torch.from_numpy(a).to(dev) for a in asg]
    outs = [torch.empty((T, d_model), device=dev) for _ in layers]
    L = len(layers)
    n = L * 4
    graphs = []
    for i in range(n):
        layers[i % L].forward_device(xd[i % 4], ad[i % 4], out=outs[i % L])
    torch.cuda.synchronize()
    if os.environ.get("ONEGRAPH") == "1":  # all n steps in one graph (a model forward's launch pattern)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(n):
                layers[i % L].forward_device(xd[i % 4], ad[i % 4], out=outs[i % L])
        graphs.append(g)
        n_per_graph = n
    else:
        n_per_graph = 1
        for i in range(n):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                layers[i % L].forward_device(xd[i % 4], ad[i % 4], out=outs[i % L])
            graphs.append(g)
    for g in graphs:
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        for g in graphs:
            g.replay()
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / (reps * len(graphs) * n_per_graph) * 1e3
    nbytes = np.mean([layers[i % L].touched_bytes(asg[i % 4]) for i in range(n)])
    # per-pass timings (outside graphs)
    s = torch.cuda.current_stream()
    tw = {"plan": [], "wi": [], "wo": []}
    for i in range(n):
        lay = layers[i % L]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s)
        lay.plan(ad[i % 4], s)
        ev[1].record(s)
        lay.pass_wi(xd[i % 4], s)
        ev[2].record(s)
        lay.pass_wo(outs[i % L], s)
        ev[3].record(s)
        torch.cuda.synchronize()
        tw["plan"].append(ev[0].elapsed_time(ev[1]) * 1e3)
        tw["wi"].append(ev[1].elapsed_time(ev[2]) * 1e3)
        tw["wo"].append(ev[2].elapsed_time(ev[3]) * 1e3)
    print(f"H={H} T={T} step_us={step:.1f} wi_us={np.median(tw['wi']):.1f} wo_us={np.median(tw['wo']):.1f} "
          f"plan_us={np.median(tw['plan']):.1f} GB/s={nbytes / step / 1e3:.1f} experts={np.mean([len(np.unique(a)) for a in asg]):.1f}",
          flush=True)
