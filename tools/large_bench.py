"""Config 3 (Switch-large-128, batched tokens): MoE step time of the
decode-then-MMA path vs the streaming path vs bf16 (grouped bf16 GEMM and HBM
speed-of-light). Experiment harness; numbers go to DESIGN.md."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
wl = os.environ.get("WORKLOAD", "switch-large-128")
E, d_model, d_ff = WORKLOADS[wl]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
L2 = 126 << 20
layers, pool = [], 0
Tmax = max(int(t) for t in sys.argv[1:]) if len(sys.argv) > 1 else 4096
while pool < 4 * L2:
    lay = build_layer(E, d_model, d_ff, seed=len(layers), dic=dic, device=dev, max_tokens=Tmax)
    layers.append(lay)
    pool += int(lay.expert_bytes.sum())
L = len(layers)
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
Wi = torch.randn((E, d_ff, d_model), device=dev, dtype=torch.bfloat16) * 0.02
Wo = torch.randn((E, d_model, d_ff), device=dev, dtype=torch.bfloat16) * 0.02


def timed(fn, n):
    for i in range(max(3, n)):  # every pooled layer once before capture (lazy per-layer setup)
        fn(i)
    torch.cuda.synchronize()
    graphs = []
    for i in range(n):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(i)
        graphs.append(g)
    for g in graphs:
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        for g in graphs:
            g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * n) * 1e3


for T in [int(t) for t in sys.argv[1:]] or [256, 1024, 4096]:
    xs = [q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32)) for _ in range(2)]
    asg = [router.assign(x) for x in xs]
    xd = [torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in xs]
    ad = [torch.from_numpy(a).to(dev) for a in asg]
    outs = [torch.empty((T, d_model), device=dev) for _ in range(L)]
    res = {}
    for mode in ("always", "never"):
        for lay in layers:
            lay.dense_mode = mode
        res["dense" if mode == "always" else "stream"] = timed(
            lambda i: layers[i % L].forward_device(xd[i % 2], ad[i % 2], out=outs[i % L]), 2 * L)
    # bf16: tokens sorted by expert, two grouped bf16 GEMMs (torch._grouped_mm), CUDA graph
    plans = []
    for a in asg:
        plans.append((torch.from_numpy(np.argsort(a, kind="stable")).to(dev),
                      torch.from_numpy(np.cumsum(np.bincount(a, minlength=E)).astype(np.int32)).to(dev)))
    yb = [torch.empty((T, d_model), device=dev, dtype=torch.bfloat16) for _ in range(2)]

    def bf16_step(i):
        b = i % 2
        order, offs = plans[b]
        h = torch.relu(torch._grouped_mm(xd[b].index_select(0, order), Wi.transpose(1, 2), offs=offs))
        yb[b].index_copy_(0, order, torch._grouped_mm(h, Wo.transpose(1, 2), offs=offs))
    res["bf16_grouped_gemm"] = timed(bf16_step, 2)
    ne = np.mean([len(np.unique(a)) for a in asg])
    res["bf16_sol"] = ne * 2 * d_model * d_ff * 2 / (peak * 1e9) * 1e6
    cbytes = np.mean([layers[0].touched_bytes(a) for a in asg])
    print(json.dumps({"workload": wl, "T": T, "experts_touched": ne, "step_us": {k: round(v, 1) for k, v in res.items()},
                      "tokens_per_s_dense": T / res["dense"] * 1e6, "compressed_GBps_dense": cbytes / res["dense"] / 1e3}),
          flush=True)
