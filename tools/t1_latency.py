"""Per-layer latency of the fused MoE step at T=1 (token generation), with
several layers' steps captured back to back in ONE CUDA graph (as a model
forward would), so graph-launch overhead is amortised. Experiment harness."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
wl = os.environ.get("WORKLOAD", "switch-base-128")
E, d_model, d_ff = WORKLOADS[wl]
E = int(os.environ.get("EXPERTS", E))
NL = int(os.environ.get("LAYERS", 8))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
layers = [build_layer(E, d_model, d_ff, seed=l, dic=dic, device=dev, max_tokens=8) for l in range(NL)]
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
for T in (1, 8):
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    a = router.assign(x)
    xd = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    ad = torch.from_numpy(a).to(dev)
    outs = [torch.empty((T, d_model), device=dev) for _ in range(NL)]

    def fwd():
        for l in range(NL):
            layers[l].forward_device(xd, ad, out=outs[l])
    fwd()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fwd()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (20 * NL) * 1e3
    ne = len(np.unique(a))
    sol = ne * 2 * d_model * d_ff * 2 / (peak * 1e9) * 1e6
    print(json.dumps({"workload": wl, "experts": E, "T": T, "layers_per_graph": NL, "us_per_layer": round(us, 2),
                      "bf16_sol_us_per_layer": round(sol, 2)}), flush=True)
