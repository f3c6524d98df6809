"""Config 4 on one GPU: a Switch-c2048-shaped layer (2048 experts, d_model
2080, d_ff 6144, ~4.3 GB compressed) built on the GPU, one step per T tokens
(fused single-launch path), vs the uncompressed bf16 step's HBM speed of light
(a bf16 c2048 layer is 105 GB: its SOL is computed, the 8-GPU EP run shards it).
Experiment harness; numbers go to DESIGN.md."""
import os, sys, json, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
E, d_model, d_ff = WORKLOADS["switch-c2048"]
E = int(os.environ.get("C2048_EXPERTS", E))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
t0 = time.time()
lay = build_layer(E, d_model, d_ff, seed=0, dic=dic, device=dev, max_tokens=1024)
print(f"built {E} experts in {time.time() - t0:.1f} s, {lay.expert_bytes.sum() / 1e9:.2f} GB compressed, "
      f"{lay.expert_bytes.sum() * 8 / (E * 2 * d_model * d_ff):.3f} bits/param", flush=True)
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
for T in [int(t) for t in sys.argv[1:]] or [1, 8, 64, 256]:
    xs = [q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32)) for _ in range(4)]
    asg = [router.assign(x) for x in xs]
    xd = [torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in xs]
    ad = [torch.from_numpy(a).to(dev) for a in asg]
    out = torch.empty((T, d_model), device=dev)
    for i in range(3):
        lay.forward_device(xd[i % 4], ad[i % 4], out=out)
    graphs = []
    for i in range(4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            lay.forward_device(xd[i], ad[i], out=out)
        graphs.append(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        for g in graphs:
            g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    cbytes = np.mean([lay.touched_bytes(a) for a in asg])
    ne = np.mean([len(np.unique(a)) for a in asg])
    sol = ne * 2 * d_model * d_ff * 2 / (peak * 1e9) * 1e6
    print(json.dumps({"workload": "switch-c2048 (1 GPU, all experts resident)", "T": T, "experts_touched": ne,
                      "step_us": round(us, 1), "compressed_GBps": round(cbytes / us / 1e3, 1),
                      "pct_hbm": round(100 * cbytes / us / 1e3 / peak, 2), "tokens_per_s": round(T / us * 1e6),
                      "bf16_sol_us": round(sol, 1), "speedup_vs_bf16_sol": round(sol / us, 2)}), flush=True)
