"""Config 5 on one B200: a full synthetic Switch-c2048-shaped compressed model
(MoE layers only: 30 x 2048 experts x (wi 6144x2080 + wo 2080x6144), random-init
weights, ~130 GB compressed, all resident in HBM), forward of T tokens through
every layer as a CompressedMoEModel: per layer the device router (RouterSim
hash rule, bit-exact) and one fused launch computing x + moe(x) in bf16 (the
next layer's input), captured as one CUDA graph. Reports tokens/s and
per-layer latency next to the uncompressed bf16 HBM speed of light (a bf16
c2048 model is 3.1 TB: it cannot be resident on one GPU at all).
Usage: LAYERS=30 python tools/c2048_model.py [T ...]"""
import os, sys, json, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
E, d_model, d_ff = WORKLOADS["switch-c2048"]
NL = int(os.environ.get("LAYERS", 30))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
Ts = [int(t) for t in sys.argv[1:]] or [1, 8, 64]
t0 = time.time()
layers = []
for l in range(NL):
    layers.append(build_layer(E, d_model, d_ff, seed=l, dic=dic, device=dev, max_tokens=max(Ts)))
    torch.cuda.empty_cache()
nbytes = sum(int(lay.expert_bytes.sum()) for lay in layers)
print(json.dumps({"layers": NL, "experts": E, "built_s": round(time.time() - t0, 1), "compressed_GB": round(nbytes / 1e9, 2),
                  "bits_per_param": round(nbytes * 8 / (NL * E * 2 * d_model * d_ff), 3),
                  "hbm_used_GB": round(torch.cuda.memory_allocated() / 1e9, 1)}), flush=True)
# the model: residual blocks, RouterSim hash routing per layer ON THE DEVICE
# (bit-exact with the reference's rule), one fused launch per block
routers = [q.DeviceRouter(q.RouterSim(E, rule="hash", seed=l), d_model) for l in range(NL)]
model = q.CompressedMoEModel(layers, routers)
rng = np.random.default_rng(0)
for T in Ts:
    x0 = torch.from_numpy(q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))).to(dev).to(torch.bfloat16)
    _, trace = model.forward_device(x0, keep=True)  # routing of this input, per layer (for the byte count)
    ids = [t[1].cpu().numpy() for t in trace]
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        model.forward_device(x0)
    torch.cuda.current_stream().wait_stream(s_)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        model.forward_device(x0)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    touched = sum(len(np.unique(i)) for i in ids)
    sol_ms = touched * 2 * d_model * d_ff * 2 / (peak * 1e9) * 1e3
    cbytes = sum(layers[l].touched_bytes(ids[l]) for l in range(NL))
    print(json.dumps({"T": T, "forward_ms": round(ms, 3), "us_per_layer": round(1e3 * ms / NL, 2),
                      "tokens_per_s": round(T / ms * 1e3), "compressed_GBps": round(cbytes / ms / 1e6, 1),
                      "bf16_sol_ms": round(sol_ms, 3), "speedup_vs_bf16_sol": round(sol_ms / ms, 2),
                      "what": "residual blocks: device hash router + fused resid step per layer, one CUDA graph"}),
          flush=True)
