"""Phase timeline of the fused MoE step (debug hook qmoe_debug_step_trace):
per-CTA %globaltimer stamps -> when the plan, wi and wo phases end."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200 import _lib
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
wl = os.environ.get("WORKLOAD", "switch-base-128")
E, d_model, d_ff = WORKLOADS[wl]
layers = [build_layer(E, d_model, d_ff, seed=s, dic=dic, device=dev, max_tokens=256) for s in range(4)]
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
buf = torch.zeros(148 * 8, dtype=torch.int64, device=dev)
for T in [int(t) for t in sys.argv[1:]] or [1, 8, 64]:
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    a = router.assign(x)
    xd = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    ad = torch.from_numpy(a).to(dev)
    for i in range(3):
        layers[i % 4].forward_device(xd, ad)
    torch.cuda.synchronize()
    _lib.check(_lib.lib.qmoe_debug_step_trace(_lib.ptr(buf)))
    buf.zero_()
    layers[3].forward_device(xd, ad)
    torch.cuda.synchronize()
    _lib.check(_lib.lib.qmoe_debug_step_trace(None))
    t = buf.view(148, 8)[:, :4].cpu().numpy().astype(np.int64)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    wi_d = r[:, 2] - r[:, 1]
    wo_d = r[:, 3] - r[:, 2]
    print("   wi phase us percentiles 10/50/90/max:", np.percentile(wi_d, [10, 50, 90, 100]).round(1),
          " wo phase:", np.percentile(wo_d, [10, 50, 90, 100]).round(1),
          " slowest-wo CTAs:", np.argsort(-r[:, 3])[:6])
    print(f"T={T}: start {np.median(r[:,0]):.1f}/{r[:,0].max():.1f}  plan {np.median(r[:,1]):.1f}/{r[:,1].max():.1f}  "
          f"wi {np.median(r[:,2]):.1f}/{r[:,2].max():.1f}  wo {np.median(r[:,3]):.1f}/{r[:,3].max():.1f} us (median/max over CTAs)")
