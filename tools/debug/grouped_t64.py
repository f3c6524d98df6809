"""Per-launch times of the grouped path (plan kernel + wi pass + wo pass) vs the
fused step, same layers and tokens (run under ncu --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import build_layer
dic = q.generate_dictionary()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
layers = [build_layer(128, 768, 3072, seed=s, dic=dic, max_tokens=T) for s in range(10)]
x = torch.from_numpy(q.bf16_round(np.random.default_rng(0).normal(size=(T, 768)).astype(np.float32))).cuda().to(torch.bfloat16)
a = torch.from_numpy(q.RouterSim(128, rule="argmax", seed=0).assign(x.float().cpu().numpy())).cuda()
for i in range(20):
    l = layers[i % 10]
    l.fused = (i % 2 == 0)
    l.forward_device(x, a)
torch.cuda.synchronize()
