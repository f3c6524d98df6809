import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2310_16795_b200 as q
from oracle import qmoe_oracle as O
from paper_2310_16795_b200.synth import build_layer
from test_gpu_fullshape import host_streams
from conftest import bf16_ulp_diff
dic = q.generate_dictionary(); odic = O.OracleDictionary(0.885, dic.decode_words)
layer = build_layer(128, 768, 3072, seed=21, dic=dic, max_tokens=64)
T = 64
rng = np.random.default_rng(1000 + T)
x = q.bf16_round(rng.normal(size=(T, 768)).astype(np.float32))
assign = q.RouterSim(128, rule="argmax", seed=0).assign(x)
y = layer.forward_device(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(assign).cuda()).cpu().numpy()
h_gpu = layer.h.float().cpu().numpy()
toks = np.sort(rng.choice(T, size=16, replace=False))
for t in toks:
    e = int(assign[t]); wi, wo = host_streams(layer.wi[e]), host_streams(layer.wo[e])
    h = np.maximum(O.fused_matvec(*wi[:2], *wi[2:], odic.hash64, x[t], odic, workers=8), 0)
    yr = O.fused_matvec(*wo[:2], *wo[2:], odic.hash64, h, odic, workers=8)
    dh = bf16_ulp_diff(h_gpu[t, :3072], h); dy = bf16_ulp_diff(y[t], yr)
    # also: GPU wo on the ORACLE h (isolate the wo pass)
    print(t, e, "h maxulp", dh.max(), "h diffs", int((dh > 0).sum()), "y maxulp", dy.max(), "y diffs", int((dy>0).sum()),
          "at", int(dy.argmax()), y[t, dy.argmax()], yr[dy.argmax()])
    if dy.max() > 2:
        # recompute y with oracle from GPU h: is the wo pass exact given h?
        yr2 = O.fused_matvec(*wo[:2], *wo[2:], odic.hash64, h_gpu[t, :3072].copy(), odic, workers=8)
        print("   y from gpu h vs gpu y: maxulp", bf16_ulp_diff(y[t], yr2).max())
