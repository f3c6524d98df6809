import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer
dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
for wl in ("switch-base-128", "switch-large-128"):
    E, dm, dff = WORKLOADS[wl]
    lay = build_layer(E, dm, dff, seed=0, dic=dic, device=dev, max_tokens=64)
    cws = []
    for m in list(lay.wi)[:16] + list(lay.wo)[:16]:
        cws.append(m.cw[: m.n_codewords].to(torch.int32).cpu().numpy() & 0xFFFF)
    c = np.concatenate(cws)
    print(wl, "codewords", len(c), {H: round(float(np.mean(c < H)), 4) for H in (1024, 2048, 4096, 8192, 16384, 32768, 49152)})
