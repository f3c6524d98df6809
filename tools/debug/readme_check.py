import os, sys; sys.path.insert(0, os.getcwd())
import numpy as np, paper_2310_16795_b200 as q
rng = np.random.default_rng(0)
dic = q.generate_dictionary()
w = (rng.normal(size=(64, 128)) * 0.02).astype(np.float32)
x = q.bf16_round(rng.normal(size=128).astype(np.float32))
c = q.encode(q.rtn_quantize(w, q.make_grid(w)), dic)
y = q.fused_matvec(c, x, dic)
E, dm, dff = 4, 128, 256
wi = [q.encode(q.rtn_quantize(m, q.make_grid(m)), dic) for m in [(rng.normal(size=(dff, dm)) * 0.02).astype(np.float32) for _ in range(E)]]
wo = [q.encode(q.rtn_quantize(m, q.make_grid(m)), dic) for m in [(rng.normal(size=(dm, dff)) * 0.02).astype(np.float32) for _ in range(E)]]
layer = q.CompressedMoELayer([a.to_device(dic) for a in wi], [b.to_device(dic) for b in wo], dic)
tokens = q.bf16_round(rng.normal(size=(8, dm)).astype(np.float32))
ids = q.RouterSim(E, rule="argmax", seed=0).assign(tokens)
out = layer.forward(tokens, ids)
batches = [q.bf16_round(rng.normal(size=(8, dm)).astype(np.float32)) for _ in range(3)]
outs = list(q.forward_stream((layer, t, q.RouterSim(E).assign(t)) for t in batches))
print("README snippet OK", y.shape, out.shape, len(outs))
