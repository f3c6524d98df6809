"""Where the host-API step's time goes (CompressedMoELayer.forward, T tokens):
numpy -> pinned copy, graph replay + sync, pinned -> numpy copy."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200.synth import WORKLOADS, build_layer

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
E, d_model, d_ff = WORKLOADS["switch-base-128"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
lay = build_layer(E, d_model, d_ff, seed=0, dic=dic, device=dev, max_tokens=max(T, 64))
router = q.RouterSim(E, rule="argmax", seed=0)
x = q.bf16_round(np.random.default_rng(0).normal(size=(T, d_model)).astype(np.float32))
a = router.assign(x)
for _ in range(20):
    lay.forward(x, a)
N = 300
t0 = time.perf_counter()
for _ in range(N):
    lay.forward(x, a)
t1 = time.perf_counter()
print(f"forward(): {(t1 - t0) / N * 1e6:.1f} us per call")
st = next(iter(lay._stages.values()))
g = st["graphs"][False]
t0 = time.perf_counter()
for _ in range(N):
    g.replay()
    torch.cuda.current_stream().synchronize()
t1 = time.perf_counter()
print(f"graph replay + sync: {(t1 - t0) / N * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(N):
    np.copyto(st["xv"], x)
    np.copyto(st["av"], a)
t1 = time.perf_counter()
print(f"numpy -> pinned inputs: {(t1 - t0) / N * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(N):
    st["yv"].copy()
t1 = time.perf_counter()
print(f"pinned -> numpy output: {(t1 - t0) / N * 1e6:.1f} us")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph replay back to back (device): {e0.elapsed_time(e1) / N * 1e3:.1f} us")


def dev_time(fn, n=200):
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        fn()
    for _ in range(5):
        g2.replay()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(n):
        g2.replay()
    a1.record()
    torch.cuda.synchronize()
    return a0.elapsed_time(a1) / n * 1e3


print(f"H2D inputs copy alone: {dev_time(lambda: st['in_d'].copy_(st['in_h'], non_blocking=True)):.1f} us "
      f"({st['in_h'].numel()} B)")
_yd = torch.empty((T, d_model), device=dev)
print(f"D2H output copy alone: {dev_time(lambda: st['y_h'].copy_(_yd, non_blocking=True)):.1f} us")
xd = torch.from_numpy(x).to(dev)
ad = torch.from_numpy(a).to(dev)
yd = torch.empty((T, d_model), device=dev)
print(f"step alone (warm L2, one layer): {dev_time(lambda: lay.forward_device(xd, ad, out=yd)):.1f} us")

# zero-copy variants: the step reads / writes pinned host memory directly
xb = T * d_model * 4
in_h, y_h = st["in_h"], st["y_h"]
x_h = in_h[:xb].view(torch.float32).view(T, d_model)
a_h = in_h[xb:xb + T * 4].view(torch.int32)
ref = lay.forward(x, a)


def var_b():  # H2D copy, y written straight to host
    st["in_d"].copy_(in_h, non_blocking=True)
    lay.forward_device(st["in_d"][:xb].view(torch.float32).view(T, d_model),
                       st["in_d"][xb:xb + T * 4].view(torch.int32), out=y_h)


def var_c():  # no copies: x, ids read from host, y written to host
    lay.forward_device(x_h, a_h, out=y_h)


for name, fn in (("B: H2D copy + y to host", var_b), ("C: all zero-copy", var_c)):
    y_h.zero_()
    fn()
    torch.cuda.synchronize()
    ok = np.array_equal(y_h.numpy(), ref)
    gt = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gt):
        fn()
    for _ in range(5):
        gt.replay()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        gt.replay()
        torch.cuda.current_stream().synchronize()
    t1 = time.perf_counter()
    print(f"{name}: replay+sync {(t1 - t0) / N * 1e6:.1f} us, device {dev_time(fn):.1f} us, identical={ok}")
