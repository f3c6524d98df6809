"""Floor of one CUDA-graph replay holding one tiny kernel (B200), to separate
launch overhead from the MoE step kernel's own time."""
import torch
x = torch.zeros(1024, device="cuda")
for n in (1, 2):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            x.add_(1)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(n):
            x.add_(1)
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph with {n} tiny kernel(s): {e0.elapsed_time(e1) / 200 * 1e3:.2f} us per replay")

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_16795_b200 import _lib
MODES = {0: "plain", 1: "cooperative", 2: "PDL", 3: "cooperative+PDL"}
for smem, thr, mode in ((0, 768, 0), (227 * 1024, 768, 0), (227 * 1024, 768, 1), (227 * 1024, 768, 2),
                        (227 * 1024, 768, 3), (0, 768, 1)):
    thr_arg = thr | (mode << 16)
    for n in (1, 8):
        sp = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.lib.qmoe_debug_empty_launch(smem, thr_arg, sp))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(n):
                _lib.check(_lib.lib.qmoe_debug_empty_launch(smem, thr_arg, torch.cuda.current_stream().cuda_stream))
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"empty kernel x{n} per graph, {MODES[mode]}, 148 CTAs x {thr} thr, {smem >> 10} KB smem: "
              f"{e0.elapsed_time(e1) / (100 * n) * 1e3:.2f} us per kernel")
