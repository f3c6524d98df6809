"""Runs tools/ubench.cu on a large stacked matrix and prints codewords/s
(experiment harness; numbers go to DESIGN.md, not the bench line)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200 import _lib
from paper_2310_16795_b200.codebook import Codebook

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libubench.so"))
dic = q.generate_dictionary()
dev = torch.device("cuda", 0)
for rows, cols in ((3072 * 512, 768), (768 * 512, 3072)):
    w = torch.randn(rows, cols, device=dev) * 0.02
    codes, mm = q.rtn_quantize_device(w)
    dm = q.encode_device(codes, mm, dic)
    cb = Codebook(dic, [dm]); cb.apply([dm])
    x = torch.randn(cols, device=dev).to(torch.bfloat16)
    y = torch.zeros(rows, device=dev)
    for H in (16384, 40960):
        for mode in (2, 0):
            for grid in (148,):
                args = (mode, ctypes.c_void_p(cb.table.data_ptr() + 65540 * 4), H, ctypes.c_void_p(dm.cw.data_ptr()),
                        ctypes.c_void_p(dm.row_off.data_ptr()), ctypes.c_void_p(dm.row_minmax.data_ptr()), rows, cols,
                        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), grid, ctypes.c_void_p(0))
                lib.ubench_run(*args); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    lib.ubench_run(*args)
                e1.record(); torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                n = dm.n_codewords
                print(f"{rows}x{cols} H={H} mode={['naive','lookup','pipelined'][mode]} grid={grid}: {ms:.3f} ms "
                      f"{n / ms / 1e6:.1f} Gcw/s  {dm.compressed_bytes / ms / 1e6:.1f} GB/s", flush=True)
