"""Kernel-level throughput of the streaming matvec (experiment harness; the
numbers go to DESIGN.md / profiles, not the bench line).

For each shape, E expert matrices are built on the GPU (RTN of N(0, 0.02^2),
bit-exact GPU encoder), re-indexed by one frequency codebook, given row
checkpoints, and run as ONE grouped launch (one run per matrix, 1 or 2
tokens). The pool is > 4x L2, so every launch streams from HBM. Reports
codewords/s, weights/s and compressed GB/s (stats.compression_rate bytes).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q  # noqa: E402
from paper_2310_16795_b200 import _lib  # noqa: E402
from paper_2310_16795_b200.codebook import Codebook  # noqa: E402
from paper_2310_16795_b200.synth import _stacked  # noqa: E402

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
h = dic.device_handle(0)
L2 = 126 << 20


def runs_for(mats, ntok, ldx, lg=None):
    recs = (_lib.QmoeWork * len(mats))()
    t = 0
    for i, m in enumerate(mats):
        d = m.descriptor()
        mlg = d[7] if lg is None else (lg | (d[7] << 8))
        recs[i] = _lib.QmoeWork(d[0], d[1], d[2], d[3], m.cols, 0, m.rows, mlg, ntok, t, d[8],
                                tuple([0, 1 % max(1, ntok), 0, 0][:4]))
        t += ((m.rows << (mlg & 0xFF)) + 31) >> 5
    raw = torch.from_numpy(np.frombuffer(bytes(recs), dtype=np.uint8).copy()).to(dev)
    n = torch.tensor([len(mats), t], dtype=torch.int32, device=dev)
    return raw, n, t


def bench(rows, cols, lg=None, ntok=1, iters=20):
    per = 2 * rows * cols // 24 + 8 * rows
    E = max(8, int(4.5 * L2 / per))
    mats = _stacked(E, rows, cols, seed=rows + cols, dic=dic, device=dev)
    cb = Codebook(dic, mats)
    cb.apply(mats)
    for m in mats:
        m.build_checkpoints(dic, 3)
    nbytes = sum(m.compressed_bytes for m in mats)
    ncw = sum(m.n_codewords for m in mats)
    x = torch.randn(2, cols, device=dev).to(torch.bfloat16)
    y = torch.zeros(2, rows, device=dev)
    raw, n, tasks = runs_for(mats, ntok, x.stride(0), lg)
    flag = 0
    # all matrices in one launch is one "step"; y rows are overwritten per matrix (timing only)
    def launch():
        _lib.check(_lib.lib.qmoe_grouped_matvec(h, _lib.ptr(cb.table), _lib.ptr(raw), _lib.ptr(n), len(mats), cols,
                                                 ntok, _lib.ptr(x), _lib.QMOE_X_BF16, x.stride(0), _lib.ptr(y),
                                                 _lib.QMOE_Y_STORE_F32 | flag, y.stride(0), 0, 0, _lib.stream_ptr()))
    launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    lgv = lg
    print(f"raw {rows}x{cols} E={E} lg={lgv} ntok={ntok} tasks={tasks}: {ms:.3f} ms  {ncw / ms / 1e6:.1f} Gcw/s  "
          f"{E * rows * cols / ms / 1e9:.2f} Tw/s  {nbytes / ms / 1e6:.1f} GB/s (hit@H {cb.hit_rate(45000):.3f})",
          flush=True)
    del mats, cb
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for rows, cols, lg in ((3072, 768, 0), (768, 3072, 2), (6144, 2080, 1), (2080, 6144, 2)):
        for ntok in (1, 2):
            bench(rows, cols, lg=lg, ntok=ntok)
    for lg in (0, 1, 2, 3):
        bench(3072, 768, lg=lg)
        bench(768, 3072, lg=lg)
