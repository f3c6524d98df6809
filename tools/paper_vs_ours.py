"""The paper's Listing-1 kernel on B200 (the baseline design)
vs this repo's streaming kernel, same matrices, same cold pool (> 4x L2).

paper  : qmoe_paper_matvec, one launch per matrix (warp per row, 32-codeword
         fetches, 28 extracting lanes, shuffle reduction), all launches of the
         pool in one CUDA graph; dictionary order (Listing 1 has no codebook)
ours   : qmoe_fused_matvec one launch per matrix (the drop-in API kernel,
         dictionary order), and qmoe_grouped_matvec ONE launch over the whole
         pool with frequency codebook + row checkpoints (the layer's setup)
Reports codewords/s, weights/s and compressed GB/s for each."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q  # noqa: E402
from paper_2310_16795_b200 import _lib  # noqa: E402
from paper_2310_16795_b200.codebook import Codebook  # noqa: E402
from paper_2310_16795_b200.synth import _stacked  # noqa: E402

import seg_bench as SB  # noqa: E402

dev = torch.device("cuda", 0)
dic = SB.dic
h = SB.h


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for rows, cols, lg in ((768, 3072, 2), (3072, 768, 0)):
    per = 2 * rows * cols // 24 + 8 * rows
    E = max(8, int(4.5 * SB.L2 / per))
    mats = _stacked(E, rows, cols, seed=rows + cols, dic=dic, device=dev)
    nbytes = sum(m.compressed_bytes for m in mats)
    ncw = sum(m.n_codewords for m in mats)
    x = torch.randn(cols, device=dev).to(torch.bfloat16)
    y = torch.zeros(rows, device=dev)
    s = _lib.stream_ptr()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for m in mats:
            _lib.check(_lib.lib.qmoe_paper_matvec(h, _lib.ptr(m.cw), _lib.ptr(m.row_off), _lib.ptr(m.row_minmax),
                                                  rows, cols, _lib.ptr(x), _lib.QMOE_X_BF16, _lib.ptr(y), None,
                                                  _lib.stream_ptr()))
    ms_p = timed(g.replay)
    # ours, the drop-in API's device path (fused_matvec_device), one launch per matrix like Listing 1
    for m in mats:  # first use builds the per-matrix run record / checkpoints
        q.codec.fused_matvec_device(m, dic, x, y)
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        for m in mats:
            q.codec.fused_matvec_device(m, dic, x, y)
    ms_s = timed(g2.replay)
    cb = Codebook(dic, mats)
    cb.apply(mats)
    for m in mats:
        m.build_checkpoints(dic, 3)
    x2 = x[None, :].repeat(2, 1).contiguous()
    y2 = torch.zeros(2, rows, device=dev)
    raw, n, _ = SB.runs_for(mats, 1, x2.stride(0), lg)

    def ours():
        _lib.check(_lib.lib.qmoe_grouped_matvec(h, _lib.ptr(cb.table), _lib.ptr(raw), _lib.ptr(n), len(mats), cols,
                                                 1, _lib.ptr(x2), _lib.QMOE_X_BF16, x2.stride(0), _lib.ptr(y2),
                                                 _lib.QMOE_Y_STORE_F32, y2.stride(0), 0, 0, _lib.stream_ptr()))
    ms_o = timed(ours)
    for name, ms in (("paper Listing 1", ms_p), ("ours per matrix", ms_s), ("ours (grouped)", ms_o)):
        print(f"{rows}x{cols} x{E} {name:16s}: {ms:.3f} ms  {ncw / ms / 1e6:6.1f} Gcw/s  "
              f"{E * rows * cols / ms / 1e9:5.2f} Tw/s  {nbytes / ms / 1e6:6.1f} GB/s", flush=True)
    print(f"{rows}x{cols}: paper / ours per matrix = {ms_p / ms_s:.2f}x, paper / ours grouped = {ms_p / ms_o:.2f}x",
          flush=True)
    del mats, cb
    torch.cuda.empty_cache()
