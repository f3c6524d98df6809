"""Drop-in fused_matvec on one matrix (batch 1, graph of 64 calls over cold
matrices): lanes per row / hot-table size variants of the API's grouped run."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2310_16795_b200 as q
import paper_2310_16795_b200.codec as C
from paper_2310_16795_b200.synth import _stacked
dic = q.generate_dictionary()
dev = torch.device("cuda", 0)
for rows, cols in ((768, 3072), (3072, 768)):
    mats = _stacked(64, rows, cols, seed=777, dic=dic, device=dev)
    x = torch.randn(cols, device=dev).to(torch.bfloat16)
    y = torch.zeros(rows, device=dev)
    for lanes, hot, ming in ((6144, 4096, 1.5), (6144, 1024, 1.5), (12288, 1024, 1.0), (12288, 4096, 1.0),
                             (24576, 1024, 0.5), (3072, 1024, 1.5)):
        C.API_LANES, C.API_HOT_ENTRIES = lanes, hot
        src = C._api_run.__code__
        for m in mats:
            m._api_runs = None
            mg = m.n_codewords / max(1, m.rows) / 8
            lg = 0
            while lg < 5 and m.rows * (1 << lg) < lanes and mg / (1 << (lg + 1)) >= ming:
                lg += 1
            if m.ck is None or m.lg < lg:
                m.build_checkpoints(dic, lg)
            tasks = ((m.rows << lg) + 31) >> 5
            rec = q._lib.QmoeWork(m.cw.data_ptr(), m.row_off.data_ptr(), m.row_minmax.data_ptr(),
                                  m.ck.data_ptr() if m.ck is not None else 0, m.cols, 0, m.rows, lg | (m.lg << 8), 1,
                                  0, 0, (0, 0, 0, 0))
            raw = torch.from_numpy(np.frombuffer(bytes(rec), dtype=np.uint8).copy()).to(dev)
            m._api_runs = (raw, torch.tensor([1, tasks], dtype=torch.int32, device=dev)) if lg else ()
        for m in mats:
            C.fused_matvec_device(m, dic, x, y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for m in mats:
                C.fused_matvec_device(m, dic, x, y)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        print(rows, cols, "lanes", lanes, "hot", hot, "min_groups", ming, "lg", lg,
              round(e0.elapsed_time(e1) / 320 * 1e3, 2), "us/call", flush=True)
