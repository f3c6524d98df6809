"""Phase timeline of the fused MoE step (debug hook qmoe_debug_step_trace):
per-CTA %globaltimer stamps -> when the plan, wi and wo phases end."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16795_b200 as q
from paper_2310_16795_b200 import _lib
from paper_2310_16795_b200.synth import WORKLOADS, build_layer  # noqa: F401

dev = torch.device("cuda", 0)
dic = q.generate_dictionary()
wl = os.environ.get("WORKLOAD", "switch-base-128")
E, d_model, d_ff = WORKLOADS[wl]
layers = [build_layer(E, d_model, d_ff, seed=s, dic=dic, device=dev, max_tokens=256) for s in range(4)]
router = q.RouterSim(E, rule="argmax", seed=0)
rng = np.random.default_rng(0)
buf = torch.zeros(148 * 8, dtype=torch.int64, device=dev)
MHZ = float(os.environ.get("SM_MHZ", 1965))  # SM clock under load (bench clocks line)
for T in [int(t) for t in sys.argv[1:]] or [1, 8, 64]:
    x = q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32))
    a = router.assign(x)
    xd = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    ad = torch.from_numpy(a).to(dev)
    import time
    t_end = time.time() + 0.5  # sustained steps first: SM clocks ramp to their boost level
    while time.time() < t_end:
        for i in range(20):
            layers[i % 4].forward_device(xd, ad)
        torch.cuda.synchronize()
    _lib.check(_lib.lib.qmoe_debug_step_trace(_lib.ptr(buf)))
    buf.zero_()
    layers[3].forward_device(xd, ad)
    torch.cuda.synchronize()
    _lib.check(_lib.lib.qmoe_debug_step_trace(None))
    full = buf.view(148, 8).cpu().numpy().astype(np.int64)
    # [0] globaltimer ns at CTA start, [1..7] SM cycles since then
    r = np.zeros((148, 4))
    r[:, 0] = (full[:, 0] - full[:, 0].min()) / 1e3
    cyc = full[:, 1:] / MHZ  # cycles / MHz = us
    r[:, 1:] = r[:, :1] + cyc[:, :3]
    sub = cyc[:, 3:]
    print("   plan counted / runs built / plan end (us since CTA start, median):",
          np.median(sub[:, 0]).round(2), np.median(sub[:, 3]).round(2), np.median(cyc[:, 0]).round(2))
    print("   wi first window staged (us since CTA start, median/max):", np.median(sub[:, 1]).round(2), sub[:, 1].max().round(2))
    wait = r[:, :1] + sub[:, 2:3]
    slow = np.argsort(-r[:, 3])[:6]
    print("   slowest CTAs (wi end, last wo wait done, wo end):",
          [(int(c), round(r[c, 2], 1), round(float(wait[c, 0]), 1), round(r[c, 3], 1)) for c in slow])
    print("   wo wait done percentiles 10/50/90/max:", np.percentile(wait[:, 0], [10, 50, 90, 100]).round(1))
    wi_d = r[:, 2] - r[:, 1]
    wo_d = r[:, 3] - r[:, 2]
    print("   wi phase us percentiles 10/50/90/max:", np.percentile(wi_d, [10, 50, 90, 100]).round(1),
          " wo phase:", np.percentile(wo_d, [10, 50, 90, 100]).round(1),
          " slowest-wo CTAs:", np.argsort(-r[:, 3])[:6])
    print(f"T={T}: start {np.median(r[:,0]):.1f}/{r[:,0].max():.1f}  plan {np.median(r[:,1]):.1f}/{r[:,1].max():.1f}  "
          f"wi {np.median(r[:,2]):.1f}/{r[:,2].max():.1f}  wo {np.median(r[:,3]):.1f}/{r[:,3].max():.1f} us (median/max over CTAs)")


def host_split(assign, E, ntu, tasks, grid=148):
    """Host restatement of the fused step's weighted run split (one phase):
    per CTA (first task, last task + 1, runs touched)."""
    runs = []
    for e in range(E):
        toks = np.flatnonzero(assign == e)
        for c in range(0, len(toks), ntu):
            runs.append(min(ntu, len(toks) - c))
    w = np.array([11 if n > 1 else 8 for n in runs], dtype=np.int64)
    wpre = np.concatenate([[0], np.cumsum(w)])
    nch = len(runs)
    out = []
    for b in range(grid):
        se = []
        for side in (0, 1):
            target = wpre[nch] * tasks * (b + side) // grid
            lo = int(np.searchsorted(wpre * tasks, target, side="right") - 1)
            if lo >= nch:
                t = nch * tasks
            else:
                t = lo * tasks + int(min(tasks, (target - wpre[lo] * tasks) // max(1, w[lo])))
            if side and b == grid - 1:
                t = nch * tasks
            se.append(t)
        out.append((se[0], se[1], sorted({t // tasks for t in range(se[0], se[1])})))
    return runs, out
