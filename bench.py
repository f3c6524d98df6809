"""Benchmark: compressed decode+matvec HBM GB/s and MoE-layer tokens/s.

Workload (BASELINE.json configs[1], the metric's single-GPU config):
Switch-base-128 MoE layer — 128 experts, d_model 768, d_ff 3072, top-1
routing (RouterSim argmax), T tokens per step (default 64), synthetic
random-init weights compressed by the bit-exact GPU encoder. A step is one MoE
layer forward: ONE cooperative launch (qmoe_moe_step: dispatcher plan in every
CTA's shared memory, wi pass with the ReLU fused, wo pass gated per expert run).
Cold L2: a pool of distinct layers >= 4x the 126 MB L2 is rotated, so every
step streams its experts from HBM.

value  = compressed bytes of the distinct experts touched per step (wi + wo,
         stats.compression_rate accounting) / device time, whole job (GB/s).
e2e    = the same through the public host API (numpy tokens + expert ids in,
         numpy outputs out; H2D/D2H inside the timed region).

`--impl reference` times the CPU oracle port of the reference algorithm
(oracle/, numpy restatement of moepack.codec.fused_matvec composed per token)
on the host cores instead.

Run: python bench.py [--gpus N --steps K --warmup W --tokens T --workload NAME]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="switch-base-128")
    p.add_argument("--tokens", type=int, default=64)
    p.add_argument("--pool-factor", type=float, default=4.0, help="layer pool size in multiples of L2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / cpu baseline)")
    p.add_argument("--force-ep", action="store_true", help="run the expert-parallel path even at 1 rank (testing)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:
                pass
            self.stop.wait(0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- reference arm
def oracle_layer_sample(E, d_model, d_ff, T, seed, odic, experts_needed):
    """Host-side synthetic experts for the CPU oracle: numpy N(0, 0.02^2) ->
    oracle RTN -> oracle encode (only the experts the sample touches)."""
    from oracle import qmoe_oracle as O

    host = {}
    for e in experts_needed:
        pair = []
        for m, (rows, cols) in enumerate(((d_ff, d_model), (d_model, d_ff))):
            rng = np.random.default_rng(np.random.SeedSequence([seed, 0, int(e), m]))
            w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
            mm = O.make_grid_bits(w)
            codes = O.rtn_codes(w, mm)
            cw, ro = O.encode_codes(codes, odic)
            pair.append((rows, cols, cw, ro, mm))
        host[int(e)] = tuple(pair)
    return host


def host_codewords(m) -> np.ndarray:
    """The matrix's stream in dictionary order (undoes the device-private
    frequency-codebook re-indexing) — what the reference codec would hold."""
    cw = m.cw.cpu().numpy().view(np.uint16)
    return m.codebook.order[cw] if m.codebook is not None else cw


def run_oracle_steps(x_list, assign_list, host, odic, workers):
    """Composed CPU oracle MoE step(s); returns (seconds, bytes, tokens)."""
    from oracle import qmoe_oracle as O

    t0 = time.perf_counter()
    nbytes = 0
    ntok = 0
    for x, a in zip(x_list, assign_list):
        for e in np.unique(a):
            wi, wo = host[int(e)]
            nbytes += O.compressed_bytes(wi[0], len(wi[2])) + O.compressed_bytes(wo[0], len(wo[2]))
            for p in np.flatnonzero(a == e):
                h = O.fused_matvec(*wi[:2], *wi[2:], odic.hash64, x[p], odic, workers=workers)
                O.fused_matvec(*wo[:2], *wo[2:], odic.hash64, np.maximum(h, 0), odic, workers=workers)
        ntok += len(a)
    return time.perf_counter() - t0, nbytes, ntok


def reference_arm(args):
    from oracle import qmoe_oracle as O
    from paper_2310_16795_b200.synth import WORKLOADS

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    E, d_model, d_ff = WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    odic = O.OracleDictionary(0.885, O.generate_decode_words(0.885))
    # bounded sample: each step = `sample_tokens` tokens of the workload
    sample_tokens = min(args.tokens, 8)
    rng = np.random.default_rng(0)
    xs, asg = [], []
    for s in range(args.steps + args.warmup):
        x = O.bf16_round(rng.normal(size=(sample_tokens, d_model)).astype(np.float32))
        xs.append(x)
        asg.append(O.router_argmax(x, E, seed=0))
    need = np.unique(np.concatenate(asg))
    host = oracle_layer_sample(E, d_model, d_ff, sample_tokens, 0, odic, need)
    run_oracle_steps(xs[: args.warmup], asg[: args.warmup], host, odic, cores)
    sec, nbytes, ntok = run_oracle_steps(xs[args.warmup :], asg[args.warmup :], host, odic, cores)
    gbs = nbytes / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16 codewords -> f32 accumulate",
        "data": "synthetic N(0,0.02^2) RTN ternary, oracle encode",
        "config": {"workload": args.workload, "experts": E, "d_model": d_model, "d_ff": d_ff,
                   "tokens_per_step": args.tokens, "sampled_tokens_per_step": sample_tokens,
                   "routing": "top-1 RouterSim argmax seed 0", "parallelism": "cpu"},
        "tokens_per_s": ntok / sec,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} steps x {sample_tokens} tokens through the composed oracle "
                                   f"(moepack.codec.fused_matvec restated, workers={cores})"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


METRIC = "compressed decode+matvec HBM GB/s (% peak); MoE-layer tokens/s"


def bf16_baseline(E, d_model, d_ff, xs_dev, asg, steps, warmup, dev):
    """Uncompressed bf16 reference of the same MoE step on the same GPU
    (north star: "uncompressed bf16 matvec of the same shape"): per touched
    expert h = relu(Wi_e @ X_e), Y_e = Wo_e @ h with cuBLAS bf16 GEMMs over
    the expert's tokens, the whole step captured in a CUDA graph. Random
    bf16 weights for all E experts (>= 4x L2, so HBM-cold)."""
    import torch

    g = torch.Generator(device=dev).manual_seed(7)
    Wi = torch.randn((E, d_ff, d_model), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    Wo = torch.randn((E, d_model, d_ff), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    nb = len(xs_dev)
    plans = []
    for b in range(nb):
        a = asg[b]
        plans.append([(int(e), torch.from_numpy(np.flatnonzero(a == e)).to(dev)) for e in np.unique(a)])
    outs = [torch.empty((xs_dev[b].shape[0], d_model), device=dev, dtype=torch.bfloat16) for b in range(nb)]

    def step(b):
        x = xs_dev[b]
        for e, idx in plans[b]:
            xe = x.index_select(0, idx)
            h = torch.relu(xe @ Wi[e].t())
            outs[b].index_copy_(0, idx, h @ Wo[e].t())

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for b in range(nb):
            step(b)
    torch.cuda.current_stream().wait_stream(s)
    graphs = []
    for b in range(nb):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step(b)
        graphs.append(gr)
    for i in range(warmup):
        graphs[i % nb].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        graphs[i % nb].replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del Wi, Wo, graphs
    torch.cuda.empty_cache()
    return ms


def matvec_at_scale(dic, dev, hbm_peak, rows=768, cols=3072, lg=2, iters=20):
    """Streaming decode + matvec throughput at scale: ONE grouped launch over
    E distinct compressed matrices (a pool > 4x L2, so weights come from HBM),
    one token; codewords/s, weights/s and compressed GB/s (stats bytes)."""
    import torch

    import paper_2310_16795_b200 as q
    from paper_2310_16795_b200 import _lib
    from paper_2310_16795_b200.codebook import Codebook
    from paper_2310_16795_b200.synth import _stacked

    per = 2 * rows * cols // 24 + 8 * rows
    E = int(4.5 * L2_BYTES / per)
    mats = _stacked(E, rows, cols, seed=4242, dic=dic, device=dev)
    cb = Codebook(dic, mats)
    cb.apply(mats)
    recs = (_lib.QmoeWork * E)()
    t = 0
    for i, m in enumerate(mats):
        m.build_checkpoints(dic, lg)
        d = m.descriptor()
        recs[i] = _lib.QmoeWork(d[0], d[1], d[2], d[3], cols, 0, rows, lg | (lg << 8), 1, t, 0, (0, 0, 0, 0))
        t += ((rows << lg) + 31) >> 5
    raw = torch.from_numpy(np.frombuffer(bytes(recs), dtype=np.uint8).copy()).to(dev)
    n = torch.tensor([E, t], dtype=torch.int32, device=dev)
    x = torch.randn(1, cols, device=dev).to(torch.bfloat16)
    y = torch.zeros(1, rows, device=dev)
    h = dic.device_handle(dev.index)

    def launch():
        _lib.check(_lib.lib.qmoe_grouped_matvec(h, _lib.ptr(cb.table), _lib.ptr(raw), _lib.ptr(n), E, cols, 1,
                                                 _lib.ptr(x), _lib.QMOE_X_BF16, x.stride(0), _lib.ptr(y),
                                                 _lib.QMOE_Y_STORE_F32, y.stride(0), 0, 0, _lib.stream_ptr()))
    launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    nbytes = sum(m.compressed_bytes for m in mats)
    ncw = sum(m.n_codewords for m in mats)
    out = {"kernel": "pipe_matvec_kernel (one grouped launch)", "shape": f"{rows}x{cols}", "matrices": E,
           "ms_per_launch": ms, "codewords_per_s": ncw / ms * 1e3, "weights_per_s": E * rows * cols / ms * 1e3,
           "GBps": nbytes / ms / 1e6, "frac_of_hbm": nbytes / ms / 1e6 / hbm_peak,
           "bf16_sol_weights_per_s": hbm_peak * 1e9 / 2}
    del mats, cb, raw
    torch.cuda.empty_cache()
    return out


def single_matrix_api(dic, dev, rows=768, cols=3072, n=64):
    """Config 1 through the drop-in API: fused_matvec(c, x, dic) on one
    768 x 3072 matrix (batch 1) — device path per call (uploaded matrix, CUDA
    graph of n calls over n distinct matrices: cold) and the host call with
    numpy x in / numpy y out."""
    import time

    import torch

    import paper_2310_16795_b200 as q
    from paper_2310_16795_b200.codec import fused_matvec_device
    from paper_2310_16795_b200.synth import _stacked

    mats = _stacked(n, rows, cols, seed=777, dic=dic, device=dev)  # uploaded, dictionary order
    x = torch.randn(cols, device=dev).to(torch.bfloat16)
    y = torch.zeros(rows, device=dev)
    for m in mats:
        fused_matvec_device(m, dic, x, y)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for m in mats:
            fused_matvec_device(m, dic, x, y)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) / (5 * n) * 1e3
    # host API: a CompressedMatrix (uploaded once, cached), numpy x -> numpy y
    w = (np.random.default_rng(5).normal(size=(rows, cols)) * 0.02).astype(np.float32)
    c = q.encode(q.rtn_quantize(w, q.make_grid(w)), dic)
    xh = q.bf16_round(np.random.default_rng(6).normal(size=cols).astype(np.float32))
    for _ in range(10):
        q.fused_matvec(c, xh, dic)
    t0 = time.perf_counter()
    for _ in range(200):
        q.fused_matvec(c, xh, dic)
    host_us = (time.perf_counter() - t0) / 200 * 1e6
    nbytes = float(np.mean([m.compressed_bytes for m in mats]))
    del mats
    torch.cuda.empty_cache()
    return {"api": "fused_matvec (drop-in, batch 1)", "shape": f"{rows}x{cols}", "device_us_per_call": dev_us,
            "device_GBps": nbytes / dev_us / 1e3, "host_us_per_call": host_us,
            "host_what": "numpy x in, numpy y out, matrix uploaded once (cached)"}


def profiled_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/roofline_r01.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_r01.json")) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2310_16795_b200 as q
    from paper_2310_16795_b200.synth import WORKLOADS, build_layer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.force_ep:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return ep_main(args, world, rank, local)
    dev = torch.device("cuda", local)
    E, d_model, d_ff = WORKLOADS[args.workload]
    T = args.tokens
    dic = q.generate_dictionary()

    # ---- layer pool (>= pool_factor x L2 of distinct compressed bytes)
    layers = []
    pool = 0
    t_build = time.time()
    while pool < args.pool_factor * L2_BYTES or not layers:
        lay = build_layer(E, d_model, d_ff, seed=1000 * rank + len(layers), dic=dic, device=dev, max_tokens=T)
        layers.append(lay)
        pool += int(lay.expert_bytes.sum())
        if args.profile and len(layers) >= 2:
            break
    t_build = time.time() - t_build
    L = len(layers)

    # ---- token batches and routing (host RouterSim argmax, as the reference)
    router = q.RouterSim(E, rule="argmax", seed=0)
    rng = np.random.default_rng(rank)
    nb = 8
    xs = [q.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32)) for _ in range(nb)]
    asg = [router.assign(x) for x in xs]
    xd = [torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in xs]
    ad = [torch.from_numpy(a).to(dev) for a in asg]
    outs = [torch.empty((T, d_model), dtype=torch.float32, device=dev) for _ in range(L)]

    # ---- CUDA graph per (layer, batch) step
    def step_fn(i):
        l, b = i % L, i % nb
        layers[l].forward_device(xd[b], ad[b], out=outs[l])

    nsteps_graph = L * nb // np.gcd(L, nb)
    graphs = []
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(min(nsteps_graph, 3)):
            step_fn(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for i in range(nsteps_graph):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step_fn(i)
        graphs.append(g)
    step_bytes = [layers[i % L].touched_bytes(asg[i % nb]) for i in range(nsteps_graph)]

    for i in range(args.warmup):
        graphs[i % nsteps_graph].replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # timed steps replay as graphs of C consecutive layer steps (a model
    # forward's launch pattern: the layers of a forward share one graph), C the
    # largest of 10 / 5 / 4 / 2 / 1 dividing K
    C = next(c for c in (10, 5, 4, 2, 1) if args.steps % c == 0)
    chains = []
    for j in range(args.steps // C):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for u in range(C):
                step_fn(args.warmup + j * C + u)
        chains.append(g)
    # ---- timed region (device): K graph replays. The clock sampler runs over a
    # sustained replay of the same graphs (~0.5 s) that leads straight into the
    # timed region (nvidia-smi needs tens of ms per sample; K steps take ~ms).
    hbm_peak, peak_kind = peaks()
    cs = ClockSampler(local) if not args.profile else None
    if cs:
        cs.__enter__()
        t_end = time.time() + 0.5
        i = 0
        while time.time() < t_end:
            for g in chains:
                g.replay()
            torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    tot_bytes = 0
    for g in chains:
        g.replay()
    for i in range(args.steps):
        tot_bytes += step_bytes[(args.warmup + i) % nsteps_graph]
    ev1.record()
    torch.cuda.synchronize()
    if cs:
        cs.__exit__()
    ms = ev0.elapsed_time(ev1)
    t_sec = ms / 1e3
    if world > 1:
        tt = torch.tensor([t_sec], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_sec = float(tt.item())
        bb = torch.tensor([tot_bytes], device=dev, dtype=torch.float64)
        dist.all_reduce(bb)
        tot_bytes = float(bb.item())
    value = tot_bytes / t_sec / 1e9
    tokens_per_s = T * args.steps * world / t_sec

    # ---- per-kernel timing. The fused step is ONE kernel launch per step, so
    # its average launch duration over the timed region is the region's time
    # / K (CUDA events on the launch stream; includes the ~1 us graph gap
    # between kernels, so it is conservative). For reference also the eager
    # back-to-back launches (events between launches enqueued ahead).
    stream = torch.cuda.current_stream()
    nk = min(max(args.steps, 8), 4 * nsteps_graph)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(nk + 1)]
    kb = []
    evs[0].record(stream)
    for i in range(nk):
        l, b = i % L, i % nb
        layers[l].forward_device(xd[b], ad[b], out=outs[l], stream=stream)
        evs[i + 1].record(stream)
        kb.append(layers[l].touched_bytes(asg[b]))
    torch.cuda.synchronize()
    eager_ms = float(np.mean([evs[i].elapsed_time(evs[i + 1]) for i in range(nk)]))
    fused = bool(layers[0].fused) and not layers[0].use_dense(T)
    if fused:
        kern_ms = 1e3 * t_sec / args.steps
        kern_bytes = tot_bytes / args.steps
    else:
        kern_ms, kern_bytes = eager_ms, float(np.mean(kb))
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9
    # ---- uncompressed bf16 reference of the same step on the same GPU
    bf16_ms = None
    if not args.profile:
        bf16_ms = bf16_baseline(E, d_model, d_ff, xd, asg, args.steps, args.warmup, dev)
    bf16_bytes = float(np.mean([len(np.unique(a)) for a in asg])) * 2 * d_model * d_ff * 2
    bf16_sol_ms = bf16_bytes / (hbm_peak * 1e9) * 1e3

    # ---- e2e through the public host API (numpy in / numpy out)
    e2e = None
    if rank == 0 or world > 1:
        # warm-up: every pooled layer once (its per-T host graph is captured on
        # first use), then the W warm-up steps
        for i in range(L + args.warmup):
            layers[i % L].forward(xs[i % nb], asg[i % nb])
        torch.cuda.synchronize()
        ne = max(args.steps, 200)  # host-timed: enough calls to average out host jitter
        e_bytes = sum(layers[i % L].touched_bytes(asg[i % nb]) for i in range(ne))
        t0 = time.perf_counter()
        for i in range(ne):
            l, b = i % L, i % nb
            layers[l].forward(xs[b], asg[b])
        torch.cuda.synchronize()
        e_sec = time.perf_counter() - t0
        e2e = {"value": e_bytes / e_sec / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(xs[0].nbytes + asg[0].nbytes),
               "d2h_bytes_per_step": int(T * d_model * 4), "tokens_per_s": T * ne / e_sec, "steps": ne,
               "api": "CompressedMoELayer.forward(numpy x f32, numpy expert ids) -> numpy y",
               "path": "one pinned H2D copy of x + ids, fused step (one launch) writing y rows into pinned host memory, stream sync, copy out"}

    # ---- CPU baseline (oracle port on this host), rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        from oracle import qmoe_oracle as O

        cores = os.cpu_count() or 1
        odic = O.OracleDictionary(0.885, dic.decode_words)
        sample_steps, sample_T = 2, min(T, 16)
        host = {}
        for b in range(sample_steps):
            for e in np.unique(asg[b][:sample_T]):
                if int(e) in host:
                    continue
                lay = layers[0]
                host[int(e)] = tuple(
                    (m.rows, m.cols, host_codewords(m), m.row_off.cpu().numpy(),
                     m.row_minmax.cpu().numpy().view(np.uint16).reshape(m.rows, 2))
                    for m in (lay.wi[int(e)], lay.wo[int(e)]))
        sec, nbytes, ntok = run_oracle_steps([xs[b][:sample_T] for b in range(sample_steps)],
                                             [asg[b][:sample_T] for b in range(sample_steps)], host, odic, cores)
        cpu = {"value": nbytes / sec / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
               "tokens_per_s": ntok / sec,
               "sample": f"{sample_steps} steps x {sample_T} tokens of layer 0 through the composed CPU oracle "
                         f"(numpy restatement of moepack.codec.fused_matvec, workers={cores})"}

    # ---- the decode + matvec kernel at scale (first half of the metric): one
    # grouped launch over a pool (> 4x L2) of distinct 768x3072 matrices
    # (Switch-base wo shape, 4 lanes per row), 1 token, cold
    at_scale = config1 = None
    if not args.profile:
        at_scale = matvec_at_scale(dic, dev, hbm_peak)
        config1 = single_matrix_api(dic, dev)

    traffic, _ = profiled_traffic()
    if rank == 0:
        clocks = cs.summary() if cs else None
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_sec / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16 codewords -> f32 accumulate (bf16 x, bf16-rounded y)",
            "data": "synthetic: random-init N(0,0.02^2) weights, GPU RTN ternary + bit-exact GPU encoder",
            "config": {"workload": args.workload, "experts": E, "d_model": d_model, "d_ff": d_ff,
                       "tokens_per_step": T, "routing": "top-1 RouterSim argmax seed 0", "layer_pool": L,
                       "graph_steps": C,
                       "pool_bytes": pool, "l2": f"cold: rotating {L} distinct layers = {pool / L2_BYTES:.1f}x L2",
                       "parallelism": f"ep{world}" if world > 1 else "single"},
            "pct_peak": 100 * value / hbm_peak,
            "tokens_per_s": tokens_per_s,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": ("moe_step_kernel (the whole step: plan + wi + wo in one cooperative launch)"
                                    if fused else "grouped passes"),
                         "bytes_per_launch": kern_bytes, "ms_per_launch": kern_ms,
                         "ms_per_launch_source": ("timed region / K (one fused kernel per step)" if fused
                                                  else "eager back-to-back launches"),
                         "eager_ms_per_launch": eager_ms,
                         "traffic_source": "profiles/roofline_r01.json (ncu --set full, dram__bytes_read+write per "
                                           "launch of the same kernel on the same workload)"},
            "bf16_baseline": {"ms_per_step_cublas": bf16_ms,
                              "ms_per_step_hbm_sol": bf16_sol_ms,
                              "speedup_vs_bf16_cublas": (bf16_ms / (1e3 * t_sec / args.steps)) if bf16_ms else None,
                              "speedup_vs_bf16_sol": bf16_sol_ms / (1e3 * t_sec / args.steps),
                              "what": "same routed MoE step with uncompressed bf16 weights: measured with cuBLAS "
                                      "GEMMs per touched expert in a CUDA graph, and its HBM speed-of-light "
                                      "(bf16 bytes of the touched experts / measured HBM peak)"},
            "kernel_at_scale": at_scale,
            "config1_single_matrix": config1,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": (1 if fused else 3) * args.steps,
            "clocks": dict(clocks or {}, window="sustained replay of the step graphs (0.5 s) into the timed region"),
            "build_s": t_build,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def ep_main(args, world, rank, local):
    """--gpus N > 1: expert-parallel layer, experts sharded in contiguous
    blocks over the ranks, NCCL all-to-all dispatch/combine (weak scaling:
    every rank brings T tokens). value = compressed bytes all ranks streamed /
    max-over-ranks device time."""
    import time

    import torch
    import torch.distributed as dist

    import paper_2310_16795_b200 as q
    from paper_2310_16795_b200.ep import ExpertParallelMoE
    from paper_2310_16795_b200.synth import WORKLOADS, build_layer

    dev = torch.device("cuda", local)
    E, d_model, d_ff = WORKLOADS[args.workload]
    E_loc = E // world
    T = args.tokens
    dic = q.generate_dictionary()
    layers, pool = [], 0
    while pool < args.pool_factor * L2_BYTES or not layers:
        lay = build_layer(E_loc, d_model, d_ff, seed=1000 * rank + len(layers), dic=dic, device=dev,
                          max_tokens=T * world)
        layers.append(lay)
        pool += int(lay.expert_bytes.sum())
        if len(layers) >= 96:  # each rank holds E / N experts per layer: more layers for a cold L2
            break
    L = len(layers)
    router = q.RouterSim(E, rule="argmax", seed=0)
    nb = 4
    # every rank's tokens are a pure function of (rank, batch): each rank can
    # count, on the host, the experts of its block that step i touches
    all_x = [[q.bf16_round(np.random.default_rng(1000 * r + b).normal(size=(T, d_model)).astype(np.float32))
              for b in range(nb)] for r in range(world)]
    all_a = [[router.assign(x) for x in xr] for xr in all_x]
    xs, asg = all_x[rank], all_a[rank]
    xd = [torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in xs]
    ad = [torch.from_numpy(a).to(dev) for a in asg]

    def step_bytes(i):
        ids = np.concatenate([all_a[r][i % nb] for r in range(world)])
        mine = ids[(ids >= rank * E_loc) & (ids < (rank + 1) * E_loc)] - rank * E_loc
        return layers[i % L].touched_bytes(mine) if mine.size else 0

    cur = {"l": 0}

    def local_fn(x_recv, local_ids):
        if local_ids.numel() == 0:
            return torch.zeros((0, d_model), device=dev)
        return layers[cur["l"]].forward_device(x_recv, local_ids)

    ep = ExpertParallelMoE(E, local_fn)

    def step(i):
        cur["l"] = i % L
        return ep.forward(xd[i % nb], ad[i % nb])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    dist.barrier()
    # the EP step is device-only (fixed-slot exchange): capture each (layer,
    # batch) step — fused local step + NCCL all-to-alls — in a CUDA graph;
    # eager if the capture is refused
    nsg = L * nb // int(np.gcd(L, nb))
    graphs, graph_note = [], "cuda graph per step (NCCL all-to-alls captured)"
    try:
        for i in range(nsg):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(i)
            graphs.append(g)
        torch.cuda.synchronize()
        dist.barrier()
    except Exception as exc:  # noqa: BLE001 - report and run eager
        graphs, graph_note = [], f"eager (capture refused: {type(exc).__name__})"
        torch.cuda.synchronize()
        dist.barrier()
    ok = torch.tensor([1 if graphs else 0], device=dev, dtype=torch.int32)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank replays graphs, or none does
    if not int(ok.item()) and graphs:
        graphs, graph_note = [], "eager (another rank could not capture)"

    def run(i):
        if graphs:
            cur["l"] = i % L
            graphs[i % nsg].replay()
        else:
            step(i)

    for i in range(args.warmup):
        run(i)
    torch.cuda.synchronize()
    dist.barrier()
    my_bytes = float(sum(step_bytes(args.warmup + i) for i in range(args.steps)))
    cs = ClockSampler(local)
    cs.__enter__()
    t_end = time.time() + 0.5
    while time.time() < t_end:  # sustained steps into the timed region (clock sampling window)
        for i in range(8):
            run(i)
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        run(args.warmup + i)
    e1.record()
    torch.cuda.synchronize()
    cs.__exit__()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    b = torch.tensor([my_bytes], device=dev, dtype=torch.float64)
    dist.all_reduce(b)
    t_sec, tot = float(t.item()), float(b.item())
    # e2e: host tokens + ids in, host outputs back, through the EP layer
    xh = [torch.from_numpy(x).pin_memory() for x in xs]
    ah = [torch.from_numpy(a).pin_memory() for a in asg]
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        cur["l"] = i % L
        y = ep.forward(xh[i % nb].to(dev, non_blocking=True), ah[i % nb].to(dev, non_blocking=True))
        y.cpu()
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_sec = float(te.item())
    eb = torch.tensor([float(sum(step_bytes(i) for i in range(args.steps)))], device=dev, dtype=torch.float64)
    dist.all_reduce(eb)
    e2e_bytes = float(eb.item())
    hbm_peak, peak_kind = peaks()
    if rank == 0:
        per_gpu = tot / world / t_sec / 1e9
        print(json.dumps({
            "metric": METRIC, "value": tot / t_sec / 1e9, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_sec / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16 codewords -> f32 accumulate (bf16 x)",
            "data": "synthetic random-init weights, GPU RTN + bit-exact GPU encoder",
            "config": {"workload": args.workload, "experts": E, "experts_per_rank": E_loc, "d_model": d_model,
                       "d_ff": d_ff, "tokens_per_step_per_rank": T, "parallelism": f"ep{world}",
                       "exchange": "NCCL all_to_all_single dispatch + combine (fixed slots, no host sync)",
                       "launch": graph_note, "layer_pool_per_rank": L,
                       "l2": "cold: rotating layers, pool >= 4x L2 per rank"},
            "tokens_per_s": T * world * args.steps / t_sec, "pct_peak": 100 * per_gpu / hbm_peak,
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": hbm_peak, "unit": "GB/s",
                         "frac": per_gpu / hbm_peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "whole EP step per GPU (fused local step + NCCL exchange)"},
            "e2e": {"value": e2e_bytes / e2e_sec / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": int(xs[0].nbytes + asg[0].nbytes),
                    "d2h_bytes_per_step": int(T * d_model * 4), "tokens_per_s": T * world * args.steps / e2e_sec,
                    "api": "ExpertParallelMoE.forward(host tokens + ids copied in, outputs copied out)"},
            "gpu_launches": args.steps, "cpu_baseline": None,
            "clocks": dict(cs.summary(), window="sustained EP steps (0.5 s) into the timed region"),
        }))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
