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
    p.add_argument("--workload", default=None,
                   help="BASELINE config (default: switch-base-128 as a plain process; switch-c2048 expert-sharded "
                        "under torchrun, N >= 1, so the scaling series is one workload)")
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


# ----------------------------------------------------------------------------- shared workload
# BASELINE.json configs: name -> (experts, d_model, d_ff). Kept here (not
# imported from the package) so the reference arm never loads libqmoe.so.
WORKLOADS = {
    "switch-base-128": (128, 768, 3072),
    "switch-large-128": (128, 1024, 4096),
    "switch-c2048": (2048, 2080, 6144),
}
SEED_BASE = 0   # SURVEY 8(d) weight recipe: layer 0 of the pool, both arms
N_BATCHES = 8   # token batches; step i runs batch i % N_BATCHES


def seeded_weights(base, layer, e, m, rows, cols):
    """W_(layer, e, m) ~ N(0, 0.02^2) fp32 from
    default_rng(SeedSequence([base, layer, e, m])), m = 0 wi / 1 wo (the same
    recipe as paper_2310_16795_b200.synth.seeded_weights)."""
    rng = np.random.default_rng(np.random.SeedSequence([base, layer, e, m]))
    return (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)


def token_batches(T, d_model, E, seed):
    """bf16-valued N(0, 1) tokens and their RouterSim argmax experts (seed 0),
    via the oracle restatements (pinned to the reference's goldens)."""
    from oracle import qmoe_oracle as O

    rng = np.random.default_rng(seed)
    xs = [O.bf16_round(rng.normal(size=(T, d_model)).astype(np.float32)) for _ in range(N_BATCHES)]
    return xs, [O.router_argmax(x, E, seed=0) for x in xs]


# ----------------------------------------------------------------------------- reference arm
_REF_DIC = None


def _ref_init():
    global _REF_DIC
    from oracle import qmoe_oracle as O

    _REF_DIC = O.OracleDictionary(0.885, O.generate_decode_words(0.885))


def _ref_expert(job):
    """Oracle RTN + oracle encode of one expert (process-pool worker)."""
    from oracle import qmoe_oracle as O

    e, d_model, d_ff = job
    pair = []
    for m, (rows, cols) in enumerate(((d_ff, d_model), (d_model, d_ff))):
        w = seeded_weights(SEED_BASE, 0, e, m, rows, cols)
        mm = O.make_grid_bits(w)
        cw, ro = O.encode_codes(O.rtn_codes(w, mm), _REF_DIC)
        pair.append((rows, cols, cw, ro, mm))
    return e, tuple(pair)


def run_oracle_steps(x_list, assign_list, host, odic, workers):
    """Composed CPU oracle MoE step(s); returns (seconds, bytes, tokens, outputs)."""
    from oracle import qmoe_oracle as O

    t0 = time.perf_counter()
    nbytes = 0
    ntok = 0
    outs = []
    for x, a in zip(x_list, assign_list):
        y = None
        for e in np.unique(a):  # O.moe_layer's order: experts ascending, tokens in buffer order
            if e < 0:
                continue
            wi, wo = host[int(e)]
            nbytes += O.compressed_bytes(wi[0], len(wi[2])) + O.compressed_bytes(wo[0], len(wo[2]))
            if y is None:
                y = np.zeros((len(a), wo[0]), np.float32)
            for p in np.flatnonzero(a == e):
                h = O.fused_matvec(*wi[:2], *wi[2:], odic.hash64, x[p], odic, workers=workers)
                y[p] = O.fused_matvec(*wo[:2], *wo[2:], odic.hash64, np.maximum(h, 0.0), odic, workers=workers)
        outs.append(y)
        ntok += len(a)
    return time.perf_counter() - t0, nbytes, ntok, outs


def host_codewords(m) -> np.ndarray:
    """The matrix's stream in dictionary order (undoes the device-private
    frequency-codebook re-indexing) — what the reference codec would hold."""
    cw = m.cw.cpu().numpy().view(np.uint16)
    return m.codebook.order[cw] if m.codebook is not None else cw


def reference_arm(args):
    """The reference algorithm on the host cores: the composed CPU oracle
    (moepack.codec.fused_matvec restated, pinned to the reference's outputs)
    on the SAME workload as our arm — layer 0 of the pool (weights from the
    survey's seeded recipe, oracle RTN + encode), the same 8 token batches of
    T tokens, step i = batch i % 8. Imports nothing from the package."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp

    from oracle import qmoe_oracle as O

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    E, d_model, d_ff = WORKLOADS[args.workload]
    T = args.tokens
    cores = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    _ref_init()
    odic = _REF_DIC
    xs, asg = token_batches(T, d_model, E, seed=0)
    # bounded sample: at most ~25 G weight-MACs of oracle work in the timed
    # steps (Switch-base: all K steps; a c2048 layer: 1 step of T tokens)
    cap = max(1, int(25e9 / (T * d_model * d_ff * 2)))
    steps, warmup = min(args.steps, cap), min(args.warmup, max(0, cap - args.steps))
    nsteps = steps + warmup
    need = np.unique(np.concatenate([asg[i % N_BATCHES] for i in range(nsteps)]))
    t_build = time.time()
    with ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("fork"), initializer=_ref_init) as ex:
        host = dict(ex.map(_ref_expert, [(int(e), d_model, d_ff) for e in need]))
    t_build = time.time() - t_build
    order = [i % N_BATCHES for i in range(nsteps)]
    run_oracle_steps([xs[b] for b in order[:warmup]], [asg[b] for b in order[:warmup]], host, odic, cores)
    sec, nbytes, ntok, _ = run_oracle_steps([xs[b] for b in order[warmup:]], [asg[b] for b in order[warmup:]],
                                            host, odic, cores)
    gbs = nbytes / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": 1e3 * sec / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16 codewords -> f32 accumulate",
        "data": "synthetic: SURVEY 8(d) seeded N(0,0.02^2) weights (layer 0), oracle RTN + encode",
        "config": {"workload": args.workload, "experts": E, "d_model": d_model, "d_ff": d_ff,
                   "tokens_per_step": T, "routing": "top-1 RouterSim argmax seed 0",
                   "token_batches": N_BATCHES, "parallelism": "cpu"},
        "tokens_per_s": ntok / sec,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"{steps} steps x {T} tokens of layer 0 through the composed oracle "
                                   f"(moepack.codec.fused_matvec restated, workers={cores}); experts built in "
                                   f"{t_build:.0f} s"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


METRIC = "compressed decode+matvec HBM GB/s (% peak); MoE-layer tokens/s"


def _time_graphs(graphs, steps, warmup):
    """Mean ms per replay of a rotating list of CUDA graphs (CUDA events)."""
    import torch

    for i in range(max(warmup, 3)):
        graphs[i % len(graphs)].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        graphs[i % len(graphs)].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def _capture(fn):
    import torch

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def bf16_baseline(E, d_model, d_ff, xs_dev, asg, steps, warmup, dev):
    """Uncompressed bf16 reference of the same MoE step on the same GPU
    (north star: "uncompressed bf16 matvec of the same shape"): tokens sorted
    by expert, h = relu(X_e @ Wi_e^T), Y_e = h @ Wo_e^T as two GROUPED bf16
    GEMMs over all experts (torch._grouped_mm: one launch per pass, empty
    groups skipped, so only the touched experts' weights are read), tokens
    scattered back; the step is one CUDA graph. Random bf16 weights for all E
    experts (>= 4x L2, so HBM-cold). Falls back to one GEMM pair per touched
    expert if the grouped GEMM is unavailable (reported in `impl`)."""
    import torch

    g = torch.Generator(device=dev).manual_seed(7)
    Wi = torch.randn((E, d_ff, d_model), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    Wo = torch.randn((E, d_model, d_ff), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    nb = len(xs_dev)
    plans = []
    for b in range(nb):
        a = asg[b]
        order = np.argsort(a, kind="stable")
        offs = np.cumsum(np.bincount(a, minlength=E)).astype(np.int32)
        plans.append((torch.from_numpy(order).to(dev), torch.from_numpy(offs).to(dev),
                      [(int(e), torch.from_numpy(np.flatnonzero(a == e)).to(dev)) for e in np.unique(a)]))
    outs = [torch.empty((xs_dev[b].shape[0], d_model), device=dev, dtype=torch.bfloat16) for b in range(nb)]

    def grouped(b):
        order, offs, _ = plans[b]
        xs = xs_dev[b].index_select(0, order)
        h = torch.relu(torch._grouped_mm(xs, Wi.transpose(1, 2), offs=offs))
        outs[b].index_copy_(0, order, torch._grouped_mm(h, Wo.transpose(1, 2), offs=offs))

    def looped(b):
        x = xs_dev[b]
        for e, idx in plans[b][2]:
            xe = x.index_select(0, idx)
            h = torch.relu(xe @ Wi[e].t())
            outs[b].index_copy_(0, idx, h @ Wo[e].t())

    impl = "torch._grouped_mm (grouped bf16 GEMM, 2 launches + gather/scatter per step)"
    try:
        graphs = [_capture(lambda b=b: grouped(b)) for b in range(nb)]
        ref = torch.empty_like(outs[0])
        x = xs_dev[0]
        for e, idx in plans[0][2]:  # the grouped GEMM computes the same step
            ref.index_copy_(0, idx, torch.relu(x.index_select(0, idx) @ Wi[e].t()) @ Wo[e].t())
        graphs[0].replay()
        torch.cuda.synchronize()
        if not torch.allclose(ref.float(), outs[0].float(), rtol=2e-2, atol=2e-3):
            raise RuntimeError("grouped GEMM result differs")
    except Exception as exc:  # noqa: BLE001 - fall back, and say so
        impl = f"per-expert cuBLAS GEMM pairs (grouped GEMM unavailable: {type(exc).__name__})"
        graphs = [_capture(lambda b=b: looped(b)) for b in range(nb)]
    ms = _time_graphs(graphs, steps, warmup)
    del Wi, Wo, graphs
    torch.cuda.empty_cache()
    return ms, impl


def bf16_gemv(rows, cols, dev, hbm_peak, n=None, iters=5):
    """cuBLAS bf16 matvec y = W x of one rows x cols matrix (the paper's
    per-layer comparator): a CUDA graph of n calls over n
    distinct matrices (>= 4x L2: cold), us per call."""
    import torch

    n = n or max(8, int(4.5 * L2_BYTES / (2 * rows * cols)))
    W = torch.randn((n, rows, cols), device=dev, dtype=torch.bfloat16) * 0.02
    x = torch.randn(cols, device=dev).to(torch.bfloat16)
    y = torch.empty((n, rows), device=dev, dtype=torch.bfloat16)

    def body():
        for i in range(n):
            torch.mv(W[i], x, out=y[i])
    ms = _time_graphs([_capture(body)], iters, 2)
    us = ms * 1e3 / n
    del W
    torch.cuda.empty_cache()
    return {"shape": f"{rows}x{cols}", "us_per_call": us, "GBps": 2 * rows * cols / us / 1e3,
            "sol_us": 2 * rows * cols / (hbm_peak * 1e3)}


def bf16_expert_token(d_model, d_ff, dev, hbm_peak, iters=5):
    """Uncompressed bf16 expert FFN for ONE token (generation): wi gemv ->
    ReLU -> wo gemv with cuBLAS, over a cold pool of distinct experts (CUDA
    graph of one token per expert), us per token."""
    import torch

    per = 2 * 2 * d_model * d_ff
    n = max(8, int(4.5 * L2_BYTES / per))
    Wi = torch.randn((n, d_ff, d_model), device=dev, dtype=torch.bfloat16) * 0.02
    Wo = torch.randn((n, d_model, d_ff), device=dev, dtype=torch.bfloat16) * 0.02
    x = torch.randn(d_model, device=dev).to(torch.bfloat16)
    h = torch.empty((n, d_ff), device=dev, dtype=torch.bfloat16)
    y = torch.empty((n, d_model), device=dev, dtype=torch.bfloat16)

    def body():
        for i in range(n):
            torch.mv(Wi[i], x, out=h[i])
            torch.relu_(h[i])
            torch.mv(Wo[i], h[i], out=y[i])
    ms = _time_graphs([_capture(body)], iters, 2)
    us = ms * 1e3 / n
    del Wi, Wo
    torch.cuda.empty_cache()
    return us, per / (hbm_peak * 1e3)


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
        recs[i] = _lib.QmoeWork(d[0], d[1], d[2], d[3], cols, 0, rows, lg | (lg << 8), 1, t, d[8], (0, 0, 0, 0))
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
    # the instruction-issue roof: warp-instructions per codeword
    # of this launch from the committed ncu capture, at 4 issues / SM / cycle
    issue = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_summaries.json")) as fh:
            inst = json.load(fh)["pipe"][0]["inst_executed"]
        ipc = inst / ncw
        roof = 4 * 148 * 1.965e9 / ipc
        issue = {"warp_inst_per_codeword": ipc, "codewords_per_s": roof, "GBps": roof * nbytes / ncw / 1e9,
                 "source": "profiles/r02_ncu_summaries.json (pipe: smsp__inst_executed of this launch shape)"}
    except Exception:
        pass
    out = {"kernel": "pipe_matvec_kernel (one grouped launch)", "shape": f"{rows}x{cols}", "matrices": E,
           "issue_roof": issue,
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
    # the paper's Listing-1 kernel on the same cold matrices
    from paper_2310_16795_b200.codec import paper_matvec_device

    g2 = torch.cuda.CUDAGraph()
    for m in mats[:1]:
        paper_matvec_device(m, dic, x, y)
    torch.cuda.synchronize()
    with torch.cuda.graph(g2):
        for m in mats:
            paper_matvec_device(m, dic, x, y)
    listing1_us = _time_graphs([g2], 5, 2) * 1e3 / n
    del mats, g2
    torch.cuda.empty_cache()
    return {"api": "fused_matvec (drop-in, batch 1)", "shape": f"{rows}x{cols}", "device_us_per_call": dev_us,
            "paper_listing1_us_per_call": listing1_us,
            "device_GBps": nbytes / dev_us / 1e3, "host_us_per_call": host_us,
            "host_what": "numpy x in, numpy y out, matrix uploaded once (cached)"}


def decompress_at_scale(dic, dev, hbm_peak, rows=98304, cols=3072):
    """decompress (codec.py:175-193) throughput: ONE launch over a stacked
    compressed matrix (128 Switch-base wo experts' rows, 25 MB compressed,
    302 MB of u8 codes out). Algorithmic bytes = B + rows*cols."""
    import torch

    from paper_2310_16795_b200.codec import decompress_device, encode_device
    from paper_2310_16795_b200.quantize import rtn_quantize_device

    w = torch.randn((rows, cols), device=dev) * 0.02
    codes, mm = rtn_quantize_device(w)
    del w
    big = encode_device(codes, mm, dic)
    del codes
    out, _ = decompress_device(big, dic)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out, _ = decompress_device(big, dic)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    nbytes = big.compressed_bytes + rows * cols
    res = {"kernel": "decompress_kernel (one launch)", "rows": rows, "cols": cols, "ms": ms,
           "weights_per_s": rows * cols / ms * 1e3, "GBps": nbytes / ms / 1e6, "frac_of_hbm": nbytes / ms / 1e6 / hbm_peak,
           "bytes": "compressed B + rows*cols u8 codes written"}
    del big, out
    torch.cuda.empty_cache()
    return res


def profiled_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/roofline_r02.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_r02.json")) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    # under torchrun (any N, N = 1 included) the run is the expert-parallel
    # c2048 layer, so every point of a scaling series measures one workload;
    # a plain process measures the single-GPU headline (Switch-base-128)
    launched = "WORLD_SIZE" in os.environ
    if args.workload is None:
        args.workload = "switch-c2048" if launched else "switch-base-128"
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2310_16795_b200 as q
    from paper_2310_16795_b200.synth import build_layer, build_layer_seeded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.force_ep or (launched and args.workload == "switch-c2048"):
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
        if not layers:  # layer 0: the survey's seeded host recipe (what the reference arm regenerates)
            lay = build_layer_seeded(E, d_model, d_ff, base=SEED_BASE + rank, layer=0, dic=dic, device=dev,
                                     max_tokens=T)
        else:
            lay = build_layer(E, d_model, d_ff, seed=1000 * rank + len(layers), dic=dic, device=dev, max_tokens=T)
        layers.append(lay)
        pool += int(lay.expert_bytes.sum())
        if args.profile and len(layers) >= 2:
            break
    t_build = time.time() - t_build
    L = len(layers)

    # ---- token batches and routing (host RouterSim argmax, as the reference)
    router = q.RouterSim(E, rule="argmax", seed=0)
    rng = np.random.default_rng(rank)  # rank 0: the reference arm's batches (token_batches(seed=0))
    nb = N_BATCHES
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
    bf16_ms, bf16_impl = None, None
    if not args.profile:
        bf16_ms, bf16_impl = bf16_baseline(E, d_model, d_ff, xd, asg, args.steps, args.warmup, dev)
    bf16_bytes = float(np.mean([len(np.unique(a)) for a in asg])) * 2 * d_model * d_ff * 2
    bf16_sol_ms = bf16_bytes / (hbm_peak * 1e9) * 1e3

    # ---- e2e through the public host API (numpy in / numpy out)
    e2e = None
    if rank == 0 or world > 1:
        # warm-up: every pooled layer once (its per-T host graph is captured on
        # first use), then the W warm-up steps
        for i in range(L + args.warmup):
            layers[i % L].forward(xs[i % nb], asg[i % nb])
        items = lambda n: ((layers[i % L], xs[i % nb], asg[i % nb]) for i in range(n))  # noqa: E731
        for _ in q.forward_stream(items(2 * L + args.warmup)):  # both pipeline slots' graphs of every layer
            pass
        torch.cuda.synchronize()
        ne = max(args.steps, 200)  # host-timed: enough calls to average out host jitter
        e_bytes = sum(layers[i % L].touched_bytes(asg[i % nb]) for i in range(ne))
        # (a) the pipelined host API: step i + 1's inputs staged while step i runs
        t0 = time.perf_counter()
        n_out, y_last = 0, None
        for y_last in q.forward_stream(items(ne)):  # each step's rows consumed as they arrive
            n_out += 1
        torch.cuda.synchronize()
        e_sec = time.perf_counter() - t0
        # (b) one synchronous call per step
        t0 = time.perf_counter()
        for i in range(ne):
            l, b = i % L, i % nb
            layers[l].forward(xs[b], asg[b])
        torch.cuda.synchronize()
        s_sec = time.perf_counter() - t0
        assert n_out == ne and y_last.shape == (T, d_model)
        e2e = {"value": e_bytes / e_sec / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(xs[0].nbytes + asg[0].nbytes),
               "d2h_bytes_per_step": int(T * d_model * 4), "tokens_per_s": T * ne / e_sec, "steps": ne,
               "api": "paper_2310_16795_b200.forward_stream((layer, numpy x f32, numpy expert ids) per step) -> numpy y per step",
               "path": "per step: numpy x + ids into pinned memory, one H2D copy, fused step (one launch) writing y rows "
                       "into pinned host memory, event sync, copy out; two steps in flight (host staging overlaps the GPU)",
               "sync_api": {"value": e_bytes / s_sec / 1e9, "tokens_per_s": T * ne / s_sec,
                            "api": "CompressedMoELayer.forward(numpy x, numpy ids) -> numpy y, one blocking call per step"}}

    # ---- per-token (T = 1, generation) latency: the fused step vs the
    # uncompressed bf16 expert FFN (two cuBLAS gemv) — the north star's
    # "within 5% of an uncompressed bf16 matvec of the same shape"
    per_token = None
    if rank == 0 and world == 1 and not args.profile:
        outs1 = [torch.empty((1, d_model), dtype=torch.float32, device=dev) for _ in range(L)]
        C1 = 10
        chains1 = [_capture(lambda j=j: [layers[(j * C1 + u) % L].forward_device(
            xd[(j * C1 + u) % nb][:1], ad[(j * C1 + u) % nb][:1], out=outs1[(j * C1 + u) % L]) for u in range(C1)])
            for j in range(max(1, nsteps_graph // C1))]
        ours1_us = _time_graphs(chains1, 4 * len(chains1), 3) * 1e3 / C1
        del chains1
        bf16_1_us, sol1_us = bf16_expert_token(d_model, d_ff, dev, hbm_peak)
        # the c2048 shape (2080 / 6144): a 256-expert slice of a c2048-shaped
        # layer (542 MB compressed, > 4x L2), one token per step, distinct
        # experts step to step; vs the bf16 expert FFN of that shape
        Ec, dmc, dfc = WORKLOADS["switch-c2048"]
        lay_c = build_layer(256, dmc, dfc, seed=9, dic=dic, device=dev, max_tokens=1)
        xc = torch.from_numpy(q.bf16_round(np.random.default_rng(3).normal(size=(64, dmc)).astype(np.float32)))
        xc = xc.to(dev).to(torch.bfloat16)
        ac = [torch.tensor([e], dtype=torch.int32, device=dev) for e in range(0, 256, 4)]
        oc = torch.empty((1, dmc), device=dev)
        gc = [_capture(lambda j=j: [lay_c.forward_device(xc[(j * 10 + u) % 64:(j * 10 + u) % 64 + 1],
                                                         ac[(j * 10 + u) % len(ac)], out=oc) for u in range(10)])
              for j in range(6)]
        ours_c_us = _time_graphs(gc, 12, 3) * 1e3 / 10
        del gc, lay_c
        torch.cuda.empty_cache()
        bf16_c_us, sol_c_us = bf16_expert_token(dmc, dfc, dev, hbm_peak)
        per_token = {"tokens_per_step": 1, "ours_us_per_step": ours1_us, "bf16_cublas_us_per_token": bf16_1_us,
                     "bf16_hbm_sol_us": sol1_us, "ours_vs_bf16_cublas": bf16_1_us / ours1_us,
                     "c2048_shape": {"ours_us_per_step": ours_c_us, "bf16_cublas_us_per_token": bf16_c_us,
                                     "bf16_hbm_sol_us": sol_c_us, "ours_vs_bf16_cublas": bf16_c_us / ours_c_us},
                     "what": "one MoE layer step for one token (routed expert wi -> ReLU -> wo): the fused step "
                             "(graphs of 10 layer steps, cold pool) vs uncompressed bf16 cuBLAS gemv -> relu -> "
                             "gemv over a cold pool of experts"}

    # ---- the pool as a model (config 5's structure on this workload): L
    # residual blocks, each = device hash router + ONE fused launch computing
    # x + moe(x) in bf16, the whole forward one CUDA graph; vs L x the bf16
    # expert FFN per token measured above
    model_fwd = None
    if rank == 0 and world == 1 and not args.profile:
        routers = [q.DeviceRouter(q.RouterSim(E, rule="hash", seed=100 + l), d_model) for l in range(L)]
        model = q.CompressedMoEModel(layers, routers)
        model_fwd = {"layers": L, "routing": "RouterSim hash per layer, on the device (bit-exact)"}
        for Tm in (1, T):
            xm = xd[0][:Tm].contiguous()
            gm = _capture(lambda: model.forward_device(xm))
            ms_f = _time_graphs([gm], 10, 3)
            model_fwd[f"T{Tm}"] = {"forward_us": ms_f * 1e3, "us_per_layer": ms_f * 1e3 / L,
                                   "tokens_per_s": Tm / ms_f * 1e3}
            del gm
        if per_token:
            model_fwd["bf16_cublas_T1_forward_us"] = per_token["bf16_cublas_us_per_token"] * L


    # rank 0 at N=1 only: layer 0 (the survey's seeded weights) on batch 0,
    # all T tokens, through the composed CPU oracle on the device streams
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        from oracle import qmoe_oracle as O

        cores = os.cpu_count() or 1
        odic = O.OracleDictionary(0.885, dic.decode_words)
        lay = layers[0]
        host = {int(e): tuple((m.rows, m.cols, host_codewords(m), m.row_off.cpu().numpy(),
                               m.row_minmax.cpu().numpy().view(np.uint16).reshape(m.rows, 2))
                              for m in (lay.wi[int(e)], lay.wo[int(e)]))
                for e in np.unique(asg[0]) if e >= 0}
        y_gpu = lay.forward_device(xd[0], ad[0]).cpu().numpy()
        sec, nbytes, ntok, (y_ref,) = run_oracle_steps([xs[0]], [asg[0]], host, odic, cores)
        ulp = np.abs(y_gpu.view(np.int32).astype(np.int64) - y_ref.view(np.int32).astype(np.int64)) >> 16
        rel = float(np.max(np.linalg.norm(y_gpu - y_ref, axis=1) / np.maximum(np.linalg.norm(y_ref, axis=1), 1e-30)))
        # the GPU RTN + encoder against the oracle's, on one expert's seeded weights
        e0 = int(np.unique(asg[0])[0])
        w0 = seeded_weights(SEED_BASE, 0, e0, 1, d_model, d_ff)
        mm0 = O.make_grid_bits(w0)
        cw0, ro0 = O.encode_codes(O.rtn_codes(w0, mm0), odic)
        m0 = lay.wo[e0]
        enc_ok = (np.array_equal(host_codewords(m0), cw0) and np.array_equal(m0.row_off.cpu().numpy(), ro0)
                  and np.array_equal(m0.row_minmax.cpu().numpy().view(np.uint16).reshape(-1, 2), mm0))
        parity = {"max_ulp": int(ulp.max()), "identical": float(np.mean(ulp == 0)), "max_rel_l2": rel, "tokens": T,
                  "layer": 0, "encode_bit_exact": bool(enc_ok),
                  "tolerance": ">= 99% of outputs identical, per-token relative L2 <= 1e-2 (SURVEY 8(c) MoE bar; "
                               "a 1-ulp hidden difference can move a near-cancelling output by a few of its "
                               "ulps); encode bit-exact",
                  "against": "composed CPU oracle (moepack.codec.fused_matvec restated) on the same streams"}
        parity["ok"] = bool(parity["identical"] >= 0.99 and rel <= 1e-2 and enc_ok)
        cpu = {"value": nbytes / sec / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
               "tokens_per_s": ntok / sec,
               "sample": f"1 step x {T} tokens of layer 0 through the composed CPU oracle "
                         f"(numpy restatement of moepack.codec.fused_matvec, workers={cores})"}

    # ---- the decode + matvec kernel at scale (first half of the metric): one
    # grouped launch over a pool (> 4x L2) of distinct 768x3072 matrices
    # (Switch-base wo shape, 4 lanes per row), 1 token, cold
    at_scale = config1 = decomp = None
    if not args.profile:
        at_scale = matvec_at_scale(dic, dev, hbm_peak)
        decomp = decompress_at_scale(dic, dev, hbm_peak)
        config1 = single_matrix_api(dic, dev)
        config1["bf16_cublas_gemv"] = [bf16_gemv(768, 3072, dev, hbm_peak), bf16_gemv(3072, 768, dev, hbm_peak)]

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
                         "traffic_source": "profiles/roofline_r02.json (ncu --set full, dram__bytes_read+write per "
                                           "launch of the same kernel on the same workload)"},
            "bf16_baseline": {"ms_per_step_cublas": bf16_ms, "cublas_impl": bf16_impl,
                              "ms_per_step_hbm_sol": bf16_sol_ms,
                              "speedup_vs_bf16_cublas": (bf16_ms / (1e3 * t_sec / args.steps)) if bf16_ms else None,
                              "speedup_vs_bf16_sol": bf16_sol_ms / (1e3 * t_sec / args.steps),
                              "what": "same routed MoE step with uncompressed bf16 weights: measured (grouped "
                                      "bf16 GEMM over the touched experts in a CUDA graph), and its HBM "
                                      "speed-of-light (bf16 bytes of the touched experts / measured HBM peak)"},
            "per_token": per_token,
            "model_forward": model_fwd,
            "parity": parity,
            "kernel_at_scale": at_scale,
            "decompress_at_scale": decomp,
            "config1_single_matrix": config1,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": (1 if fused else 3) * args.steps,
            "clocks": dict(clocks or {}, window="sustained replay of the step graphs (0.5 s) into the timed region"),
            "build_s": t_build,
        }
        print(json.dumps(line), flush=True)
        if parity is not None and not parity["ok"]:
            sys.exit(f"parity check failed: {parity}")
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
    from paper_2310_16795_b200.synth import build_layer

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

    ep = ExpertParallelMoE(E, local_fn, max_tokens=T)

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
                         "kernel": "whole EP step per GPU (fused local step + NCCL exchange)",
                         "exchange_bytes_per_rank_step": {
                             "dispatch": world * T * (d_model * 2 + 4), "combine": world * T * d_model * 2,
                             "what": "fixed slots: T per destination rank, bf16 token rows + int32 expert ids "
                                     "out, bf16 output rows back (NVLink / NVSwitch)"}},
            "e2e": {"value": e2e_bytes / e2e_sec / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": int(xs[0].nbytes + asg[0].nbytes),
                    "d2h_bytes_per_step": int(T * d_model * 4), "tokens_per_s": T * world * args.steps / e2e_sec,
                    "api": "ExpertParallelMoE.forward(host tokens + ids copied in, outputs copied out)"},
            # per step: ep_slots_kernel, ep_rows_kernel, the fused local step, ep_combine_kernel
            "gpu_launches": 4 * args.steps, "cpu_baseline": None,
            "clocks": dict(cs.summary(), window="sustained EP steps (0.5 s) into the timed region"),
        }))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
