"""Compressed MoE layer: routed-expert dispatcher + grouped decode/matvec.

One step for T tokens with top-1 expert ids:
  1. qmoe_moe_plan      stable counting sort of the assignment (buffer order
                        within an expert, pipeline.py:86-90) and the run
                        lists of both FFN passes (one run per expert token
                        chunk), written on the device;
  2. grouped wi pass    h[t] = relu(bf16(wi_e @ x[t])) written as bf16 (the
                        ReLU and the bf16 store fused into the epilogue) for
                        every token, one persistent launch over all experts;
  3. grouped wo pass    y[t] = bf16(wo_e @ h[t]) accumulated into fp32 y.
Each touched expert's compressed matrices are streamed from HBM once per
step: the tokens routed to one expert share a work unit (inner token loop,
2 per run on the streaming path), so decode is not repeated per token.
No host synchronisation: the whole step is CUDA-graph capturable.

Numerics equal the composed reference oracle (per token wi matvec -> ReLU ->
wo matvec through moepack.codec.fused_matvec) up to the matvec tolerance.
"""

from __future__ import annotations

import contextlib
import ctypes
import threading

import numpy as np

from . import _lib
from .codec import DeviceMatrix
from .dictionary import Dictionary
from .errors import CorruptionError as CorruptionError_


class CompressedMoELayer:
    """E experts, expert e = (wi_e: d_ff x d_model, wo_e: d_model x d_ff),
    all DeviceMatrix on one device."""

    def __init__(self, wi: list[DeviceMatrix], wo: list[DeviceMatrix], dic: Dictionary, max_tokens: int = 64,
                 tokens_per_unit: int = 2, codebook: bool = True, fused: bool = True, dense: str = "auto"):
        """dense: "auto" (decode-then-MMA from DENSE_MIN_TOKENS tokens per
        touched expert), "never" or "always"; fused: one cooperative launch
        per streaming step (else plan kernel + two grouped passes)."""
        import torch

        if len(wi) != len(wo) or not wi:
            raise ValueError("need matching wi/wo lists")
        if dense not in ("auto", "never", "always"):
            raise ValueError("dense must be 'auto', 'never' or 'always'")
        self.E = len(wi)
        self.d_ff, self.d_model = wi[0].rows, wi[0].cols
        for a, b in zip(wi, wo):
            if (a.rows, a.cols) != (self.d_ff, self.d_model) or (b.rows, b.cols) != (self.d_model, self.d_ff):
                raise ValueError("expert shapes disagree")
            if a.bad_rows or b.bad_rows:
                raise ValueError("expert matrix failed row validation")
        self.device = wi[0].cw.device
        self.handle = dic.device_handle(self.device.index)
        sparse = bool(dic.device_info(self.device.index)["sparse_path"])
        self._sparse_path = sparse
        # layer-level frequency codebook (kernel-private stream re-indexing).
        # Matrices cached on a host CompressedMatrix (c.to_device) are shared
        # with the drop-in API, which reads them in dictionary order: the layer
        # re-indexes private copies of their streams instead.
        self.codebook = None
        if codebook and sparse:
            from .codebook import Codebook

            mats = list(wi) + list(wo)
            if all(m.codebook is None for m in mats):
                wi = [m.private_copy() if m.shared else m for m in wi]
                wo = [m.private_copy() if m.shared else m for m in wo]
                mats = list(wi) + list(wo)
                self.codebook = Codebook(dic, mats)
                self.codebook.apply(mats)
            elif len({id(m.codebook) for m in mats}) == 1:
                self.codebook = mats[0].codebook
        self.wi, self.wo, self.dic = wi, wo, dic
        # mean 8-codeword groups per row (wi, wo): lane-segment sizing
        self.mean_groups = tuple(float(np.mean([m.n_codewords / max(1, m.rows) / 8 for m in ms])) for ms in (wi, wo))
        # most lanes per row a step may use: segments of >= ~2 groups, one
        # level finer than that (tiny generation steps split rows further)
        self.max_lg = tuple(max(0, min(self.MAX_LG, int(np.floor(np.log2(max(1.0, mg / 2)))) + 1))
                            for mg in self.mean_groups)
        for kind, ms in enumerate((wi, wo)):  # kernel-private row checkpoints
            for m in ms:
                if m.ck is None and m.lg == 0 and self.max_lg[kind] > 0:
                    # checkpoints for 2^max_lg lanes per row; a run may use any 2^lg <= that
                    m.build_checkpoints(dic, lg=self.max_lg[kind])
        self.mats = None
        self._write_descriptors()
        self.tokens_per_unit = min(int(tokens_per_unit), _lib.NT_STREAM)
        self.expert_bytes = np.array([wi[e].compressed_bytes + wo[e].compressed_bytes for e in range(self.E)],
                                     np.int64)
        self._lanes = {}
        self._T = max_tokens
        self._retired = []
        self._stages = {}
        self.dense_mode = dense
        # the fused step publishes its dispatcher plan (self.order /
        # self.expert_count, as qmoe_moe_plan) only on request: it costs the
        # step's tail
        self.publish_plan = False
        # one cooperative launch per step (sparse dictionaries)
        self.fused = sparse and fused
        self._alloc(max_tokens)

    def _alloc(self, T: int) -> None:
        """(Re)allocate the per-step device buffers for up to T tokens. CUDA
        graphs captured earlier (the host API's per-T graphs, or a caller's)
        hold raw pointers to the previous buffers, so those are retired — kept
        alive with the layer — instead of freed: a replay of an old graph
        stays consistent with the buffers it was captured on."""
        import torch

        if hasattr(self, "h"):
            self._retired.append((self.units_wi, self.units_wo, self.n_units, self.expert_count, self.order,
                                  self.h, self.bad, self.counters))
        self.max_tokens = T
        self.max_units = max(1, T)  # runs per pass: one per expert token chunk <= T
        dev = self.device
        self.units_wi = torch.empty(self.max_units * _lib.WORK_BYTES, dtype=torch.uint8, device=dev)
        self.units_wo = torch.empty(self.max_units * _lib.WORK_BYTES, dtype=torch.uint8, device=dev)
        self.n_units = torch.zeros(4, dtype=torch.int32, device=dev)  # runs wi, tasks wi, runs wo, tasks wo
        self.expert_count = torch.zeros(self.E, dtype=torch.int32, device=dev)
        self.order = torch.zeros(max(1, T), dtype=torch.int32, device=dev)
        # FFN hidden: relu(bf16(wi @ x)) per token, bf16 rows (wo-pass x)
        ldh = (self.d_ff + 7) // 8 * 8  # 16-byte aligned hidden rows (bulk staging)
        hb = _lib.padded_empty(max(1, T) * ldh, torch.bfloat16, dev).view(max(1, T), ldh)
        if ldh > self.d_ff:
            hb[:, self.d_ff:].zero_()  # row padding: defined bytes for the dense pass's 16-byte tail copies
        self.h = hb[:, : self.d_ff]
        self.bad = torch.tensor([0, 2**31 - 1], dtype=torch.int32, device=dev)
        # fused step: {u64 arrival tickets, capacity C, -, 2 x C per-run counters} (qmoe_moe_step)
        self.counters = torch.zeros(2 * max(1, T) + 4, dtype=torch.int32, device=dev)
        self.counters[2] = max(1, T)

    def _write_descriptors(self) -> None:
        """Device array of qmoe_matrix descriptors (wi_e = 2e, wo_e = 2e + 1).
        Rewritten IN PLACE once allocated (e.g. when the decode-then-MMA column
        points are added), so graphs already holding its address stay valid."""
        import torch

        descs = (_lib.QmoeMatrix * (2 * self.E))()
        for e in range(self.E):
            descs[2 * e] = _lib.QmoeMatrix(*self.wi[e].descriptor())
            descs[2 * e + 1] = _lib.QmoeMatrix(*self.wo[e].descriptor())
        raw = torch.from_numpy(np.frombuffer(bytes(descs), dtype=np.uint8).copy())
        if getattr(self, "mats", None) is None:
            self.mats = raw.to(self.device)
        else:
            torch.cuda.current_stream(self.device).synchronize()  # no step in flight reads it
            self.mats.copy_(raw)

    @staticmethod
    def _aligned_rows(x) -> bool:
        esz = x.element_size()
        return (x.data_ptr() % 16 == 0 and (x.stride(0) * esz) % 16 == 0 and (x.shape[1] * esz) % 16 == 0
                and x.stride(1) == 1)

    # ------------------------------------------------------------------ device step
    LANES = 148 * 768  # resident lanes of the streaming kernel on a B200 (1 CTA x 24 warps per SM)
    MAX_LG = 3  # RAW layout: checkpoints stored for up to 8 lanes per row (16 measured no faster)

    def _runs_est(self, T: int) -> float:
        """expected distinct experts of a step under uniform top-1 routing"""
        return max(1.0, self.E * (1.0 - (1.0 - 1.0 / self.E) ** T))

    def lanes_per_row(self, T: int) -> tuple[int, int]:
        """log2 lanes per row (wi, wo) for a step of T tokens: enough lane
        segments to fill the GPU about twice, but segments of at least
        ~2 groups (shorter ones waste their partial groups) — ~1 group when
        the step is tiny (a generation step: latency, not lane efficiency,
        decides; T = 1 Switch-base-128: 18.3 -> 16.8 us)."""
        hit = self._lanes.get(T)
        if hit is None:
            runs = self._runs_est(T)
            out = []
            for kind, (rows, mg) in enumerate(((self.d_ff, self.mean_groups[0]), (self.d_model, self.mean_groups[1]))):
                cap = min(m.lg for m in (self.wi if kind == 0 else self.wo))
                # segments of at most ~8 groups (long rows: c2048), then more
                # lanes while the step's lanes fill the GPU less than half
                # (wi) / twice (wo: its runs start staggered behind wi's)
                lg = min(cap, max(0, int(np.ceil(np.log2(max(1.0, mg / 8.0))))))
                base_min = 2.0
                fill = self.LANES // 2 if kind == 0 else 2 * self.LANES
                while lg < cap and runs * rows * (1 << lg) < fill:
                    min_groups = base_min if runs * rows * (1 << lg) >= self.LANES // 4 else base_min / 2
                    if mg / (1 << (lg + 1)) < min_groups:
                        break
                    lg += 1
                out.append(lg)
            hit = self._lanes[T] = tuple(out)
        return hit

    # the fused step stages at most 32K entries (91-92% of lookups): a smaller
    # per-step fill than the whole table, measured 2% faster at T = 64 / 256
    STEP_HOT_MAX = 32768

    def hot_entries(self, T: int, wi: bool) -> int:
        """table entries to stage per SM: ~4x the codewords one SM decodes in
        the pass (small steps stage little: the fill is per CTA per launch)"""
        cw = self._runs_est(T) * (self.d_ff if wi else self.d_model) * 8 * self.mean_groups[0 if wi else 1]
        want = 4 * cw / 148
        h = 4096
        while h < want and h < 65536:
            h *= 2
        return h

    def plan(self, assign, stream=None) -> None:
        T = assign.shape[0]
        self._T = T
        lg_wi, lg_wo = self.lanes_per_row(T)
        _lib.check(_lib.lib.qmoe_moe_plan(
            _lib.ptr(assign), T, self.E, _lib.ptr(self.mats), self.tokens_per_unit, lg_wi, lg_wo, self.max_units,
            _lib.ptr(self.units_wi), _lib.ptr(self.units_wo),
            _lib.ptr(self.n_units), _lib.ptr(self.expert_count), _lib.ptr(self.order), _lib.stream_ptr(stream)))

    def _table(self) -> int:
        return self.codebook.table.data_ptr() if self.codebook is not None else 0

    def pass_wi(self, x, stream=None) -> None:
        import torch

        xt = _lib.QMOE_X_BF16 if x.dtype == torch.bfloat16 else _lib.QMOE_X_F32
        _lib.check(_lib.lib.qmoe_grouped_matvec(
            self.handle, self._table(), _lib.ptr(self.units_wi), _lib.ptr(self.n_units), self.max_units,
            self.d_model, self.tokens_per_unit, _lib.ptr(x), xt, x.stride(0), _lib.ptr(self.h),
            _lib.QMOE_Y_RELU_BF16, self.h.stride(0), self.hot_entries(self._T, True),
            _lib.ptr(self.bad), _lib.stream_ptr(stream)))

    def pass_wo(self, out, stream=None) -> None:
        _lib.check(_lib.lib.qmoe_grouped_matvec(
            self.handle, self._table(), _lib.ptr(self.units_wo), self.n_units.data_ptr() + 8, self.max_units,
            self.d_ff, self.tokens_per_unit, _lib.ptr(self.h), _lib.QMOE_X_BF16, self.h.stride(0), _lib.ptr(out),
            _lib.QMOE_Y_STORE_F32, out.stride(0), self.hot_entries(self._T, False),
            _lib.ptr(self.bad), _lib.stream_ptr(stream)))

    def forward_device(self, x, assign, out=None, stream=None):
        """x: (T, d_model) CUDA bf16/f32, assign: (T,) CUDA int32 expert ids.
        Returns out (T, d_model) float32 = per-token expert FFN output
        wo_e @ relu(wi_e @ x_t) with the reference's per-matvec rounding."""
        import torch

        T = x.shape[0]
        if out is None:
            out = torch.empty((T, self.d_model), dtype=torch.float32, device=self.device)
        if T == 0:
            return out
        if T > self.max_tokens:
            self._alloc(T)
        if x.dtype not in (torch.bfloat16, torch.float32):
            x = x.float()
        if not self._aligned_rows(x):
            buf = _lib.padded_empty(T * self.d_model, x.dtype, x.device).view(T, self.d_model)
            buf.copy_(x)
            x = buf
        if self.use_dense(T):
            self._zero_out(out, stream)
            self.plan(assign, stream)
            self.pass_dense(x, 0, self.h, _lib.QMOE_Y_RELU_BF16, stream)
            self.pass_dense(self.h, 1, out, _lib.QMOE_Y_STORE_F32, stream)
            return out
        if self.fused:
            try:
                self.step(x, assign, out, stream)
                return out
            except _lib.QmoeError as err:  # plan does not fit the fused kernel's shared memory
                if err.status != _lib.QMOE_EUNSUPPORTED:
                    raise
        if True:
            self._zero_out(out, stream)
            self.plan(assign, stream)
            self.pass_wi(x, stream)
            self.pass_wo(out, stream)
        return out

    @staticmethod
    def _zero_out(out, stream=None):
        """The grouped / dense passes store only the rows of tokens that have
        an expert; tokens without one (ids outside [0, E)) keep zero rows, as
        the composed reference leaves them (the fused step zeroes them in its
        kernel). A memset, capture-friendly."""
        import torch

        if stream is None:
            out.zero_()
        else:
            with torch.cuda.stream(stream):
                out.zero_()

    DENSE_MIN_TOKENS = 6.0  # tokens per touched expert from which decode-then-MMA wins (measured round 2, decode-once kernel: 4 -> streaming, 6 -> dense)

    def use_dense(self, T: int) -> bool:
        """Batched regime: each expert block decoded once and multiplied with
        all its tokens on the tensor cores (qmoe_dense_moe_pass)."""
        if not self._sparse_path or self.dense_mode == "never":
            return False
        return self.dense_mode == "always" or T / self._runs_est(T) >= self.DENSE_MIN_TOKENS

    def pass_dense(self, x, which: int, y, y_mode: int, stream=None) -> None:
        import torch

        T = self._T
        bn = 64 if T / self._runs_est(T) > 24 else 32
        rows, cols = (self.d_ff, self.d_model) if which == 0 else (self.d_model, self.d_ff)
        if x.dtype != torch.bfloat16 or x.stride(0) % 8 or x.data_ptr() % 16:
            # the pass reads 16-byte bf16 pieces of token rows (x is bf16-valued:
            # the layer input of the reference pipeline, or the bf16 hidden)
            with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
                xb = torch.zeros((x.shape[0], (cols + 7) // 8 * 8), dtype=torch.bfloat16, device=x.device)
                xb[:, :cols] = x[:, :cols]
            x = xb
        _lib.check(_lib.lib.qmoe_dense_moe_pass(
            self.handle, self._table(), _lib.ptr(self.mats), self.E, which, _lib.ptr(self.expert_count),
            _lib.ptr(self.order), rows, cols, _lib.ptr(x), _lib.QMOE_X_BF16, x.stride(0), _lib.ptr(y), y_mode,
            y.stride(0), bn, 0, _lib.stream_ptr(stream)))

    def step(self, x, assign, out, stream=None, gate=None) -> None:
        """The whole step as one cooperative launch (qmoe_moe_step; with
        `gate` (f32[T] on the device) the output rows are scaled by it,
        qmoe_moe_step_gated)."""
        import torch

        T = assign.shape[0]
        self._T = T
        lg_wi, lg_wo = self.lanes_per_row(T)
        xt = _lib.QMOE_X_BF16 if x.dtype == torch.bfloat16 else _lib.QMOE_X_F32
        _lib.check(_lib.lib.qmoe_moe_step_gated(
            self.handle, self._table(), _lib.ptr(assign), T, self.E, _lib.ptr(self.mats), self.tokens_per_unit,
            lg_wi, lg_wo, self.d_model, self.d_ff, _lib.ptr(x), xt, x.stride(0), _lib.ptr(self.h), self.h.stride(0),
            _lib.ptr(out), out.stride(0), _lib.ptr(self.counters),
            _lib.ptr(self.order) if self.publish_plan else 0, _lib.ptr(self.expert_count) if self.publish_plan else 0,
            min(self.STEP_HOT_MAX, max(self.hot_entries(T, True), self.hot_entries(T, False))), _lib.ptr(gate),
            _lib.stream_ptr(stream)))

    def step_resid(self, x, assign, out, gate=None, stream=None, hash_mult=None, assign_out=None) -> None:
        """One residual block in one launch (qmoe_moe_step_resid): out (bf16,
        T x d_model) = bf16(x + [gate *] moe(x)), x a bf16 CUDA tensor with
        16-byte aligned rows; tokens without an expert pass x through. With
        hash_mult (a DeviceRouter's hash multipliers) the launch routes the
        tokens itself (RouterSim hash rule) and `assign` may be None; the ids
        are written to assign_out when given."""
        T = x.shape[0]
        if T > self.max_tokens:
            self._alloc(T)
        self._T = T
        lg_wi, lg_wo = self.lanes_per_row(T)
        _lib.check(_lib.lib.qmoe_moe_step_resid(
            self.handle, self._table(), _lib.ptr(assign), T, self.E, _lib.ptr(self.mats), self.tokens_per_unit,
            lg_wi, lg_wo, self.d_model, self.d_ff, _lib.ptr(x), x.stride(0), _lib.ptr(self.h), self.h.stride(0),
            _lib.ptr(out), out.stride(0), _lib.ptr(self.counters),
            min(self.STEP_HOT_MAX, max(self.hot_entries(T, True), self.hot_entries(T, False))), _lib.ptr(gate),
            _lib.ptr(hash_mult), _lib.ptr(assign_out), _lib.stream_ptr(stream)))

    def forward_routed(self, x, router, gated: bool = False, out=None, stream=None):
        """Router + layer on the device: expert ids (and, with `gated`, the
        top-1 softmax probability scaling each output row — the Switch combine;
        the reference has none) from `router` (pipeline.DeviceRouter), then the
        step. Returns (out, assign, gate)."""
        import torch

        assign, gate = router(x, gated=gated, stream=stream)
        T = x.shape[0]
        if out is None:
            out = torch.empty((T, self.d_model), dtype=torch.float32, device=self.device)
        if self.fused and not self.use_dense(T) and T <= self.max_tokens:
            try:
                self.step(x, assign, out, stream, gate=gate)
                return out, assign, gate
            except _lib.QmoeError as err:
                if err.status != _lib.QMOE_EUNSUPPORTED:
                    raise
        self.forward_device(x, assign, out=out, stream=stream)
        if gate is not None:
            out.mul_(gate[:, None])
        return out, assign, gate

    GRAPH_CACHE = 8  # (token count, path, slot) keys with a captured host-API graph per layer
    _HOST_STAGING = threading.local()  # per thread: (bytes, T, d_model) -> pinned (input, output) buffers

    def forward(self, x: np.ndarray, assign: np.ndarray) -> np.ndarray:
        """Host API: numpy tokens + expert ids in, numpy outputs back.

        Per token count T the layer keeps pinned host staging buffers, device
        buffers and (after the first call) a CUDA graph holding the H2D copies,
        the step and the D2H copy, so a call is: copy into pinned memory,
        one graph launch, one stream sync, copy out. A layer (its hidden,
        counters and captured graphs) serves one thread at a time."""
        import torch

        x = np.ascontiguousarray(x, np.float32)
        a = np.ascontiguousarray(assign, np.int32)
        T = int(x.shape[0])
        if x.ndim != 2 or x.shape[1] != self.d_model or a.shape != (T,):
            raise ValueError(f"expected x (T, {self.d_model}) and assign (T,)")
        st = self._launch_host(x, a, slot=0, overlap=False)
        st["done"].synchronize()
        return st["yv"].copy()

    def _launch_host(self, x: np.ndarray, a: np.ndarray, slot: int, overlap: bool) -> dict:
        """Stage x / ids into the pinned buffers of `slot` and launch the step
        (a CUDA graph captured on first use per (T, path, slot, overlap)),
        recording its completion event. overlap=False: one graph holds the
        input copy and the step (lowest latency for a blocking call);
        overlap=True: the input copy runs on a copy stream, so it overlaps the
        step in flight (forward_stream), and the graph holds the step only."""
        import torch

        T = int(x.shape[0])
        key = (T, self.use_dense(T), slot)  # the captured graph holds one path
        st = self._stages.get(key)
        if st is None:
            st = self._host_stage(T, key)
        np.copyto(st["xv"], x)
        np.copyto(st["av"], a)
        stream = torch.cuda.current_stream(self.device)
        if overlap:
            with torch.cuda.stream(st["copy_stream"]):
                st["in_d"].copy_(st["in_h"], non_blocking=True)
                st["in_ready"].record()
            stream.wait_event(st["in_ready"])
            body = st["step"]
        else:
            body = st["copy_step"]
        g = st["graphs"].get(overlap)
        if g is not None:
            g.replay()
        else:
            body()  # first call runs eagerly (lazy setup), then the graph is captured
            stream.synchronize()
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    body()
                st["graphs"][overlap] = g
                g.replay()
            except RuntimeError:  # capture not possible here: stay eager
                body()
        st["done"].record()
        return st

    def _host_stage(self, T: int, key) -> dict:
        """Pinned staging for T tokens: ONE input buffer (x f32 rows, then the
        int32 expert ids) so the step's inputs cross the link in one copy; the
        step writes its output rows straight into pinned host memory (mapped,
        UVA), which saves the D2H copy node and its dependency latency
        (measured: tools/e2e_breakdown.py)."""
        import torch

        if len(self._stages) >= self.GRAPH_CACHE:
            self._stages.pop(next(iter(self._stages)))
        xb = T * self.d_model * 4
        nb = xb + ((T * 4 + 15) & ~15)
        # pinned staging shared by every layer of the same shape (calls are
        # synchronous): a model's layers reuse host memory that stays in the
        # CPU caches
        shared = CompressedMoELayer._HOST_STAGING.__dict__.setdefault("bufs", {})  # per thread
        hkey = (nb, T, self.d_model, key[2])  # one set per pipeline slot (forward_stream)
        if hkey not in shared:
            shared[hkey] = (torch.empty(nb, dtype=torch.uint8, pin_memory=True),
                            torch.empty((T, self.d_model), dtype=torch.float32, pin_memory=True))
        in_h, y_h = shared[hkey]
        in_d = torch.empty(nb, dtype=torch.uint8, device=self.device)
        x_d = in_d[:xb].view(torch.float32).view(T, self.d_model)
        a_d = in_d[xb:xb + T * 4].view(torch.int32)

        direct = self.fused and not key[1]  # the fused step writes every output row (dropped ones: zero)
        y_d = None if direct else torch.empty((T, self.d_model), dtype=torch.float32, device=self.device)

        def step():  # the step only (its input copy enqueued separately)
            if direct:
                self.forward_device(x_d, a_d, out=y_h)
            else:  # grouped / decode-then-MMA passes: device output, then one D2H copy
                self.forward_device(x_d, a_d, out=y_d)
                y_h.copy_(y_d, non_blocking=True)

        def copy_step():
            in_d.copy_(in_h, non_blocking=True)
            step()

        st = {
            "in_h": in_h, "in_d": in_d, "y_h": y_h, "step": step, "copy_step": copy_step, "graphs": {},
            "xv": in_h[:xb].numpy().view(np.float32).reshape(T, self.d_model),
            "av": in_h[xb:xb + T * 4].numpy().view(np.int32),
            "yv": y_h.numpy(),
            "done": torch.cuda.Event(),
            "in_ready": torch.cuda.Event(),
            "copy_stream": self._copy_stream(),
        }
        self._stages[key] = st
        return st

    _COPY_STREAMS = {}

    def _copy_stream(self):
        """One host-to-device copy stream per device (host API input copies)."""
        import torch

        key = self.device.index if self.device.index is not None else torch.cuda.current_device()
        if key not in CompressedMoELayer._COPY_STREAMS:
            CompressedMoELayer._COPY_STREAMS[key] = torch.cuda.Stream(self.device)
        return CompressedMoELayer._COPY_STREAMS[key]

    def touched_bytes(self, assign: np.ndarray) -> int:
        """Compressed bytes one step must stream: each distinct expert once."""
        return int(self.expert_bytes[np.unique(np.asarray(assign))].sum())


def load_moe_layer(wi_path: str, wo_path: str, dic: Dictionary, max_tokens: int = 64, device=None,
                   rows_per_expert: tuple[int, int] | None = None, **layer_kw) -> CompressedMoELayer:
    """A compressed MoE layer from two stacked checkpoints:
    every expert's wi (d_ff x d_model) stacked by rows in one QMOE0001 file
    and every wo (d_model x d_ff) in another — what the reference CLI writes
    for a stacked quantized layer (cli.py:150-153 _stack_quantized, :194-201
    encode + write_checkpoint, rows_per_expert in its report). d_model = the
    wi file's cols, d_ff = the wo file's cols, E = wi rows / d_ff. Each file is
    read into pinned memory, checked exactly as read_checkpoint, copied to the
    device once and split into per-expert matrices (codec.read_stacked_device)."""
    import struct

    from .codec import read_stacked_device

    shapes = []
    for path in (wi_path, wo_path):
        with open(path, "rb") as fh:
            head = np.frombuffer(fh.read(32), dtype=np.uint8)
        if len(head) < 32 or bytes(head[:8]) != b"QMOE0001":
            raise CorruptionError_("not a checkpoint file (bad magic)")
        shapes.append(struct.unpack_from("<QQ", head, 8))
    (wi_rows, d_model), (wo_rows, d_ff) = shapes
    if d_ff == 0 or d_model == 0 or wi_rows % d_ff or wo_rows % d_model or wi_rows // d_ff != wo_rows // d_model:
        raise ValueError(f"stacked checkpoints disagree: wi {wi_rows}x{d_model}, wo {wo_rows}x{d_ff}")
    if rows_per_expert is not None and tuple(rows_per_expert) != (d_ff, d_model):
        raise ValueError(f"rows_per_expert {tuple(rows_per_expert)} != (d_ff, d_model) = ({d_ff}, {d_model})")
    wi = read_stacked_device(wi_path, dic, d_ff, device)
    wo = read_stacked_device(wo_path, dic, d_model, device)
    return CompressedMoELayer(wi, wo, dic, max_tokens=max_tokens, **layer_kw)


def forward_stream(items, depth: int = 2):
    """Pipelined host API: `items` yields (layer, x, assign) — numpy tokens
    (T, d_model) and expert ids, any CompressedMoELayer per item — and this
    yields each step's numpy output rows in order, like layer.forward(x,
    assign). Up to `depth` steps are in flight: while the GPU runs step i
    (its H2D copy, fused step and output rows written to pinned host memory,
    one CUDA graph), the host stages step i + 1's inputs into the other pinned
    buffers and copies step i - 1's outputs out. Each pipeline slot has its own
    pinned buffers and graphs; a layer serves one thread at a time."""
    from collections import deque

    pending = deque()
    for i, (layer, x, assign) in enumerate(items):
        if len(pending) == depth:  # the slot about to be reused: its step must be done
            st = pending.popleft()
            st["done"].synchronize()
            yield st["yv"].copy()
        x = np.ascontiguousarray(x, np.float32)
        a = np.ascontiguousarray(assign, np.int32)
        if x.ndim != 2 or x.shape[1] != layer.d_model or a.shape != (x.shape[0],):
            raise ValueError(f"expected x (T, {layer.d_model}) and assign (T,)")
        pending.append(layer._launch_host(x, a, slot=i % depth, overlap=True))
    while pending:
        st = pending.popleft()
        st["done"].synchronize()
        yield st["yv"].copy()


class CompressedMoEModel:
    """A stack of residual compressed MoE blocks, the synthetic model of
    BASELINE config 5: for every layer l, expert ids (and, when gated, the
    top-1 softmax gate) from its router on the device (pipeline.DeviceRouter,
    the reference's RouterSim rules), then ONE fused launch computing
    x_{l+1} = bf16(x_l + [gate *] wo_e relu(wi_e x_l)) (qmoe_moe_step_resid).
    Activations stay bf16 in HBM; the whole forward is device-only and
    CUDA-graph capturable: ONE launch per layer with ungated hash routing (the
    block hashes its tokens itself), three with argmax (score + select +
    block)."""

    def __init__(self, layers: list, routers: list, gated: bool = False):
        if len(layers) != len(routers) or not layers:
            raise ValueError("need one router per layer")
        d = layers[0].d_model
        if any(lay.d_model != d for lay in layers) or any(r.dim != d for r in routers):
            raise ValueError("layers and routers must share d_model")
        self.layers, self.routers, self.gated = layers, routers, gated
        self.d_model = d
        self._bufs = {}

    def _buffers(self, T: int, device):
        import torch

        b = self._bufs.get(T)
        if b is None:
            ld = (self.d_model + 7) // 8 * 8  # 16-byte aligned bf16 rows
            b = self._bufs[T] = [_lib.padded_empty(max(1, T) * ld, torch.bfloat16, device).view(max(1, T), ld)
                                 [:T, : self.d_model] for _ in range(2)]
        return b

    def forward_device(self, x, stream=None, keep: bool = False):
        """x: (T, d_model) bf16 CUDA tensor -> the last layer's output (a new
        bf16 tensor); keep=True also returns every layer's input and routing."""
        import torch

        T = x.shape[0]
        bufs = self._buffers(T, x.device)
        cur = bufs[0]
        cur.copy_(x)
        trace = []
        for l, (lay, router) in enumerate(zip(self.layers, self.routers)):
            nxt = bufs[(l + 1) % 2]
            if router.rule == _lib.QMOE_ROUTE_HASH and not self.gated:  # router fused into the block
                ids = torch.empty(T, dtype=torch.int32, device=x.device) if keep else None
                xin = cur.clone() if keep else None
                lay.step_resid(cur, None, nxt, stream=stream, hash_mult=router.mult, assign_out=ids)
                if keep:
                    trace.append((xin, ids))
            else:
                assign, gate = router(cur, gated=self.gated, stream=stream)
                if keep:
                    trace.append((cur.clone(), assign.clone()))
                lay.step_resid(cur, assign, nxt, gate=gate, stream=stream)
            cur = nxt
        out = cur.clone()
        return (out, trace) if keep else out
