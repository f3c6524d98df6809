"""Expert-parallel (EP) compressed MoE layer across ranks.

Layout: E experts in contiguous blocks, expert e lives on rank e // (E / P);
each rank holds only its block's compressed matrices (plus the replicated
dictionary / codebook). One forward, per rank, for that rank's T local tokens:

  1. route   top-1 expert ids (host RouterSim or GPU router) -> destination
             rank = id // (E / P); tokens are grouped by destination rank,
             stable in buffer order;
  2. dispatch  all_to_all_single of the token rows (+ their expert ids) into
             fixed slots: every rank reserves C slots per destination, C =
             the layer's token capacity (`max_tokens`, the same on every
             rank; a rank may bring any T <= C tokens), a token's slot = its
             stable rank among the tokens going to the same rank, empty slots
             carry expert id -1. Equal splits mean no host round trip for the
             counts, so the whole layer is device-only and CUDA-graph
             capturable — NCCL over NVLink on B200 boxes, gloo on CPU for the
             tests;
  3. compute   the local CompressedMoELayer on the received W x C slots
             (expert ids rebased to the local block; -1 slots are dropped by
             its dispatcher plan);
  4. combine   all_to_all_single of the slot outputs back — bf16 rows on the
             device path (exact: an expert output is a bf16-rounded value,
             codec.py:243) — gathered to the tokens' original positions.

Per-token arithmetic never depends on placement, so outputs are bit-identical
to the single-device layer (tested with gloo, world size 2, tests/test_ep.py).
The exchange is a real data dependency (tokens must reach their expert), so it
is the only collective on the path.
"""

from __future__ import annotations

from typing import Callable

import numpy as np


class ExpertParallelMoE:
    def __init__(self, num_experts: int, local_fn: Callable, group=None, max_tokens: int | None = None):
        """local_fn(x_recv (n, d) tensor, local_ids (n,) int32 tensor) ->
        y_recv (n, d_out) float32 tensor, for experts of this rank's block.
        max_tokens: slots per destination rank (every rank must pass the same
        value); None = the largest T of the first forward over all ranks (one
        all-reduce, on the first call only). A forward with more tokens than
        the capacity raises ValueError."""
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if num_experts % self.world:
            raise ValueError("num_experts must divide evenly over the ranks")
        self.E = num_experts
        self.per_rank = num_experts // self.world
        self.local_fn = local_fn
        self.capacity = max_tokens
        self.last_split = None

    def _all_to_all(self, out, inp) -> None:
        """Equal-split all-to-all. NCCL moves device tensors directly (NVLink
        on a B200 box); a gloo group (CPU tests, several ranks sharing one
        GPU) stages device tensors through host memory."""
        if inp.is_cuda and self.dist.get_backend(self.group) == "gloo":
            o = out.new_empty(out.shape, device="cpu")
            self.dist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
        else:
            self.dist.all_to_all_single(out, inp, group=self.group)

    def owner(self, expert_ids):
        return expert_ids // self.per_rank

    def forward(self, x, assign):
        """x: (T, d) tensor, assign: (T,) int32 tensor of global expert ids
        (ids outside [0, E) get no expert: zero output rows). Returns y
        (T, d_out) float32 in the original token order."""
        import torch

        dist = self.dist
        T, W = x.shape[0], self.world
        if self.capacity is None:  # first call, on every rank: agree on the slot count
            on_dev = x.is_cuda and dist.get_backend(self.group) != "gloo"
            t = torch.tensor([T], dtype=torch.int64, device=x.device if on_dev else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            self.capacity = max(1, int(t.item()))
        if T > self.capacity:
            raise ValueError(f"{T} tokens exceed the layer's capacity of {self.capacity} per rank")
        C = self.capacity
        if x.is_cuda and W <= 64 and (x.shape[1] * x.element_size()) % 16 == 0:
            return self._forward_device(x, assign, C)
        a64 = assign.to(torch.int64)
        valid = (a64 >= 0) & (a64 < self.E)
        dest = torch.where(valid, a64 // self.per_rank, torch.zeros_like(a64))
        onehot = torch.nn.functional.one_hot(dest, W) * valid[:, None].to(torch.int64)
        pos = (torch.cumsum(onehot, 0) - onehot).gather(1, dest[:, None])[:, 0]  # stable rank per destination
        slot = torch.where(valid, dest * C + pos, torch.full_like(dest, W * C))  # W*C: a spill slot for invalid
        x_send = torch.zeros((W * C + 1, x.shape[1]), dtype=x.dtype, device=x.device)
        id_send = torch.full((W * C + 1,), -1, dtype=torch.int32, device=x.device)
        x_send[slot] = x
        id_send[slot] = torch.where(valid, a64 - dest * self.per_rank, torch.full_like(a64, -1)).to(torch.int32)
        x_send, id_send = x_send[: W * C], id_send[: W * C]
        self.last_split = (onehot.sum(0), None)  # tokens sent to each rank (device tensor)
        x_recv = torch.empty_like(x_send)
        id_recv = torch.empty_like(id_send)
        self._all_to_all(x_recv, x_send)
        self._all_to_all(id_recv, id_send)
        y_recv = self.local_fn(x_recv, id_recv).to(torch.float32).contiguous()
        y_back = torch.empty_like(y_recv)
        self._all_to_all(y_back, y_recv)
        y_back = torch.cat([y_back, torch.zeros((1, y_back.shape[1]), dtype=y_back.dtype, device=y_back.device)])
        y = y_back[slot]  # invalid tokens read the zero spill row
        return y


    def _forward_device(self, x, assign, C: int):
        """CUDA path of forward: slots + row scatter / gather as small library
        kernels (qmoe_ep_slots, qmoe_ep_rows, qmoe_ep_combine) around the
        NCCL all-to-alls — device-only, graph-capturable. The combine moves
        bf16 rows (half the bytes of f32, and exact for expert outputs)."""
        import torch

        from . import _lib

        T, W, d = x.shape[0], self.world, x.shape[1]
        x = x.contiguous()
        a = assign.to(torch.int32).contiguous()
        slot = torch.empty(max(1, T), dtype=torch.int32, device=x.device)
        id_send = torch.empty(W * C, dtype=torch.int32, device=x.device)
        counts = torch.empty(W, dtype=torch.int32, device=x.device)
        x_send = torch.zeros((W * C, d), dtype=x.dtype, device=x.device)
        s = _lib.stream_ptr()
        _lib.check(_lib.lib.qmoe_ep_slots(_lib.ptr(a), T, self.E, W, C, _lib.ptr(slot), _lib.ptr(id_send),
                                          _lib.ptr(counts), s))
        _lib.check(_lib.lib.qmoe_ep_rows(_lib.ptr(x), _lib.ptr(x_send), T, d * x.element_size(), _lib.ptr(slot), 1, s))
        self.last_split = (counts, None)
        x_recv = torch.empty_like(x_send)
        id_recv = torch.empty_like(id_send)
        self._all_to_all(x_recv, x_send)
        self._all_to_all(id_recv, id_send)
        y_recv = self.local_fn(x_recv, id_recv).to(torch.bfloat16).contiguous()  # exact (bf16-valued rows)
        y_back = torch.empty_like(y_recv)
        self._all_to_all(y_back, y_recv)
        d_out = y_back.shape[1]
        y = torch.empty((T, d_out), dtype=torch.float32, device=x.device)
        _lib.check(_lib.lib.qmoe_ep_combine(_lib.ptr(y_back), _lib.ptr(y), T, d_out, _lib.ptr(slot), s))
        return y


def shard_experts(E: int, world: int, rank: int) -> range:
    """Expert ids owned by `rank` (contiguous block)."""
    per = E // world
    return range(rank * per, (rank + 1) * per)


def token_split(assign: np.ndarray, E: int, world: int) -> np.ndarray:
    """Tokens each rank sends to each destination (host helper for tests)."""
    dest = np.asarray(assign) // (E // world)
    return np.bincount(dest, minlength=world)
