"""Expert-parallel (EP) compressed MoE layer across ranks.

Layout: E experts in contiguous blocks, expert e lives on rank e // (E / P);
each rank holds only its block's compressed matrices (plus the replicated
dictionary / codebook). One forward, per rank, for that rank's T local tokens:

  1. route   top-1 expert ids (host RouterSim or GPU router) -> destination
             rank = id // (E / P); tokens are grouped by destination rank,
             stable in buffer order;
  2. dispatch  all_to_all_single of the token rows (+ their expert ids) —
             NCCL over NVLink on B200 boxes, gloo on CPU for the tests;
  3. compute   the local CompressedMoELayer on the received tokens (expert
             ids rebased to the local block);
  4. combine   all_to_all_single of the outputs back, scattered to the
             tokens' original positions.

Per-token arithmetic never depends on placement, so outputs are bit-identical
to the single-device layer (tested with gloo, world size 2, tests/test_ep.py).
The exchange is a real data dependency (tokens must reach their expert), so it
is the only collective on the path.
"""

from __future__ import annotations

from typing import Callable

import numpy as np


class ExpertParallelMoE:
    def __init__(self, num_experts: int, local_fn: Callable, group=None):
        """local_fn(x_recv (n, d) tensor, local_ids (n,) int32 tensor) ->
        y_recv (n, d_out) float32 tensor, for experts of this rank's block."""
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
        self.last_split = None

    def owner(self, expert_ids):
        return expert_ids // self.per_rank

    def forward(self, x, assign):
        """x: (T, d) tensor, assign: (T,) int32 tensor of global expert ids.
        Returns y (T, d_out) float32 in the original token order."""
        import torch

        dist = self.dist
        T = x.shape[0]
        dest = (assign.to(torch.int64) // self.per_rank).to(torch.int64)
        order = torch.argsort(dest, stable=True)  # group by destination, buffer order kept
        send_counts = torch.bincount(dest, minlength=self.world).to(torch.int64)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc = send_counts.cpu().tolist()
        rc = recv_counts.cpu().tolist()
        self.last_split = (sc, rc)
        x_send = x[order].contiguous()
        id_send = assign[order].to(torch.int32).contiguous()
        n_recv = int(sum(rc))
        x_recv = torch.empty((n_recv, x.shape[1]), dtype=x.dtype, device=x.device)
        id_recv = torch.empty(n_recv, dtype=torch.int32, device=x.device)
        dist.all_to_all_single(x_recv, x_send, rc, sc, group=self.group)
        dist.all_to_all_single(id_recv, id_send, rc, sc, group=self.group)
        local_ids = id_recv - self.rank * self.per_rank
        y_recv = self.local_fn(x_recv, local_ids).to(torch.float32).contiguous()
        y_send = torch.empty((T, y_recv.shape[1]), dtype=torch.float32, device=x.device)
        dist.all_to_all_single(y_send, y_recv, sc, rc, group=self.group)
        y = torch.empty_like(y_send)
        y[order] = y_send
        return y


def shard_experts(E: int, world: int, rank: int) -> range:
    """Expert ids owned by `rank` (contiguous block)."""
    per = E // world
    return range(rank * per, (rank + 1) * per)


def token_split(assign: np.ndarray, E: int, world: int) -> np.ndarray:
    """Tokens each rank sends to each destination (host helper for tests)."""
    dest = np.asarray(assign) // (E // world)
    return np.bincount(dest, minlength=world)
