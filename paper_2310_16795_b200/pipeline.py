"""Routing and token-buffer semantics the MoE layer follows (drop-in subset of
moepack/pipeline.py: `RouterSim`, `ListBuffer.gather_expert_tokens` order).

`RouterSim(rule="argmax")` is the reference's deterministic top-1 router
(pipeline.py:142-182): argmax of x . P (+ skew ramp) with P ~ N(0, 1) drawn
from the seed, in float64. It runs on the host exactly as in the reference so
both the GPU path and the CPU oracle see identical expert ids; the GPU router
(`route_device`) computes the same argmax on the device for the fused step.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

ROUTER_RULES = ("hash", "argmax")


@dataclass(frozen=True)
class RouterSim:
    num_experts: int
    rule: str = "hash"
    seed: int = 0
    skew: float = 0.0

    def __post_init__(self):
        if self.num_experts < 1:
            raise ValueError("need at least one expert")
        if self.rule not in ROUTER_RULES:
            raise ValueError(f"unknown router rule {self.rule!r}")

    def projection(self, dim: int) -> np.ndarray:
        """The fixed (dim, E) float64 map of the argmax rule."""
        return np.random.default_rng(self.seed).normal(size=(dim, self.num_experts))

    def bias(self, dim: int) -> np.ndarray:
        return self.skew * math.sqrt(dim) * np.linspace(1.0, 0.0, self.num_experts)

    def assign(self, tokens: np.ndarray) -> np.ndarray:
        tokens = np.asarray(tokens, dtype=np.float32)
        if tokens.ndim != 2:
            raise ValueError("tokens must be (n, dim)")
        rng = np.random.default_rng(self.seed)
        if self.rule == "hash":
            mult = rng.integers(1, 1 << 63, size=tokens.shape[1], dtype=np.uint64) | 1
            bits = np.ascontiguousarray(tokens).view(np.uint32).astype(np.uint64)
            h = (bits * mult[None, :]).sum(axis=1, dtype=np.uint64)
            h ^= h >> np.uint64(33)
            h *= np.uint64(0xFF51AFD7ED558CCD)
            h ^= h >> np.uint64(33)
            return (h % np.uint64(self.num_experts)).astype(np.int32)
        proj = rng.normal(size=(tokens.shape[1], self.num_experts))
        scores = tokens.astype(np.float64) @ proj
        return np.argmax(scores + self.bias(tokens.shape[1])[None, :], axis=1).astype(np.int32)


def route_device(x, proj_dev, bias_dev):
    """GPU top-1 argmax router: float64 scores x @ P + bias on the device
    (same arithmetic type as RouterSim; ties resolve to the lowest index as
    np.argmax). x: (T, d) CUDA tensor, proj_dev: (d, E) float64."""
    import torch

    s = x.to(torch.float64) @ proj_dev
    if bias_dev is not None:
        s = s + bias_dev[None, :]
    return torch.argmax(s, dim=1).to(torch.int32)


def gather_order(assign: np.ndarray, num_experts: int) -> list[np.ndarray]:
    """Per expert, token positions in buffer order (pipeline.py:86-90)."""
    return [np.flatnonzero(assign == e) for e in range(num_experts)]
