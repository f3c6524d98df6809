"""Routing and token-buffer semantics the MoE layer follows (drop-in subset of
moepack/pipeline.py: `RouterSim`, `ListBuffer.gather_expert_tokens` order).

`RouterSim(rule="argmax")` is the reference's deterministic top-1 router
(pipeline.py:142-182): argmax of x . P (+ skew ramp) with P ~ N(0, 1) drawn
from the seed, in float64. It runs on the host exactly as in the reference so
both the GPU path and the CPU oracle see identical expert ids; `DeviceRouter`
computes the same routing on the device (qmoe_route kernels) for the fused
step, optionally with the top-1 softmax gate for combine scaling.
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


class DeviceRouter:
    """RouterSim on the device through the library's qmoe_route
    kernels: the same projection / multipliers the reference draws from the
    seed (pipeline.py:168-182), resident in HBM; tokens never leave the GPU.
    Hash routing is bit-exact; argmax routing matches up to near-ties (the
    float64 summation order differs from numpy's matmul)."""

    def __init__(self, sim: RouterSim, dim: int, device=None):
        import torch

        from . import _lib

        self.sim, self.dim = sim, int(dim)
        self.device = torch.device(device if device is not None else "cuda")
        rng = np.random.default_rng(sim.seed)
        self.rule = _lib.QMOE_ROUTE_HASH if sim.rule == "hash" else _lib.QMOE_ROUTE_ARGMAX
        self.mult = self.proj = self.bias = None
        if sim.rule == "hash":
            mult = rng.integers(1, 1 << 63, size=self.dim, dtype=np.uint64) | np.uint64(1)
            self.mult = torch.from_numpy(mult.view(np.int64).copy()).to(self.device)
        else:
            self.proj = torch.from_numpy(rng.normal(size=(self.dim, sim.num_experts))).to(self.device)
            if sim.skew != 0.0:
                self.bias = torch.from_numpy(sim.bias(self.dim)).to(self.device)
        self._scores = None

    def __call__(self, x, gated: bool = False, stream=None):
        """x: (T, dim) CUDA bf16 / f32 -> (expert ids int32[T], gate f32[T] or None)."""
        import torch

        from . import _lib

        if x.ndim != 2 or x.shape[1] != self.dim or not x.is_cuda or (x.shape[0] > 0 and x.stride(1) != 1):
            raise ValueError(f"tokens must be a row-major CUDA (n, {self.dim}) tensor")
        if x.shape[0] == 0:
            empty = torch.empty(0, dtype=torch.int32, device=self.device)
            return empty, (torch.empty(0, dtype=torch.float32, device=self.device) if gated else None)
        if x.dtype not in (torch.bfloat16, torch.float32):
            x = x.float()
        T, E = x.shape[0], self.sim.num_experts
        assign = torch.empty(T, dtype=torch.int32, device=self.device)
        gate = torch.empty(T, dtype=torch.float32, device=self.device) if gated else None
        if self.rule == _lib.QMOE_ROUTE_ARGMAX:
            need = int(_lib.lib.qmoe_route_scratch(T, self.dim, E))
            if self._scores is None or self._scores.numel() < need:
                self._scores = torch.empty(need, dtype=torch.float64, device=self.device)
        xt = _lib.QMOE_X_BF16 if x.dtype == torch.bfloat16 else _lib.QMOE_X_F32
        _lib.check(_lib.lib.qmoe_route(self.rule, _lib.ptr(x), xt, x.stride(0), T, self.dim, E,
                                       _lib.ptr(self.proj), _lib.ptr(self.bias), _lib.ptr(self.mult),
                                       _lib.ptr(self._scores), _lib.ptr(assign), _lib.ptr(gate),
                                       _lib.stream_ptr(stream)))
        return assign, gate


def route_device(x, sim: RouterSim, device=None):
    """Convenience: expert ids of x (CUDA tensor) under `sim`, on the device."""
    return DeviceRouter(sim, x.shape[1], device if device is not None else x.device)(x)[0]


def gather_order(assign: np.ndarray, num_experts: int) -> list[np.ndarray]:
    """Per expert, token positions in buffer order (pipeline.py:86-90)."""
    return [np.flatnonzero(assign == e) for e in range(num_experts)]
