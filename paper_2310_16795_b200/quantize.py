"""Ternary quantization types and the RTN producer of synthetic weights
(drop-in subset of moepack/quantize.py: `TernaryMatrix`, `QuantGrid`,
`make_grid`, `rtn_quantize`, `reconstruction_levels`).

The GPTQ solver (quantize.py:238-430) is an offline compression step and is
out of scope for this hot-path build. RTN itself runs on the GPU
(libqmoe `rtn_kernel`): it produces the random-init ternary experts that the
benchmarks compress with the bit-exact GPU encoder.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .bf16 import bf16_bits_to_f32, f32_to_bf16_bits

MODE_TERNARY = "ternary"
MODE_2BIT = "2bit"  # the reference's 2-bit grid (quantize.py:24-25): named, not supported (ternary codec only)


def reconstruction_levels(mode: str, row_minmax: np.ndarray) -> np.ndarray:
    """(rows, 3) float32 [0, f32(bf16 min), f32(bf16 max)] (quantize.py:38-51)."""
    if mode != MODE_TERNARY:
        raise ValueError(f"unsupported grid mode {mode!r} (ternary only)")
    mn = bf16_bits_to_f32(row_minmax[:, 0])
    mx = bf16_bits_to_f32(row_minmax[:, 1])
    return np.stack([np.zeros_like(mn), mn, mx], axis=1)


@dataclass(frozen=True)
class QuantGrid:
    mode: str
    row_min: np.ndarray
    row_max: np.ndarray

    def __post_init__(self):
        if self.mode != MODE_TERNARY:
            raise ValueError(f"unsupported grid mode {self.mode!r} (ternary only)")
        if self.row_min.shape != self.row_max.shape or self.row_min.ndim != 1:
            raise ValueError("row_min and row_max must be equal-length vectors")

    @property
    def rows(self) -> int:
        return self.row_min.shape[0]

    def minmax_bits(self) -> np.ndarray:
        return np.stack([f32_to_bf16_bits(self.row_min), f32_to_bf16_bits(self.row_max)], axis=1)

    def levels(self) -> np.ndarray:
        return reconstruction_levels(self.mode, self.minmax_bits())


def make_grid(w: np.ndarray, mode: str = MODE_TERNARY) -> QuantGrid:
    """Row extrema grid (quantize.py:91-107)."""
    w = np.asarray(w)
    if w.ndim != 2 or w.shape[0] < 1 or w.shape[1] < 1:
        raise ValueError("weights must be a non-empty 2d array")
    if not np.isfinite(w).all():
        raise ValueError("weights must be finite")
    return QuantGrid(mode=mode, row_min=w.min(axis=1).astype(np.float32), row_max=w.max(axis=1).astype(np.float32))


@dataclass
class TernaryMatrix:
    """codes in {0, 1, 2}: 0 -> 0.0, 1 -> row min, 2 -> row max (quantize.py:136-172)."""

    codes: np.ndarray
    row_minmax: np.ndarray

    mode = MODE_TERNARY

    def __post_init__(self):
        if self.codes.ndim != 2 or self.codes.dtype != np.uint8:
            raise ValueError("codes must be a 2d uint8 array")
        if self.codes.size and int(self.codes.max()) >= 3:
            raise ValueError("codes must lie in [0, 3)")
        if self.row_minmax.shape != (self.codes.shape[0], 2):
            raise ValueError("row_minmax must be (rows, 2)")
        if self.row_minmax.dtype != np.uint16:
            raise ValueError("row_minmax must hold uint16 bit patterns")

    @property
    def rows(self) -> int:
        return self.codes.shape[0]

    @property
    def cols(self) -> int:
        return self.codes.shape[1]

    def levels(self) -> np.ndarray:
        return reconstruction_levels(self.mode, self.row_minmax)

    def dequant(self) -> np.ndarray:
        return np.take_along_axis(self.levels(), self.codes.astype(np.intp), axis=1)

    def zero_mask(self) -> np.ndarray:
        return self.codes == 0


def rtn_quantize_device(w, minmax_in=None, stream=None):
    """GPU RTN of a CUDA float32 (rows, cols) tensor -> (codes u8 tensor,
    row_minmax int32 tensor of packed bf16 pairs). minmax_in: optional packed
    grid (int32 tensor); None derives it from the row extrema (make_grid)."""
    import torch

    assert w.is_cuda and w.dtype == torch.float32 and w.dim() == 2
    w = w.contiguous()
    rows, cols = w.shape
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=w.device)
    mm = torch.empty(rows, dtype=torch.int32, device=w.device)
    _lib.check(_lib.lib.qmoe_rtn_quantize(_lib.ptr(w), rows, cols, _lib.ptr(minmax_in), _lib.ptr(codes),
                                          _lib.ptr(mm), _lib.stream_ptr(stream)))
    return codes, mm


def rtn_quantize(w: np.ndarray, grid: QuantGrid) -> TernaryMatrix:
    """Nearest grid level per weight, ties toward the smaller magnitude
    (quantize.py:219-235), computed on the GPU."""
    import torch

    w = np.asarray(w, dtype=np.float32)
    if w.ndim != 2 or w.shape[0] != grid.rows:
        raise ValueError("weights do not match the grid")
    mmb = grid.minmax_bits()
    packed = (mmb[:, 0].astype(np.uint32) | (mmb[:, 1].astype(np.uint32) << np.uint32(16))).view(np.int32)
    wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    mmd = torch.from_numpy(packed.copy()).cuda()
    codes, _ = rtn_quantize_device(wd, mmd)
    return TernaryMatrix(codes=codes.cpu().numpy(), row_minmax=mmb.astype(np.uint16))
