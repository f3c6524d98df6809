"""Synthetic random-init compressed MoE layers, built on the GPU.

Recipe: W ~ N(0, 0.02^2) fp32 per expert matrix, make_grid +
RTN to ternary (GPU rtn_kernel, bit-exact with quantize.rtn_quantize), then the
GPU encoder (bit-exact with codec.encode). Two weight sources:
  build_layer         device-generated weights (torch.randn): fast, for the
                      pools of distinct layers the benchmarks rotate through;
  build_layer_seeded  the survey's host recipe, W = N(0, 0.02^2) drawn from
                      numpy default_rng(SeedSequence([base, layer, e, m]))
                      (m = 0 wi, 1 wo) — what the reference CPU path can
                      regenerate bit for bit (bench.py's reference arm and
                      parity leg).
All experts of one kind (wi or wo) are encoded as ONE stacked matrix — rows
are independent, so the stream of each expert is exactly what encoding it
alone gives — then split into per-expert DeviceMatrix views.
"""

from __future__ import annotations

from . import _lib
from .codec import DeviceMatrix, encode_device
from .dictionary import Dictionary
from .moe import CompressedMoELayer
from .quantize import rtn_quantize_device


def _stacked(E: int, rows: int, cols: int, seed: int, dic: Dictionary, device, chunk_rows: int = 1 << 17):
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    mats: list[DeviceMatrix] = []
    per = max(1, chunk_rows // rows)
    for e0 in range(0, E, per):
        ne = min(per, E - e0)
        w = torch.randn((ne * rows, cols), device=device, generator=g, dtype=torch.float32) * 0.02
        codes, mm = rtn_quantize_device(w)
        del w
        big = encode_device(codes, mm, dic)
        del codes
        ro = big.row_off
        starts = ro[:: rows].tolist()  # row_off at every expert boundary (ne + 1 values)
        for k in range(ne):
            a, b = starts[k], starts[k + 1]
            cw = _lib.padded_copy(big.cw[a:b])
            r = _lib.padded_copy(ro[k * rows : (k + 1) * rows + 1] - a)
            m = _lib.padded_copy(mm[k * rows : (k + 1) * rows])
            mats.append(DeviceMatrix(rows, cols, cw, r, m, dic.hash64))
        del big, mm
    return mats


def seeded_weights(base: int, layer: int, e: int, m: int, rows: int, cols: int):
    """SURVEY 8(d) recipe: fp32 N(0, 0.02^2) of expert e's matrix m (0 wi, 1 wo)."""
    import numpy as np

    rng = np.random.default_rng(np.random.SeedSequence([base, layer, e, m]))
    return (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)


def build_layer_seeded(E: int, d_model: int, d_ff: int, base: int, layer: int, dic: Dictionary, device=None,
                       max_tokens: int = 64) -> CompressedMoELayer:
    """A layer from the host recipe (seeded_weights), RTN + encoded on the GPU."""
    import torch

    device = device or torch.device("cuda", torch.cuda.current_device())
    mats = ([], [])
    for m, (rows, cols) in enumerate(((d_ff, d_model), (d_model, d_ff))):
        for e in range(E):
            w = torch.from_numpy(seeded_weights(base, layer, e, m, rows, cols)).to(device)
            codes, mm = rtn_quantize_device(w)
            del w
            mats[m].append(encode_device(codes, mm, dic))
    return CompressedMoELayer(mats[0], mats[1], dic, max_tokens=max_tokens)


def build_layer(E: int, d_model: int, d_ff: int, seed: int, dic: Dictionary, device=None,
                max_tokens: int = 64) -> CompressedMoELayer:
    import torch

    device = device or torch.device("cuda", torch.cuda.current_device())
    wi = _stacked(E, d_ff, d_model, 2 * seed + 1, dic, device)
    wo = _stacked(E, d_model, d_ff, 2 * seed + 2, dic, device)
    return CompressedMoELayer(wi, wo, dic, max_tokens=max_tokens)


WORKLOADS = {
    # name: (experts, d_model, d_ff)  — BASELINE.json configs
    "switch-base-128": (128, 768, 3072),
    "switch-large-128": (128, 1024, 4096),
    "switch-c2048": (2048, 2080, 6144),
}
