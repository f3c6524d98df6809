"""Frequency codebook: kernel-private re-indexing of a layer's codeword streams.

The streaming matvec stages the first H entries of the packed entry table in
shared memory (~40K of 65,536 fit beside the pipeline buffers); the rest is
read through L1/L2, which is ~10x more expensive per lookup. In dictionary
order the staged prefix covers only ~74-80% of a random-init layer's
codewords; ranking codewords by their frequency in the layer raises that to
~95% at the same H (measured: DESIGN.md "codebook").

A Codebook maps codeword c -> rank r (a permutation of 0..65535), rewrites the
device streams to ranks (same uint16 size, so the compressed byte count is
unchanged) and holds the packed entry table in rank order. Decode stays
bit-exact: entry(r) = dictionary entry(c). The on-disk / host format is never
touched; this is a device-resident layout decision like an offset checkpoint.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .dictionary import DICT_SIZE, Dictionary

MT_STRIDE = 65540  # entries per table variant (csrc/qmoe_internal.h)


class Codebook:
    def __init__(self, dic: Dictionary, mats, device=None):
        import torch

        if not mats:
            raise ValueError("need at least one matrix")
        dev = mats[0].cw.device if device is None else device
        h = dic.device_handle(dev.index)
        if not dic.device_info(dev.index)["sparse_path"]:
            raise ValueError("frequency codebooks need a <= 3-non-zero dictionary")
        counts = torch.zeros(DICT_SIZE, dtype=torch.int32, device=dev)
        sp = _lib.stream_ptr()
        for m in mats:
            if m.codebook is not None:
                raise ValueError("matrix already re-indexed")
            _lib.check(_lib.lib.qmoe_histogram(_lib.ptr(m.cw), m.n_codewords, _lib.ptr(counts), sp))
        c = counts.cpu().numpy().view(np.uint32).astype(np.int64)
        # rank -> codeword by descending frequency, with dictionary entry 0 (one
        # zero pair, no non-zero value) pinned to rank 0: the streaming kernel
        # decodes the masked codewords of a partial group as rank 0
        c0 = c.copy()
        c0[0] = np.iinfo(np.int64).max
        self.order = np.argsort(-c0, kind="stable").astype(np.uint16)
        self.rank_of = np.empty(DICT_SIZE, np.uint16)
        self.rank_of[self.order] = np.arange(DICT_SIZE, dtype=np.uint16)
        self.counts = c
        self.table = torch.empty(2 * MT_STRIDE, dtype=torch.int32, device=dev)
        _lib.check(_lib.lib.qmoe_codebook_table(h, _lib.ptr(self.order), _lib.ptr(self.table)))
        self._rank_dev = torch.from_numpy(self.rank_of.view(np.int16).copy()).to(dev)

    def hit_rate(self, entries: int) -> float:
        """Fraction of the layer's codewords inside the first `entries` ranks."""
        s = np.sort(self.counts)[::-1]
        return float(s[:entries].sum() / max(1, s.sum()))

    def apply(self, mats) -> None:
        """Rewrite each DeviceMatrix stream in place to ranks."""
        sp = _lib.stream_ptr()
        for m in mats:
            if m.codebook is not None:
                raise ValueError("matrix already re-indexed")
            _lib.check(_lib.lib.qmoe_remap(_lib.ptr(m.cw), m.n_codewords, _lib.ptr(self._rank_dev),
                                           _lib.ptr(m.cw), sp))
            m.codebook = self
