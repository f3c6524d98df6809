"""Compressed format + the drop-in codec entry points (moepack/codec.py).

Reference surface kept: `CompressedMatrix`, `encode`, `decompress`,
`fused_matvec`, `pad_to_even`, `simulate_warp_row`, `WarpTrace`,
`SymbolTrace`, `write_checkpoint`, `read_checkpoint` — same argument meaning,
check order and exceptions (CorruptionError, DictionaryMismatchError,
ValueError). Every compute step runs in libqmoe on the GPU; numpy inputs are
copied to the device and results copied back, CUDA tensors are used in place.

The device-resident form is `DeviceMatrix` (uploaded + row-validated once);
the MoE layer and the benchmarks work on it directly.
"""

from __future__ import annotations

import struct
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dictionary import DICT_SIZE, Dictionary
from .errors import CorruptionError, DictionaryMismatchError
from .quantize import TernaryMatrix

CHECKPOINT_MAGIC = b"QMOE0001"
INT32_MAX = 2**31 - 1


def _torch():
    import torch

    return torch


@dataclass
class CompressedMatrix:
    """Host form (codec.py:33-60): uint16 codewords, int32 row_off (rows+1),
    uint16 (rows, 2) bf16 (min, max), dictionary hash. Treated as immutable
    after construction; the device copy is cached on it."""

    rows: int
    cols: int
    codewords: np.ndarray
    row_off: np.ndarray
    row_minmax: np.ndarray
    dict_hash: int
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def validate(self) -> None:
        if self.rows < 0 or self.cols < 0 or self.cols % 2 != 0:
            raise CorruptionError("invalid compressed matrix shape")
        if self.row_off.shape != (self.rows + 1,) or self.row_off.dtype != np.int32:
            raise CorruptionError("row_off must be (rows + 1,) int32")
        if self.rows and self.row_minmax.shape != (self.rows, 2):
            raise CorruptionError("row_minmax must be (rows, 2)")
        if self.row_off[0] != 0 or self.row_off[-1] != len(self.codewords):
            raise CorruptionError("row_off does not span the codeword stream")
        if np.any(np.diff(self.row_off) < 0):
            raise CorruptionError("row_off must be monotone")

    def _key(self):
        arrs = (self.codewords, self.row_off, self.row_minmax)
        return (self.rows, self.cols, self.dict_hash) + tuple((id(a), a.ctypes.data, a.shape) for a in arrs)

    def to_device(self, dic: Dictionary, device=None) -> "DeviceMatrix":
        """Upload (once) and validate every row's decoded length on the GPU."""
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        hit = self._device.get(dev.index)
        if hit is not None and hit[0] == self._key():
            return hit[1]
        dm = DeviceMatrix.from_host(self, dic, dev)
        dm.shared = True  # cached for the drop-in API: layers re-index private copies
        self._device[dev.index] = (self._key(), dm)
        return dm


class DeviceMatrix:
    """One compressed matrix resident in HBM: cw int16 (uint16 bits), row_off
    int32, row_minmax int32 (packed bf16 pair, low = min). `bad_rows` is the
    device row-length validation result (0 for a usable matrix)."""

    def __init__(self, rows, cols, cw, row_off, row_minmax, dict_hash, bad_rows=0, first_bad=None):
        self.rows, self.cols = int(rows), int(cols)
        self.cw, self.row_off, self.row_minmax = cw, row_off, row_minmax
        self.dict_hash = int(dict_hash)
        self.bad_rows = int(bad_rows)
        self.first_bad = first_bad
        # None: stream indexed in dictionary order; else a frequency codebook
        # (codebook.Codebook) whose packed table the stream is indexed in
        self.codebook = None
        # row-segment checkpoints (G = 2^lg lanes per row), see build_checkpoints
        self.ck = None
        self.lg = 0
        # True when cached on a CompressedMatrix (shared with the drop-in API)
        self.shared = False

    @property
    def n_codewords(self) -> int:
        return int(self.cw.numel())

    @property
    def compressed_bytes(self) -> int:
        """payload + metadata bytes (stats.compression_rate, stats.py:103-114)."""
        return 2 * self.n_codewords + 4 * (self.rows + 1) + 4 * self.rows

    @classmethod
    def from_host(cls, c: CompressedMatrix, dic: Dictionary, device) -> "DeviceMatrix":
        torch = _torch()
        cw = torch.from_numpy(np.ascontiguousarray(c.codewords, np.uint16).view(np.int16)).to(device)
        ro = torch.from_numpy(np.ascontiguousarray(c.row_off, np.int32)).to(device)
        mm = np.ascontiguousarray(c.row_minmax, np.uint16).reshape(-1, 2) if c.rows else np.zeros((0, 2), np.uint16)
        mmd = torch.from_numpy(mm.copy().view(np.int32).reshape(-1)).to(device)
        dm = cls(c.rows, c.cols, _lib.padded_copy(cw), _lib.padded_copy(ro), _lib.padded_copy(mmd), c.dict_hash)
        dm.validate_rows(dic)
        return dm

    def validate_rows(self, dic: Dictionary) -> int:
        torch = _torch()
        bad = torch.tensor([0, INT32_MAX], dtype=torch.int32, device=self.cw.device)
        h = dic.device_handle(self.cw.device.index)
        _lib.check(_lib.lib.qmoe_validate_rows(h, _lib.ptr(self.cw), _lib.ptr(self.row_off), self.rows, self.cols,
                                               _lib.ptr(bad), _lib.stream_ptr()))
        b = bad.cpu().tolist()
        self.bad_rows, self.first_bad = b[0], (b[1] if b[0] else None)
        return self.bad_rows

    def private_copy(self) -> "DeviceMatrix":
        """Same matrix with its own codeword stream (row offsets, levels and
        kernel-private checkpoints are shared, read-only): what a layer
        re-indexes with its codebook when this matrix is shared."""
        dm = DeviceMatrix(self.rows, self.cols, _lib.padded_copy(self.cw), self.row_off, self.row_minmax,
                          self.dict_hash, self.bad_rows, self.first_bad)
        dm.ck, dm.lg = self.ck, self.lg
        return dm

    def descriptor(self) -> tuple:
        """qmoe_matrix fields (include/qmoe.h)."""
        return (self.cw.data_ptr(), self.row_off.data_ptr(), self.row_minmax.data_ptr(),
                self.ck.data_ptr() if self.ck is not None else 0, self.rows, self.cols, self.n_codewords, self.lg, 0, 0)

    def mean_codewords_per_row(self) -> float:
        return self.n_codewords / max(1, self.rows)

    def build_checkpoints(self, dic: Dictionary, lg: int | None = None) -> None:
        """Kernel-private row-segment checkpoints (qmoe_checkpoints): the column
        at which each of the G = 2^lg segments of every row starts, so G lanes
        walk one row independently. lg=None picks <= ~48 codewords per segment."""
        torch = _torch()
        if lg is None:  # G = 2^lg lanes per row, ~24-48 codewords per lane segment
            avg = self.mean_codewords_per_row()
            lg = 0
            while lg < 3 and avg / (1 << lg) > 48:
                lg += 1
        self.lg = int(lg)
        if self.lg == 0 or self.rows == 0:
            self.ck = None
            return
        G = 1 << self.lg
        self.ck = _lib.padded_empty(self.rows * (G - 1), torch.int16, self.cw.device)
        bad = torch.tensor([0, INT32_MAX], dtype=torch.int32, device=self.cw.device)
        table = self.codebook.table if self.codebook is not None else None
        _lib.check(_lib.lib.qmoe_checkpoints(dic.device_handle(self.cw.device.index), _lib.ptr(table),
                                             _lib.ptr(self.cw), _lib.ptr(self.row_off), self.rows, self.cols,
                                             self.lg, _lib.ptr(self.ck), _lib.ptr(bad), _lib.stream_ptr()))
        if int(bad[0].item()):
            raise CorruptionError("row decodes to the wrong number of values")


def _row_len_error():
    return CorruptionError("row decodes to the wrong number of values")


# ------------------------------------------------------------------ encode
def encode_device(codes, row_minmax, dic: Dictionary, stream=None) -> DeviceMatrix:
    """GPU encode of a CUDA uint8 (rows, cols) code tensor (codec.py:126-155):
    count pass, exclusive scan, emit pass. row_minmax: int32 packed tensor."""
    torch = _torch()
    rows, cols = codes.shape
    if cols % 2 != 0:
        raise ValueError("column count must be even; pad_to_even() first")
    codes = codes.contiguous()
    dev = codes.device
    h = dic.device_handle(dev.index)
    sp = _lib.stream_ptr(stream)
    counts = torch.empty(rows, dtype=torch.int32, device=dev)
    row_off = _lib.padded_empty(rows + 1, torch.int32, dev)
    _lib.check(_lib.lib.qmoe_encode_count(h, _lib.ptr(codes), rows, cols, _lib.ptr(counts), sp))
    _lib.check(_lib.lib.qmoe_exclusive_scan(_lib.ptr(counts), rows, _lib.ptr(row_off), sp))
    total = int(row_off[-1].item())
    if total < 0:
        raise ValueError("codeword stream exceeds 32-bit row offsets")
    cw = _lib.padded_empty(total, torch.int16, dev)
    _lib.check(_lib.lib.qmoe_encode_emit(h, _lib.ptr(codes), rows, cols, _lib.ptr(row_off), _lib.ptr(cw), sp))
    return DeviceMatrix(rows, cols, cw, row_off, _lib.padded_copy(row_minmax.contiguous()), dic.hash64)


def encode(t: TernaryMatrix, dic: Dictionary, workers: int = 1) -> CompressedMatrix:
    """Greedy longest-prefix encode (codec.py:126-155) on the GPU, one thread
    per row. `workers` is accepted for API parity (output is invariant)."""
    torch = _torch()
    if t.cols % 2 != 0:
        raise ValueError("column count must be even; pad_to_even() first")
    rows, cols = t.rows, t.cols
    if rows == 0 or cols == 0:
        return CompressedMatrix(rows, cols, np.zeros(0, np.uint16), np.zeros(rows + 1, np.int32),
                                t.row_minmax.copy(), dic.hash64)
    codes = torch.from_numpy(np.ascontiguousarray(t.codes)).cuda()
    mm = torch.zeros(rows, dtype=torch.int32, device=codes.device)
    dm = encode_device(codes, mm, dic)
    return CompressedMatrix(
        rows=rows,
        cols=cols,
        codewords=dm.cw.cpu().numpy().view(np.uint16).copy(),
        row_off=dm.row_off.cpu().numpy().astype(np.int32),
        row_minmax=t.row_minmax.copy(),
        dict_hash=dic.hash64,
    )


# ------------------------------------------------------------------ decompress
def _prepare(c, dic: Dictionary) -> DeviceMatrix:
    if isinstance(c, DeviceMatrix):
        dm = c
    else:
        c.validate()
    if c.dict_hash != dic.hash64:
        raise DictionaryMismatchError("checkpoint was encoded against a different dictionary")
    if not isinstance(c, DeviceMatrix):
        dm = c.to_device(dic)
    return dm


def decompress_device(dm: DeviceMatrix, dic: Dictionary, stream=None):
    torch = _torch()
    out = torch.empty((dm.rows, dm.cols), dtype=torch.uint8, device=dm.cw.device)
    bad = torch.tensor([0, INT32_MAX], dtype=torch.int32, device=dm.cw.device)
    h = dic.device_handle(dm.cw.device.index)
    table = dm.codebook.table if dm.codebook is not None else None
    _lib.check(_lib.lib.qmoe_decompress(h, _lib.ptr(table), _lib.ptr(dm.cw), _lib.ptr(dm.row_off), dm.rows, dm.cols,
                                        _lib.ptr(out),
                                        _lib.ptr(bad), _lib.stream_ptr(stream)))
    return out, bad


def decompress(c, dic: Dictionary, workers: int = 1) -> TernaryMatrix:
    """Exact expansion back to ternary codes (codec.py:175-193)."""
    dm = _prepare(c, dic)
    if dm.rows == 0 or dm.cols == 0:
        mm = c.row_minmax.copy() if isinstance(c, CompressedMatrix) else np.zeros((dm.rows, 2), np.uint16)
        return TernaryMatrix(codes=np.zeros((dm.rows, dm.cols), np.uint8), row_minmax=mm.reshape(dm.rows, 2))
    if dm.bad_rows:
        raise _row_len_error()
    out, bad = decompress_device(dm, dic)
    if int(bad[0].item()):
        raise _row_len_error()
    codes = out.cpu().numpy()
    if isinstance(c, CompressedMatrix):
        mm = c.row_minmax.copy()
    else:
        mm = dm.row_minmax.cpu().numpy().view(np.uint16).reshape(dm.rows, 2).copy()
    return TernaryMatrix(codes=codes, row_minmax=mm)


# ------------------------------------------------------------------ fused matvec
def _x_dtype_code(x) -> int:
    torch = _torch()
    return _lib.QMOE_X_BF16 if x.dtype == torch.bfloat16 else _lib.QMOE_X_F32


def fused_matvec_device(dm: DeviceMatrix, dic: Dictionary, x, y, stream=None, bad=None, staged=False) -> None:
    """y (CUDA f32, rows) += bf16(M @ x) for x a CUDA f32/bf16 (cols,) tensor,
    or x (ntok, cols) / y (ntok, rows) for an inner token loop. staged: x
    already satisfies the staging contract (see _staging_x)."""
    if dm.codebook is not None:
        raise ValueError("matrix is re-indexed by a layer codebook; use the grouped/MoE path")
    h = dic.device_handle(dm.cw.device.index)
    sp = _lib.stream_ptr(stream)
    xt = _lib.QMOE_X_BF16 if _x_dtype_code(x) == _lib.QMOE_X_BF16 else _lib.QMOE_X_F32
    if not staged:
        x = _staging_x(x)
    if x.dim() == 1:
        runs = _api_run(dm, dic) if _sparse_path(dic, dm.cw.device.index) else None
        if runs is not None:  # one matrix spread over ~6K lanes (row checkpoints), one grouped launch
            raw, n = runs
            ldx = ((dm.cols + 7) // 8) * 8 if xt == _lib.QMOE_X_BF16 else ((dm.cols + 3) // 4) * 4
            _lib.check(_lib.lib.qmoe_grouped_matvec(h, None, _lib.ptr(raw), _lib.ptr(n), 1, dm.cols, 1, _lib.ptr(x),
                                                    xt, ldx, _lib.ptr(y), _lib.QMOE_Y_ACCUM_F32, dm.rows,
                                                    API_HOT_ENTRIES, _lib.ptr(bad), sp))
        else:
            _lib.check(_lib.lib.qmoe_fused_matvec(h, _lib.ptr(dm.cw), _lib.ptr(dm.row_off),
                                                  _lib.ptr(dm.row_minmax), dm.rows, dm.cols, _lib.ptr(x), xt,
                                                  _lib.ptr(y), _lib.ptr(bad), sp))
    else:
        _lib.check(_lib.lib.qmoe_fused_matmat(h, _lib.ptr(dm.cw), _lib.ptr(dm.row_off), _lib.ptr(dm.row_minmax),
                                              dm.rows, dm.cols, _lib.ptr(x), xt, x.shape[0], x.stride(0),
                                              _lib.ptr(y), y.stride(0), _lib.ptr(bad), sp))


def _sparse_path(dic: Dictionary, device: int) -> bool:
    """The dictionary has <= 3 non-zeros per entry (streaming kernels apply);
    asked of the library once per (dictionary, device)."""
    cache = dic.__dict__.setdefault("_sparse_cache", {})
    hit = cache.get(device)
    if hit is None:
        hit = cache[device] = bool(dic.device_info(device)["sparse_path"])
    return hit


_MV_LOCAL = threading.local()  # per thread: (device, rows, cols) -> staging of the host fused_matvec call


def _mv_stage(device, rows: int, cols: int) -> dict:
    """One pinned host buffer [x f32, padded | y f32] and its device twin
    (16-byte aligned, readable past the end): the host call is one H2D copy,
    the launch, one D2H copy."""
    torch = _torch()
    stages = _MV_LOCAL.__dict__.setdefault("stages", {})
    key = (device.index, rows, cols)
    st = stages.get(key)
    if st is None:
        xw = ((cols + 3) // 4) * 4
        n = xw + rows
        h = torch.empty(n, dtype=torch.float32, pin_memory=True)
        d = _lib.padded_empty(n, torch.float32, device)
        st = stages[key] = {"h": h, "d": d, "xh": h[:cols].numpy(), "yh": h[xw:].numpy(),
                            "xd": d[:cols], "yd": d[xw:],
                            "yout": torch.empty(rows, dtype=torch.float32, pin_memory=True),
                            "graphs": weakref.WeakKeyDictionary()}
    return st


API_LANES = 12288  # lanes one API matvec is spread over (~384 warps)
API_HOT_ENTRIES = 1024  # table entries each CTA stages for it (the fill is per CTA per launch)
# (measured, tools/debug/api_matvec.py: 768x3072 8.9 -> 8.8 us, 3072x768 9.1 -> 8.6 us
# against 6144 lanes / 4096 entries / >= 1.5 groups per lane)


def _api_run(dm: DeviceMatrix, dic: Dictionary):
    """Work record (one run) + row checkpoints that let a single matrix use
    ~API_LANES lanes: G = 2^lg lanes per row while each keeps >= ~1 group
    of 8 codewords. Built once per uploaded matrix; None when one lane per row
    already fills the lanes (then qmoe_fused_matvec is used)."""
    hit = getattr(dm, "_api_runs", None)
    if hit is not None:
        return hit or None
    torch = _torch()
    mg = dm.n_codewords / max(1, dm.rows) / 8
    lg = 0
    while lg < 3 and dm.rows * (1 << lg) < API_LANES and mg / (1 << (lg + 1)) >= 1.0:
        lg += 1
    if lg == 0 or dm.rows == 0:
        dm._api_runs = ()
        return None
    if dm.ck is None or dm.lg < lg:
        dm.build_checkpoints(dic, lg)
    tasks = ((dm.rows << lg) + 31) >> 5
    rec = _lib.QmoeWork(dm.cw.data_ptr(), dm.row_off.data_ptr(), dm.row_minmax.data_ptr(), dm.ck.data_ptr(),
                        dm.cols, 0, dm.rows, lg | (dm.lg << 8), 1, 0, 0, (0, 0, 0, 0))
    raw = torch.from_numpy(np.frombuffer(bytes(rec), dtype=np.uint8).copy()).to(dm.cw.device)
    n = torch.tensor([1, tasks], dtype=torch.int32, device=dm.cw.device)
    dm._api_runs = (raw, n)
    return dm._api_runs


def _staging_x(x):
    """x rows must start 16-byte aligned with a 16-byte-multiple stride and be
    readable to the next 16-byte boundary (bulk-copy staging): copy into a
    padded buffer unless the tensor already satisfies it."""
    torch = _torch()
    esz = x.element_size()
    if x.dim() == 1:
        x2 = x.reshape(1, -1)
    else:
        x2 = x
    cols = x2.shape[1]
    ld = ((cols * esz + 15) // 16) * 16 // esz
    buf = _lib.padded_empty(x2.shape[0] * ld, x.dtype, x.device).view(x2.shape[0], ld)
    buf[:, :cols].copy_(x2)
    out = buf[:, :cols]
    return out.reshape(-1) if x.dim() == 1 else out


def _dense_semantics(dm: DeviceMatrix, dic: Dictionary, x32):
    """Non-finite x: the reference multiplies the dense
    dequantized row, so 0 * inf = NaN reaches every row. The sparse kernels
    skip zeros, so this case expands the rows on the GPU (qmoe_decompress)
    and runs the dense product there, reproducing the reference's NaN/inf
    propagation. Only taken when x holds inf/NaN."""
    torch = _torch()
    codes, bad = decompress_device(dm, dic)
    mm = dm.row_minmax.view(torch.int16).view(dm.rows, 2)
    lv_min = (mm[:, 0].to(torch.int32) << 16).view(torch.float32)
    lv_max = (mm[:, 1].to(torch.int32) << 16).view(torch.float32)
    w = torch.where(codes == 1, lv_min[:, None], torch.where(codes == 2, lv_max[:, None], torch.zeros((), device=codes.device)))
    part = (w.to(torch.float32) @ x32.to(torch.float32))
    # The reference rounds with no NaN special case (bf16.py:16-17); on its
    # x86 host 0 * inf yields the default NaN 0xFFC00000, which survives the
    # rounding. CUDA's canonical NaN (0x7FFFFFFF) would round to -0.0, so NaNs
    # are first set to the x86 default pattern.
    part = torch.where(torch.isnan(part), torch.tensor(-0x400000, dtype=torch.int32, device=part.device).view(torch.float32), part)
    u = part.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
    return (u << 16).to(torch.int64).to(torch.int32).view(torch.float32)


def fused_matvec(c, x, dic: Dictionary, y=None, workers: int = 1):
    """y += M @ x straight from the compressed stream (codec.py:209-244):
    fp32 products and sums per row, one bf16 RNE rounding, fp32 add into y.
    numpy x/y: copied to the GPU and back, y updated in place and returned.
    CUDA tensors: computed in place on the current stream."""
    torch = _torch()
    if isinstance(c, DeviceMatrix):
        dm_rows, dm_cols = c.rows, c.cols
    else:
        c.validate()
        dm_rows, dm_cols = c.rows, c.cols
    if c.dict_hash != dic.hash64:
        raise DictionaryMismatchError("checkpoint was encoded against a different dictionary")
    on_device = torch.is_tensor(x)
    if on_device:
        if tuple(x.shape) != (dm_cols,):
            raise ValueError(f"x must have shape ({dm_cols},)")
        if y is None:
            y = torch.zeros(dm_rows, dtype=torch.float32, device=x.device)
        elif tuple(y.shape) != (dm_rows,):
            raise ValueError(f"y must have shape ({dm_rows},)")
        xd = x if x.dtype in (torch.float32, torch.bfloat16) else x.float()
        yd = y
    else:
        x32 = np.asarray(x, dtype=np.float32)
        if x32.shape != (dm_cols,):
            raise ValueError(f"x must have shape ({dm_cols},)")
        if y is None:
            y = np.zeros(dm_rows, dtype=np.float32)
        elif y.shape != (dm_rows,):
            raise ValueError(f"y must have shape ({dm_rows},)")
    if dm_rows == 0:
        return y
    dm = c if isinstance(c, DeviceMatrix) else c.to_device(dic)
    if dm.bad_rows:
        raise _row_len_error()  # y untouched (codec.py:237-243 computes all parts first)
    staged = False
    if not on_device:
        # float32 y is updated on the GPU (y += bf16(part) in fp32, as the
        # reference); any other dtype gets the bf16 part back and adds it on
        # the host in its own dtype (codec.py:243: y[rows] += part)
        accum_dev = y.dtype == np.float32
        st = _mv_stage(dm.cw.device, dm_rows, dm_cols)
        np.copyto(st["xh"], x32)
        if accum_dev:
            np.copyto(st["yh"], y)
        else:
            st["yh"].fill(0.0)
        finite = bool(np.isfinite(x32).all())
        if finite and dm_cols > 0 and torch.cuda.current_device() == dm.cw.device.index:
            # H2D copy + kernel + D2H copy, captured once per (staging, matrix)
            # and replayed: the call is then one graph launch and one sync. The
            # graph lives in the (per-thread) staging that owns its buffers,
            # keyed weakly by the matrix whose buffers it reads.
            g = st["graphs"].get(dm)
            if g is None:
                def body():
                    st["d"].copy_(st["h"], non_blocking=True)
                    fused_matvec_device(dm, dic, st["xd"], st["yd"], staged=True)
                    st["yout"].copy_(st["yd"], non_blocking=True)
                body()  # first call eager (builds the run record / checkpoints)
                torch.cuda.current_stream().synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    body()
                st["graphs"][dm] = g
                # the eager call consumed the staged y
                if accum_dev:
                    np.copyto(st["yh"], y)
                else:
                    st["yh"].fill(0.0)
            g.replay()
            torch.cuda.current_stream().synchronize()
            _mv_out(y, st["yout"].numpy(), accum_dev)
            return y
        st["d"].copy_(st["h"], non_blocking=True)
        xd, yd, staged = st["xd"], st["yd"], True
    else:
        finite = bool(torch.isfinite(xd).all().item())
    if dm_cols == 0:
        pass
    elif finite:
        fused_matvec_device(dm, dic, xd, yd, staged=staged)
    else:
        yd += _dense_semantics(dm, dic, xd)
    if on_device:
        return y
    st["yout"].copy_(yd, non_blocking=True)
    torch.cuda.current_stream(dm.cw.device).synchronize()
    _mv_out(y, st["yout"].numpy(), accum_dev)
    return y


def _mv_out(y: np.ndarray, out: np.ndarray, accum_dev: bool) -> None:
    if accum_dev:
        y[...] = out
    else:
        y += out  # out = bf16-rounded part (f32), added in y's dtype


def paper_matvec_device(dm: DeviceMatrix, dic: Dictionary, x, y, trace=None, stream=None) -> None:
    """The paper's Listing-1 kernel (baseline design) on the GPU."""
    h = dic.device_handle(dm.cw.device.index)
    _lib.check(_lib.lib.qmoe_paper_matvec(h, _lib.ptr(dm.cw), _lib.ptr(dm.row_off), _lib.ptr(dm.row_minmax), dm.rows,
                                          dm.cols, _lib.ptr(x), _x_dtype_code(x), _lib.ptr(y), _lib.ptr(trace),
                                          _lib.stream_ptr(stream)))


def pad_to_even(t: TernaryMatrix) -> TernaryMatrix:
    """Append one zero column to odd-width matrices (codec.py:247-258)."""
    if t.cols % 2 == 0:
        return t
    codes = np.concatenate([t.codes, np.zeros((t.rows, 1), dtype=np.uint8)], axis=1)
    return TernaryMatrix(codes=codes, row_minmax=t.row_minmax.copy())


# ------------------------------------------------------------------ lane replay
@dataclass
class SymbolTrace:
    codeword: int
    pair_count: int
    offset: int
    lane_values: np.ndarray
    extracting_lanes: int


@dataclass
class WarpTrace:
    """Lane replay of one row through the Listing-1 schedule (codec.py:261-290)."""

    row: int
    fetch_sizes: list = field(default_factory=list)
    symbols: list = field(default_factory=list)
    lane_word: np.ndarray = field(default_factory=lambda: np.where(np.arange(32) < 28, np.arange(32) // 14, -1))
    lane_slot: np.ndarray = field(default_factory=lambda: np.where(np.arange(32) < 28, np.arange(32) % 14, -1))
    extract_counts: np.ndarray = field(default_factory=lambda: np.zeros(32, np.int64))

    def extracted_values(self) -> np.ndarray:
        parts = [s.lane_values[: s.extracting_lanes] for s in self.symbols]
        return np.concatenate(parts) if parts else np.zeros(0, np.uint8)


def simulate_warp_row(c: CompressedMatrix, row: int, dic: Dictionary) -> WarpTrace:
    """Replay row `row` through the paper kernel (codec.py:293-338). The lane
    records come from the GPU Listing-1 kernel's trace buffer; the replayed
    values must equal decompress for that row."""
    torch = _torch()
    c.validate()
    if not (0 <= row < c.rows):
        raise ValueError("row out of range")
    s, e = int(c.row_off[row]), int(c.row_off[row + 1])
    # replay just this row: a one-row matrix view of the stream
    sub = CompressedMatrix(1, c.cols, np.ascontiguousarray(c.codewords[s:e]), np.array([0, e - s], np.int32),
                           np.ascontiguousarray(c.row_minmax[row : row + 1]), dic.hash64)
    dm = DeviceMatrix.from_host(sub, dic, torch.device("cuda", torch.cuda.current_device()))
    trace = torch.zeros(max(1, e - s) * 5, dtype=torch.int32, device=dm.cw.device)
    x = torch.zeros(c.cols, dtype=torch.float32, device=dm.cw.device)
    y = torch.zeros(1, dtype=torch.float32, device=dm.cw.device)
    if e > s:
        paper_matvec_device(dm, dic, x, y, trace=trace)
    rec = trace.cpu().numpy().reshape(-1, 5)[: e - s]
    tr = WarpTrace(row=row)
    tr.fetch_sizes = [int(min(32, (e - s) - b)) for b in range(0, e - s, 32)]
    lanes = np.arange(28)
    for cw_, n, off, v0, v1 in rec.tolist():
        words = (np.uint32(v0 & 0xFFFFFFFF), np.uint32(v1 & 0xFFFFFFFF))
        lane_vals = np.array([(int(words[l // 14]) >> (2 * (l % 14))) & 3 for l in lanes], np.uint8)
        tr.symbols.append(SymbolTrace(codeword=int(cw_), pair_count=int(n), offset=int(off), lane_values=lane_vals,
                                      extracting_lanes=2 * int(n)))
        tr.extract_counts[: 2 * int(n)] += 1
    total = sum(2 * s_.pair_count for s_ in tr.symbols)
    if total != c.cols:
        raise CorruptionError("row decodes to the wrong number of values")
    direct = decompress(sub, dic).codes[0]
    if not np.array_equal(tr.extracted_values(), direct):
        raise CorruptionError("lane replay disagrees with decompress")
    return tr


# ------------------------------------------------------------------ container
def write_checkpoint(c: CompressedMatrix, path: str) -> None:
    """QMOE0001: magic, <QQQ rows/cols/dict_hash, <i4 row_off, <u2 row_minmax,
    <u2 codewords; no padding (codec.py:341-351)."""
    c.validate()
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(struct.pack("<QQQ", c.rows, c.cols, c.dict_hash))
        fh.write(c.row_off.astype("<i4").tobytes())
        fh.write(c.row_minmax.astype("<u2").tobytes())
        fh.write(c.codewords.astype("<u2").tobytes())


def _parse_checkpoint(blob: np.ndarray):
    """Strict QMOE0001 parse (codec.py:354-391) over a uint8 buffer, same
    checks, order and messages as the reference; returns views into blob."""
    if len(blob) < len(CHECKPOINT_MAGIC) + 24 or bytes(blob[: len(CHECKPOINT_MAGIC)]) != CHECKPOINT_MAGIC:
        raise CorruptionError("not a checkpoint file (bad magic)")
    pos = len(CHECKPOINT_MAGIC)
    rows, cols, dict_hash = struct.unpack_from("<QQQ", blob, pos)
    pos += 24
    if len(blob) < pos + 4 * (rows + 1) + 4 * rows:
        raise CorruptionError("checkpoint truncated in header arrays")
    row_off = np.frombuffer(blob, dtype="<i4", count=rows + 1, offset=pos)
    off_pos = pos
    pos += 4 * (rows + 1)
    row_minmax = np.frombuffer(blob, dtype="<u2", count=2 * rows, offset=pos).reshape(rows, 2)
    mm_pos = pos
    pos += 4 * rows
    if row_off[0] != 0 or np.any(np.diff(row_off) < 0):
        raise CorruptionError("checkpoint row offsets are not monotone from zero")
    n = int(row_off[-1])
    if len(blob) != pos + 2 * n:
        raise CorruptionError("checkpoint size disagrees with row offsets")
    cw = np.frombuffer(blob, dtype="<u2", count=n, offset=pos)
    return int(rows), int(cols), int(dict_hash), row_off, row_minmax, cw, (off_pos, mm_pos, pos)


def read_checkpoint(path: str) -> CompressedMatrix:
    """Strict reader (codec.py:354-391): magic, header arrays, monotone
    offsets from zero, exact total size, then validate()."""
    with open(path, "rb") as fh:
        blob = np.frombuffer(fh.read(), dtype=np.uint8)
    rows, cols, dict_hash, row_off, row_minmax, cw, _ = _parse_checkpoint(blob)
    c = CompressedMatrix(rows, cols, cw.astype(np.uint16), row_off.astype(np.int32),
                         row_minmax.astype(np.uint16), dict_hash)
    c.validate()
    return c


def _read_pinned(path: str):
    """The whole file in pinned host memory (torch uint8) + a numpy view."""
    import os

    torch = _torch()
    size = os.path.getsize(path)
    buf = torch.empty(max(1, size), dtype=torch.uint8, pin_memory=True)
    view = buf.numpy()[:size]
    with open(path, "rb") as fh:
        got = fh.readinto(memoryview(view))
    if got != size:
        raise CorruptionError("checkpoint changed while reading")
    return buf, view


def _validate_many(mats, dic: Dictionary) -> None:
    """Device row-length validation of several matrices, one sync."""
    torch = _torch()
    if not mats:
        return
    dev = mats[0].cw.device
    bad = torch.tensor([0, INT32_MAX] * len(mats), dtype=torch.int32, device=dev)
    h = dic.device_handle(dev.index)
    for i, m in enumerate(mats):
        _lib.check(_lib.lib.qmoe_validate_rows(h, _lib.ptr(m.cw), _lib.ptr(m.row_off), m.rows, m.cols,
                                               bad.data_ptr() + 8 * i, _lib.stream_ptr()))
    b = bad.view(-1, 2).cpu().numpy()
    for m, (n, first) in zip(mats, b):
        m.bad_rows, m.first_bad = int(n), (int(first) if n else None)


def _load_device(path: str, dic: Dictionary, device, rows_per_part=None):
    """Pinned read + strict parse + hash check + ONE host-to-device copy of
    the file; the matrix (or its row blocks of rows_per_part rows, stacked
    by rows as the reference CLI writes them) as aligned DeviceMatrix
    arrays carved out of the device copy, then validated on the GPU."""
    torch = _torch()
    buf, blob = _read_pinned(path)
    rows, cols, dict_hash, row_off, _, _, (off_pos, mm_pos, cw_pos) = _parse_checkpoint(blob)
    if cols % 2 != 0:
        raise CorruptionError("invalid compressed matrix shape")
    if dict_hash != dic.hash64:
        raise DictionaryMismatchError("checkpoint was encoded against a different dictionary")
    R = rows if rows_per_part is None else int(rows_per_part)
    if rows and (R <= 0 or rows % R != 0):
        raise ValueError(f"{rows} stacked rows are not a multiple of rows_per_expert = {R}")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    blob_d = buf[: len(blob)].to(dev, non_blocking=True)  # the one H2D copy
    ro_all = blob_d[off_pos: off_pos + 4 * (rows + 1)].view(torch.int32)
    mm_all = blob_d[mm_pos: mm_pos + 4 * rows].view(torch.int32)
    cw_all = blob_d[cw_pos:].view(torch.int16)
    parts = []
    for p0 in range(0, rows, R) if rows else [0]:
        p1 = min(rows, p0 + R)
        s, e = int(row_off[p0]), int(row_off[p1])
        parts.append(DeviceMatrix(p1 - p0, cols, _lib.padded_copy(cw_all[s:e]),
                                  _lib.padded_copy(ro_all[p0: p1 + 1] - s), _lib.padded_copy(mm_all[p0:p1]),
                                  dict_hash))
    _validate_many(parts, dic)
    del blob_d
    if any(m.bad_rows for m in parts):
        raise _row_len_error()
    return parts


def read_checkpoint_device(path: str, dic: Dictionary, device=None) -> DeviceMatrix:
    """Loader straight to HBM (format codec.py:341-391): the
    file is read into pinned memory, parsed and checked on the host exactly as
    read_checkpoint (then DictionaryMismatchError), copied to the device in
    one transfer and row-validated on the GPU (CorruptionError)."""
    return _load_device(path, dic, device)[0]


def read_stacked_device(path: str, dic: Dictionary, rows_per_expert: int, device=None) -> list:
    """A stacked multi-expert checkpoint (experts' matrices concatenated by
    rows into one QMOE0001 file, reference cli.py:150-153 / :194-201, with
    rows_per_expert from its report) -> one DeviceMatrix per expert, carved
    from a single host-to-device copy."""
    return _load_device(path, dic, device, rows_per_expert)
