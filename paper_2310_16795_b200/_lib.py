"""ctypes binding of libqmoe.so (the C-ABI declared in include/qmoe.h).

There is deliberately no fallback: if the shared library is missing the
import of this module raises, and every compute entry point of the package
goes through here. PyTorch is used only to own device memory and streams
(tensors are passed as raw pointers).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QMOE_LIB_PATH") or os.path.join(_HERE, "_lib", "libqmoe.so")  # override: experiments

QMOE_OK, QMOE_EINVAL, QMOE_ECORRUPT, QMOE_ECUDA, QMOE_EUNSUPPORTED = 0, 1, 2, 3, 4
QMOE_X_F32, QMOE_X_BF16 = 0, 1
QMOE_ROUTE_ARGMAX, QMOE_ROUTE_HASH = 0, 1
DICT_SIZE = 65536
NT_MAX = 4

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libqmoe.so not found at {LIB_PATH}; build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
    )

lib = ctypes.CDLL(LIB_PATH)

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u32p = ctypes.POINTER(ctypes.c_uint32)
vp = ctypes.c_void_p
i64 = ctypes.c_int64
i32 = ctypes.c_int32


class QmoeMatrix(ctypes.Structure):
    _fields_ = [("cw", vp), ("row_off", vp), ("row_minmax", vp), ("ck", vp), ("rows", i32), ("cols", i32),
                ("n_cw", i32), ("lg", i32), ("row_id", vp), ("colpts", vp)]


class QmoeWork(ctypes.Structure):
    _fields_ = [("cw", vp), ("row_off", vp), ("row_minmax", vp), ("ck", vp), ("cols", i32), ("row0", i32),
                ("row1", i32), ("lg", i32), ("ntok", i32), ("task0", i32), ("row_id", vp),
                ("tok", i32 * NT_MAX)]


QMOE_Y_ACCUM_F32, QMOE_Y_RELU_BF16, QMOE_Y_STORE_F32, QMOE_Y_RESID_BF16 = 0, 1, 2, 3


WORK_BYTES = ctypes.sizeof(QmoeWork)
NT_STREAM = 2  # tokens per run on the streaming (sparse-table) path
MATRIX_BYTES = ctypes.sizeof(QmoeMatrix)

_SIGS = {
    "qmoe_version": (ctypes.c_char_p, []),
    "qmoe_last_error": (ctypes.c_char_p, []),
    "qmoe_generate_decode_words": (ctypes.c_int, [ctypes.c_double, vp]),
    "qmoe_build_trie": (ctypes.c_int, [vp, vp, vp]),
    "qmoe_dict_create": (ctypes.c_int, [vp, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(vp)]),
    "qmoe_dict_destroy": (ctypes.c_int, [vp]),
    "qmoe_dict_info": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int)]),
    "qmoe_validate_rows": (ctypes.c_int, [vp, vp, vp, i64, i64, vp, vp]),
    "qmoe_decompress": (ctypes.c_int, [vp, vp, vp, vp, i64, i64, vp, vp, vp]),
    "qmoe_fused_matvec": (ctypes.c_int, [vp, vp, vp, vp, i64, i64, vp, ctypes.c_int, vp, vp, vp]),
    "qmoe_fused_matmat": (ctypes.c_int, [vp, vp, vp, vp, i64, i64, vp, ctypes.c_int, i64, i64, vp, i64, vp, vp]),
    "qmoe_grouped_matvec": (ctypes.c_int, [vp, vp, vp, vp, i32, i32, i32, vp, ctypes.c_int, i64, vp,
                                           ctypes.c_int, i64, i32, vp, vp]),
    "qmoe_histogram": (ctypes.c_int, [vp, i64, vp, vp]),
    "qmoe_codebook_table": (ctypes.c_int, [vp, vp, vp]),
    "qmoe_remap": (ctypes.c_int, [vp, i64, vp, vp, vp]),
    "qmoe_checkpoints": (ctypes.c_int, [vp, vp, vp, vp, i64, i64, ctypes.c_int, vp, vp, vp]),
    "qmoe_paper_matvec": (ctypes.c_int, [vp, vp, vp, vp, i64, i64, vp, ctypes.c_int, vp, vp, vp]),
    "qmoe_encode_count": (ctypes.c_int, [vp, vp, i64, i64, vp, vp]),
    "qmoe_encode_emit": (ctypes.c_int, [vp, vp, i64, i64, vp, vp, vp]),
    "qmoe_exclusive_scan": (ctypes.c_int, [vp, i64, vp, vp]),
    "qmoe_rtn_quantize": (ctypes.c_int, [vp, i64, i64, vp, vp, vp, vp]),
    "qmoe_moe_plan": (ctypes.c_int, [vp, i32, i32, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "qmoe_moe_step": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, i32, i32, i32, i32, i32, vp, ctypes.c_int, i64, vp,
                                     i64, vp, i64, vp, vp, vp, i32, vp]),
    "qmoe_moe_step_gated": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, i32, i32, i32, i32, i32, vp, ctypes.c_int, i64,
                                           vp, i64, vp, i64, vp, vp, vp, i32, vp, vp]),
    "qmoe_moe_step_resid": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, i32, i32, i32, i32, i32, vp, i64, vp, i64,
                                           vp, i64, vp, i32, vp, vp, vp, vp]),
    "qmoe_route_scratch": (i64, [i32, i32, i32]),
    "qmoe_ep_slots": (ctypes.c_int, [vp, i32, i32, i32, i32, vp, vp, vp, vp]),
    "qmoe_ep_combine": (ctypes.c_int, [vp, vp, i32, i32, vp, vp]),
    "qmoe_ep_rows": (ctypes.c_int, [vp, vp, i32, i64, vp, ctypes.c_int, vp]),
    "qmoe_route": (ctypes.c_int, [ctypes.c_int, vp, ctypes.c_int, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]),
    "qmoe_debug_step_trace": (ctypes.c_int, [vp]),
    "qmoe_debug_empty_launch": (ctypes.c_int, [i32, i32, vp]),
    "qmoe_dense_moe_pass": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, vp, i32, i32, vp, ctypes.c_int, i64, vp,
                                           ctypes.c_int, i64, i32, i32, vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


class QmoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libqmoe status {status}: {msg}")
        self.status = status


def last_error() -> str:
    return lib.qmoe_last_error().decode()


def check(status: int) -> None:
    """Map a C-ABI status to the package's exceptions."""
    if status == QMOE_OK:
        return
    from .errors import CorruptionError

    msg = last_error()
    if status == QMOE_ECORRUPT:
        raise CorruptionError(msg)
    if status == QMOE_EINVAL:
        raise ValueError(msg)
    raise QmoeError(status, msg)


def ptr(a) -> int:
    """Raw address of a numpy array or torch tensor (0 for None)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def padded_empty(n: int, dtype, device):
    """Device buffer of n elements whose storage is 16-byte aligned and
    readable at least 32 bytes past element n (the contract of the bulk-copy
    staging and the 32-byte codeword group loads in libqmoe)."""
    import torch

    esz = torch.empty((), dtype=dtype).element_size()
    pad = (64 + esz - 1) // esz  # the streaming kernel reads whole 32-byte groups
    buf = torch.empty(n + pad, dtype=dtype, device=device)
    buf[n:].zero_()  # the over-read tail is defined (its values are never used)
    return buf[:n]


def padded_copy(t):
    """Contiguous padded device copy of tensor t (see padded_empty)."""
    out = padded_empty(t.numel(), t.dtype, t.device).view(t.shape) if t.dim() <= 1 else None
    if out is None:
        flat = padded_empty(t.numel(), t.dtype, t.device)
        flat.copy_(t.reshape(-1))
        return flat.view(t.shape)
    out.copy_(t)
    return out


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def version() -> str:
    return lib.qmoe_version().decode()
