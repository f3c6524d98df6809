"""CPU ORACLE for the QMoE compressed decode + matvec path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference package `moepack`
(/root/reference/pkg/src/moepack). It exists to CHECK the CUDA path: only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import it. The product package (paper_2310_16795_b200) never imports,
links or executes anything under oracle/.

Parity pinning: every function here is checked against golden vectors that
were produced by running the reference itself (tests/golden/make_golden.py;
tests/test_oracle_golden.py), so the oracle is "pinned", not free-standing.

Each function cites the reference file:line it restates. Paths are relative
to /root/reference/pkg/src/moepack/.
"""

from __future__ import annotations

import hashlib
import heapq
import math
import struct
from concurrent.futures import ThreadPoolExecutor

import numpy as np

DICT_SIZE = 1 << 16  # dictionary.py:32
MAX_PAIRS = 14  # dictionary.py:33


class OracleCorruption(Exception):
    """Stands for moepack.errors.CorruptionError (errors.py:12-15)."""


class OracleMismatch(Exception):
    """Stands for moepack.errors.DictionaryMismatchError (errors.py:18-20)."""


# --------------------------------------------------------------------------- bf16
def f32_to_bf16_bits(x) -> np.ndarray:
    """RNE f32 -> bf16 bit pattern, no NaN special case (bf16.py:11-18)."""
    a = np.asarray(x, dtype=np.float32)
    u = np.atleast_1d(a).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16).reshape(a.shape)


def bf16_bits_to_f32(bits) -> np.ndarray:
    """Exact widening (bf16.py:21-25)."""
    b = np.asarray(bits, dtype=np.uint16)
    return (np.atleast_1d(b).astype(np.uint32) << np.uint32(16)).view(np.float32).reshape(b.shape)


def bf16_round(x) -> np.ndarray:
    """bf16.py:28-30."""
    return bf16_bits_to_f32(f32_to_bf16_bits(x))


# --------------------------------------------------------------------------- dictionary
def generate_decode_words(p0: float) -> np.ndarray:
    """Best-first enumeration of the 2^16 most probable pair sequences
    (dictionary.py:234-279). Heap key (-logp, n_pairs, value bytes) gives
    the tie-break: probability, then shorter, then lexicographic (:247-248).
    Returns the (65536, 2) uint32 packed decode words (:137-147)."""
    if not (1.0 / 3.0 < p0 < 1.0):
        raise ValueError("dictionary generation requires 1/3 < p0 < 1")
    lp0 = math.log(p0)
    lq = math.log((1.0 - p0) / 2.0)
    pairs = [(a, b) for a in range(3) for b in range(3)]
    vals = np.zeros((DICT_SIZE, 28), np.uint8)
    npairs = np.zeros(DICT_SIZE, np.uint8)
    heap = [(-0.0, 0, b"", -1, 0)]
    filled = 0
    while filled < DICT_SIZE:
        nlp, n, seq, parent, z = heapq.heappop(heap)
        me = -1
        if n:
            me = filled
            filled += 1
            npairs[me] = n
            if parent >= 0:
                vals[me, : 2 * n - 2] = vals[parent, : 2 * n - 2]
            vals[me, 2 * n - 2] = seq[-2]
            vals[me, 2 * n - 1] = seq[-1]
        if n >= MAX_PAIRS:
            continue
        for a, b in pairs:
            cz = z + (a == 0) + (b == 0)
            cnz = 2 * (n + 1) - cz
            heapq.heappush(heap, (-(cz * lp0 + cnz * lq), n + 1, seq + bytes((a, b)), me, cz))
    return pack_words(vals, npairs)


def pack_words(vals: np.ndarray, npairs: np.ndarray) -> np.ndarray:
    """dictionary.py:137-147: word w = n | sum_i v[14w+i] << (4+2i)."""
    sh = (4 + 2 * np.arange(14, dtype=np.uint32))[None, :]
    v = vals.astype(np.uint32)
    n = npairs.astype(np.uint32)
    w0 = n + (v[:, :14] << sh).sum(axis=1, dtype=np.uint32)
    w1 = n + (v[:, 14:] << sh).sum(axis=1, dtype=np.uint32)
    return np.stack([w0, w1], axis=1)


def unpack_words(words: np.ndarray):
    """dictionary.py:150-167 (validation included)."""
    w0, w1 = words[:, 0], words[:, 1]
    n = (w0 & 0xF).astype(np.uint8)
    if not np.array_equal(n, (w1 & 0xF).astype(np.uint8)):
        raise OracleCorruption("pair counts differ between decode words")
    if n.min(initial=MAX_PAIRS) < 1 or n.max(initial=1) > MAX_PAIRS:
        raise OracleCorruption("pair count out of range")
    sh = (4 + 2 * np.arange(14, dtype=np.uint32))[None, :]
    vals = np.empty((words.shape[0], 28), np.uint8)
    vals[:, :14] = (w0[:, None] >> sh) & 3
    vals[:, 14:] = (w1[:, None] >> sh) & 3
    return vals, n


def dictionary_hash(p0: float, words: np.ndarray) -> int:
    """dictionary.py:227-231: first 8 LE bytes of SHA-256(<d p0 || LE words)."""
    d = hashlib.sha256(struct.pack("<d", p0) + words.astype("<u4").tobytes()).digest()
    return int.from_bytes(d[:8], "little")


class OracleDictionary:
    """dictionary.py:197-224 with the trie of :170-194."""

    def __init__(self, p0: float, words: np.ndarray | None = None):
        self.p0 = float(p0)
        self.decode_words = generate_decode_words(p0) if words is None else words
        self.values, self.pair_counts = unpack_words(self.decode_words)
        self.hash64 = dictionary_hash(self.p0, self.decode_words)
        self.next_node, self.entry_of_node = self._trie()

    def _trie(self):
        """Parents-first trie rebuild (dictionary.py:170-194)."""
        n = DICT_SIZE
        nxt = np.full((n + 1, 9), -1, np.int32)
        ent = np.full(n + 1, -1, np.int32)
        for i in range(n):
            node = 0
            k = int(self.pair_counts[i])
            row = self.values[i]
            for j in range(k - 1):
                node = nxt[node, 3 * row[2 * j] + row[2 * j + 1]]
                if node < 0:
                    raise OracleCorruption("entry table is not prefix-closed")
            sym = 3 * row[2 * k - 2] + row[2 * k - 1]
            if nxt[node, sym] != -1:
                raise OracleCorruption("duplicate entry")
            nxt[node, sym] = i + 1
            ent[i + 1] = i
        return nxt, ent


# --------------------------------------------------------------------------- codec
def row_ranges(rows: int, workers: int):
    """codec.py:63-66."""
    w = max(1, min(workers, rows)) if rows else 1
    b = np.linspace(0, rows, w + 1).astype(int)
    return [(int(a), int(c)) for a, c in zip(b[:-1], b[1:]) if a < c]


def validate(rows, cols, cw, row_off, row_minmax) -> None:
    """CompressedMatrix.validate (codec.py:50-60)."""
    if rows < 0 or cols < 0 or cols % 2:
        raise OracleCorruption("invalid shape")
    if row_off.shape != (rows + 1,) or row_off.dtype != np.int32:
        raise OracleCorruption("row_off must be (rows + 1,) int32")
    if rows and row_minmax.shape != (rows, 2):
        raise OracleCorruption("row_minmax must be (rows, 2)")
    if row_off[0] != 0 or row_off[-1] != len(cw):
        raise OracleCorruption("row_off does not span the codeword stream")
    if np.any(np.diff(row_off) < 0):
        raise OracleCorruption("row_off must be monotone")


def encode_codes(codes: np.ndarray, dic: OracleDictionary):
    """Greedy longest-prefix encode, rows independent (codec.py:69-155).
    Restated as a lock-step trie walk over all rows at once (:100-114):
    a row either follows its trie edge or emits its current entry and
    retries the same pair from the root."""
    rows, cols = codes.shape
    if cols % 2:
        raise ValueError("column count must be even")
    npair = cols // 2
    pairs = (3 * codes[:, 0::2].astype(np.int32) + codes[:, 1::2]).astype(np.int32)
    counts = np.zeros(rows, np.int64)
    emitted = [[] for _ in range(rows)]
    if npair and rows:
        state = np.zeros(rows, np.int32)
        cur = np.zeros(rows, np.int32)
        live = np.arange(rows)
        while live.size:
            step = dic.next_node[state[live], pairs[live, cur[live]]]
            stall = live[step < 0]
            for r, e in zip(stall, dic.entry_of_node[state[stall]]):
                emitted[r].append(int(e))
            state[stall] = 0
            go = live[step >= 0]
            state[go] = step[step >= 0]
            cur[go] += 1
            done = go[cur[go] == npair]
            for r, e in zip(done, dic.entry_of_node[state[done]]):
                emitted[r].append(int(e))
            live = live[cur[live] < npair]
    for r in range(rows):
        counts[r] = len(emitted[r])
    row_off = np.zeros(rows + 1, np.int64)
    np.cumsum(counts, out=row_off[1:])
    cw = np.array([e for r in emitted for e in r], dtype=np.uint16)
    return cw, row_off.astype(np.int32)


def decode_range(cols, cw, row_off, dic, r0, r1) -> np.ndarray:
    """codec.py:158-172: lengths 2*n, cumulative cuts, per-row length check,
    masked gather of the expanded values."""
    lo, hi = int(row_off[r0]), int(row_off[r1])
    idx = cw[lo:hi].astype(np.intp)
    ln = 2 * dic.pair_counts[idx].astype(np.int64)
    cuts = np.concatenate([[0], np.cumsum(ln)])
    per_row = cuts[row_off[r0 + 1 : r1 + 1] - lo] - cuts[row_off[r0:r1] - lo]
    if np.any(per_row != cols):
        raise OracleCorruption("row decodes to the wrong number of values")
    keep = np.arange(28)[None, :] < ln[:, None]
    return dic.values[idx][keep].reshape(r1 - r0, cols)


def decompress(rows, cols, cw, row_off, row_minmax, dict_hash, dic, workers=1) -> np.ndarray:
    """codec.py:175-193 -> codes (rows, cols) uint8."""
    validate(rows, cols, cw, row_off, row_minmax)
    if dict_hash != dic.hash64:
        raise OracleMismatch("dictionary mismatch")
    rr = row_ranges(rows, workers)
    if not rr:
        return np.zeros((rows, cols), np.uint8)
    if len(rr) == 1:
        return decode_range(cols, cw, row_off, dic, 0, rows)
    with ThreadPoolExecutor(len(rr)) as ex:
        return np.concatenate(list(ex.map(lambda r: decode_range(cols, cw, row_off, dic, *r), rr)))


def levels(row_minmax) -> np.ndarray:
    """reconstruction_levels('ternary') (quantize.py:38-51): [0, min, max]."""
    mn = bf16_bits_to_f32(row_minmax[:, 0])
    mx = bf16_bits_to_f32(row_minmax[:, 1])
    return np.stack([np.zeros_like(mn), mn, mx], axis=1)


def matvec_range(cols, cw, row_off, row_minmax, dic, x32, r0, r1) -> np.ndarray:
    """codec.py:196-206: 128-row chunks, dense fp32 dequant, sgemv."""
    out = np.empty(r1 - r0, np.float32)
    lv = levels(row_minmax[r0:r1])
    for b0 in range(r0, r1, 128):
        b1 = min(r1, b0 + 128)
        codes = decode_range(cols, cw, row_off, dic, b0, b1)
        w = np.take_along_axis(lv[b0 - r0 : b1 - r0], codes.astype(np.intp), axis=1)
        out[b0 - r0 : b1 - r0] = w @ x32
    return out


def fused_matvec(rows, cols, cw, row_off, row_minmax, dict_hash, x, dic, y=None, workers=1):
    """codec.py:209-244: y[r] += bf16_round(fp32 dot(level_r, x))."""
    validate(rows, cols, cw, row_off, row_minmax)
    if dict_hash != dic.hash64:
        raise OracleMismatch("dictionary mismatch")
    x32 = np.asarray(x, np.float32)
    if x32.shape != (cols,):
        raise ValueError("bad x shape")
    if y is None:
        y = np.zeros(rows, np.float32)
    elif y.shape != (rows,):
        raise ValueError("bad y shape")
    rr = row_ranges(rows, workers)
    if len(rr) <= 1:
        parts = [matvec_range(cols, cw, row_off, row_minmax, dic, x32, 0, rows)] if rows else []
    else:
        with ThreadPoolExecutor(len(rr)) as ex:
            parts = list(ex.map(lambda r: matvec_range(cols, cw, row_off, row_minmax, dic, x32, *r), rr))
    for (a, b), p in zip(rr, parts):
        y[a:b] += bf16_round(p)
    return y


def warp_trace(cols, cw, row_off, dic, row):
    """simulate_warp_row (codec.py:293-338): fetch blocks of 32, per symbol
    lanes 0..27 read word lane//14 slot lane%14, offset += 2n."""
    c = cw[int(row_off[row]) : int(row_off[row + 1])]
    fetch = [int(min(32, len(c) - b)) for b in range(0, len(c), 32)]
    lanes = np.arange(28)
    offs, npairs, lane_vals = [], [], []
    counts = np.zeros(32, np.int64)
    off = 0
    for e in c.tolist():
        w = dic.decode_words[e]
        n = int(w[0] & 0xF)
        if n != int(w[1] & 0xF):
            raise OracleCorruption("pair count differs")
        lane_vals.append(((w[lanes // 14].astype(np.uint32) >> (4 + 2 * (lanes % 14))) & 3).astype(np.uint8))
        offs.append(off)
        npairs.append(n)
        counts[: 2 * n] += 1
        off += 2 * n
    if off != cols:
        raise OracleCorruption("row decodes to the wrong number of values")
    return {"fetch_sizes": fetch, "codewords": c.tolist(), "offsets": offs,
            "pair_counts": npairs, "extract_counts": counts, "lane_values": lane_vals}


# --------------------------------------------------------------------------- quantize
def make_grid_bits(w: np.ndarray) -> np.ndarray:
    """make_grid (quantize.py:91-107) + minmax_bits (:80-84)."""
    w = np.asarray(w)
    return np.stack([f32_to_bf16_bits(w.min(axis=1).astype(np.float32)),
                     f32_to_bf16_bits(w.max(axis=1).astype(np.float32))], axis=1)


def rtn_codes(w: np.ndarray, minmax_bits: np.ndarray) -> np.ndarray:
    """rtn_quantize (quantize.py:219-235): nearest level in float64, ties to
    the smaller-magnitude level, equal magnitudes in code order (:110-126)."""
    lv = levels(minmax_bits).astype(np.float64)
    order = np.argsort(np.abs(lv), axis=1, kind="stable")
    srt = np.take_along_axis(lv, order, axis=1)
    d = np.abs(np.asarray(w, np.float64)[..., None] - srt[:, None, :])
    pick = np.argmin(d, axis=-1)
    return np.take_along_axis(np.broadcast_to(order[:, None, :], d.shape), pick[..., None], axis=-1)[..., 0].astype(np.uint8)


# --------------------------------------------------------------------------- MoE composition
def router_argmax(tokens: np.ndarray, num_experts: int, seed: int = 0, skew: float = 0.0) -> np.ndarray:
    """RouterSim(rule='argmax').assign (pipeline.py:164-182), float64."""
    t = np.asarray(tokens, np.float32)
    proj = np.random.default_rng(seed).normal(size=(t.shape[1], num_experts))
    s = t.astype(np.float64) @ proj
    bias = skew * math.sqrt(t.shape[1]) * np.linspace(1.0, 0.0, num_experts)
    return np.argmax(s + bias[None, :], axis=1).astype(np.int32)


def moe_layer(x, assign, experts, dic, workers=1):
    """Composed CPU MoE oracle (gather order pipeline.py:86-90):
    per expert in index order, tokens in buffer order, y_t = wo @ relu(wi @ x_t)
    with both matvecs through fused_matvec. `experts[e] = (wi, wo)` where each
    is (rows, cols, cw, row_off, row_minmax)."""
    T, d = x.shape
    y = np.zeros((T, experts[0][1][0]), np.float32)
    for e in range(len(experts)):
        wi, wo = experts[e]
        for p in np.flatnonzero(assign == e):
            h = fused_matvec(*wi[:2], *wi[2:], dic.hash64, x[p], dic, workers=workers)
            h = np.maximum(h, 0.0)
            y[p] = fused_matvec(*wo[:2], *wo[2:], dic.hash64, h, dic, workers=workers)
    return y


# --------------------------------------------------------------------------- accounting
def compressed_bytes(rows: int, n_codewords: int) -> int:
    """(payload + metadata) bits / 8 from compression_rate (stats.py:103-114)."""
    return 2 * n_codewords + 4 * (rows + 1) + 4 * rows
