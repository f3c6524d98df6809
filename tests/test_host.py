"""CPU tests of the library boundary and the drop-in host logic (no GPU):
every include/qmoe.h symbol is exported, host-side generation/trie/tables
match the oracle and golden vectors, and the reference's error contract for
containers, dictionaries, shapes and routing holds. Modelled on the
reference's pkg/tests/test_dictionary.py, test_codec.py (container),
test_stats.py and test_bf16.py."""

import os
import re
import struct

import numpy as np
import pytest

import paper_2310_16795_b200 as q
from conftest import GOLDEN, ROOT, make_ternary, random_codes
from oracle import qmoe_oracle as O
from paper_2310_16795_b200 import _lib


# ----------------------------------------------------------------- C ABI
def header_functions():
    with open(os.path.join(ROOT, "include", "qmoe.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(qmoe_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), f"libqmoe.so does not export {n}"
    assert set(names) == set(_lib.EXPORTED)


def test_struct_layouts_match_header():
    import ctypes

    assert ctypes.sizeof(_lib.QmoeWork) == 80
    assert ctypes.sizeof(_lib.QmoeMatrix) == 64


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.lib.qmoe_generate_decode_words(0.2, _lib.ptr(np.empty((65536, 2), np.uint32))))
    assert "p0" in _lib.last_error()


# ----------------------------------------------------------------- dictionary
def test_generation_matches_reference_hash_and_oracle(dic, golden):
    g = golden("dict.npz")
    assert dic.hash64 == 0x81F83180EF6B1A92 == int(g["hash_885"])
    assert np.array_equal(dic.decode_words[g["sample_idx"]], g["words_885"])
    assert np.array_equal(dic.decode_words, O.generate_decode_words(0.885))


def test_low_p0_dictionary(dic_low, golden):
    g = golden("dict.npz")
    assert dic_low.hash64 == int(g["hash_07"])
    assert np.array_equal(dic_low.decode_words[g["sample_idx"]], g["words_07"])


def test_first_entries_structure(dic):
    for k in range(12):
        assert dic.entry(k) == ((0, 0),) * (k + 1)
    assert [dic.entry(i) for i in range(12, 16)] == [((0, 1),), ((0, 2),), ((1, 0),), ((2, 0),)]
    assert dic.entry(16) == ((0, 0),) * 13
    assert dic.entry(25) == ((0, 0),) * 14


def test_trie_matches_oracle(dic, odic):
    assert np.array_equal(dic.trie.next_node, odic.next_node)
    assert np.array_equal(dic.trie.entry_of_node, odic.entry_of_node)
    entry, used = dic.trie.longest_prefix(np.zeros(20, np.uint8), 0)
    assert dic.entry(entry) == ((0, 0),) * 14 and used == 14


def test_pack_unpack_known_answers():
    assert q.pack_decode_words([(0, 0), (1, 2)]) == (2306, 2)
    assert q.unpack_decode_words(2306, 2) == [(0, 0), (1, 2)]
    assert q.pack_decode_words([(0, 0)]) == (1, 1)
    assert q.pack_decode_words([(2, 1)]) == (1 | (2 << 4) | (1 << 6), 1)
    with pytest.raises(ValueError):
        q.pack_decode_words([])
    with pytest.raises(ValueError):
        q.pack_decode_words([(0, 3)])
    with pytest.raises(q.CorruptionError):
        q.unpack_decode_words(2, 3)


def test_corrupt_tables_rejected(dic):
    w = dic.decode_words.copy()
    w[5, 1] ^= 1  # pair counts differ
    with pytest.raises(q.CorruptionError):
        q.Dictionary(0.885, w)
    w = dic.decode_words.copy()
    w[0, 0] |= 3 << 10  # non-zero padding in a 1-pair entry
    with pytest.raises(q.CorruptionError):
        q.Dictionary(0.885, w)
    w = dic.decode_words.copy()
    w[[1, 2]] = w[[2, 1]]  # child before parent -> not prefix-closed (parents-first)
    with pytest.raises(q.CorruptionError):
        q.Dictionary(0.885, w)


def test_dictionary_file_round_trip_and_errors(dic, tmp_path):
    p = tmp_path / "d.bin"
    q.save_dictionary(dic, str(p))
    blob = p.read_bytes()
    assert len(blob) == 8 + 1 + 8 + 65536 * 8
    assert blob[:8] == b"QMOEDICT" and blob[8] == 1
    back = q.load_dictionary(str(p))
    assert back.hash64 == dic.hash64
    for bad in (b"XXXXXXXX" + blob[8:], blob[:8] + bytes([2]) + blob[9:], blob[:100], blob + b"\0"):
        p.write_bytes(bad)
        with pytest.raises(q.CorruptionError):
            q.load_dictionary(str(p))


# ----------------------------------------------------------------- container
def test_checkpoint_matches_reference_bytes(dic, tmp_path):
    ref = open(os.path.join(GOLDEN, "checkpoint.bin"), "rb").read()
    c = q.read_checkpoint(os.path.join(GOLDEN, "checkpoint.bin"))
    assert (c.rows, c.cols, c.dict_hash) == (9, 24, dic.hash64)
    p = tmp_path / "m.bin"
    q.write_checkpoint(c, str(p))
    assert p.read_bytes() == ref
    codes = np.load(os.path.join(GOLDEN, "checkpoint_codes.npy"))
    od = O.OracleDictionary(0.885, dic.decode_words)
    assert np.array_equal(O.decompress(9, 24, c.codewords, c.row_off, c.row_minmax, c.dict_hash, od), codes)


@pytest.mark.parametrize("cut", [0, 7, 20, 45])
def test_checkpoint_truncation(tmp_path, cut):
    ref = open(os.path.join(GOLDEN, "checkpoint.bin"), "rb").read()
    p = tmp_path / "m.bin"
    p.write_bytes(ref[:cut])
    with pytest.raises(q.CorruptionError):
        q.read_checkpoint(str(p))


def test_checkpoint_magic_trailing_and_odd_cols(tmp_path):
    ref = bytearray(open(os.path.join(GOLDEN, "checkpoint.bin"), "rb").read())
    p = tmp_path / "m.bin"
    bad = bytearray(ref)
    bad[:8] = b"QMOE9999"
    p.write_bytes(bytes(bad))
    with pytest.raises(q.CorruptionError):
        q.read_checkpoint(str(p))
    p.write_bytes(bytes(ref) + b"\0\0")
    with pytest.raises(q.CorruptionError):
        q.read_checkpoint(str(p))
    odd = bytearray(ref)
    struct.pack_into("<Q", odd, 16, 23)
    p.write_bytes(bytes(odd))
    with pytest.raises(q.CorruptionError):
        q.read_checkpoint(str(p))


def test_validate_contract():
    c = q.CompressedMatrix(2, 28, np.zeros(2, np.uint16), np.array([0, 1, 2], np.int32),
                           np.zeros((2, 2), np.uint16), 0)
    c.validate()
    for ro in (np.array([0, 2, 1], np.int32), np.array([0, 1, 3], np.int32), np.array([0, 1, 2], np.int64)):
        bad = q.CompressedMatrix(2, 28, np.zeros(2, np.uint16), ro, np.zeros((2, 2), np.uint16), 0)
        with pytest.raises(q.CorruptionError):
            bad.validate()
    with pytest.raises(q.CorruptionError):
        q.CompressedMatrix(1, 3, np.zeros(0, np.uint16), np.zeros(2, np.int32), np.zeros((1, 2), np.uint16),
                           0).validate()


def test_pad_to_even():
    t = make_ternary([[1, 2, 1]])
    p = q.pad_to_even(t)
    assert p.cols == 4 and np.array_equal(p.codes, [[1, 2, 1, 0]]) and p.dequant()[0, 3] == 0.0
    e = make_ternary([[1, 2]])
    assert q.pad_to_even(e) is e


# ----------------------------------------------------------------- quantize / stats / bf16
def test_ternary_matrix_validation():
    with pytest.raises(ValueError):
        q.TernaryMatrix(codes=np.array([[3]], np.uint8), row_minmax=np.zeros((1, 2), np.uint16))
    with pytest.raises(ValueError):
        q.TernaryMatrix(codes=np.array([[1]], np.uint8), row_minmax=np.zeros((2, 2), np.uint16))
    with pytest.raises(ValueError):
        q.make_grid(np.array([[np.inf]]))


def test_rates_and_limit():
    c = q.CompressedMatrix(1, 28, np.zeros(1, np.uint16), np.array([0, 1], np.int32), np.zeros((1, 2), np.uint16), 0)
    r = q.compression_rate(c)
    assert (r.payload_bits, r.metadata_bits, r.original_bits) == (16, 96, 448)
    assert r.moe_only_rate == pytest.approx(4.0)
    assert q.theoretical_limit(0.885) == pytest.approx(25.40, abs=0.01)
    t = q.sample_ternary(q.PairDistribution(0.885), 50, 400, seed=3)
    assert 0.85 < q.natural_sparsity(t) < 0.92


def test_bf16_helpers():
    u = np.array([0x3F808000, 0x3F818000, 0x3F80FFFF], np.uint32).view(np.float32)
    assert q.f32_to_bf16_bits(u).tolist() == [0x3F80, 0x3F82, 0x3F81]
    assert q.bf16_round(np.float32(1.0)) == 1.0


# ----------------------------------------------------------------- routing / EP host logic
def test_router_matches_reference(golden):
    g = golden("moe_tiny.npz")
    a = q.RouterSim(int(g["E"]), rule="argmax", seed=0).assign(g["x"])
    assert np.array_equal(a, g["assign"])
    assert np.array_equal(a, O.router_argmax(g["x"], int(g["E"]), seed=0))


def test_ep_sharding_helpers():
    from paper_2310_16795_b200.ep import shard_experts, token_split

    assert list(shard_experts(8, 4, 1)) == [2, 3]
    assert token_split(np.array([0, 7, 3, 3, 5]), 8, 2).tolist() == [3, 2]
