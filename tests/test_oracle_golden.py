"""Pins the CPU oracle (oracle/qmoe_oracle.py) against golden vectors produced
by the reference package itself (tests/golden/make_golden.py). CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import qmoe_oracle as O


@pytest.fixture(scope="module")
def od():
    return O.OracleDictionary(0.885)


def test_dictionary_hash_and_samples(od, golden):
    g = golden("dict.npz")
    assert od.hash64 == int(g["hash_885"]) == 0x81F83180EF6B1A92
    assert np.array_equal(od.decode_words[g["sample_idx"]], g["words_885"])
    assert np.array_equal(np.bincount(od.pair_counts, minlength=15), g["pair_hist_885"])
    nz = np.count_nonzero(od.values, axis=1)
    assert np.array_equal(np.bincount(nz, minlength=29), g["nz_hist_885"])
    assert np.array_equal(od.next_node[0], g["next_node_root"])


def test_low_p0_dictionary(golden):
    g = golden("dict.npz")
    words = O.generate_decode_words(0.7)
    assert O.dictionary_hash(0.7, words) == int(g["hash_07"])
    assert np.array_equal(words[g["sample_idx"]], g["words_07"])


def test_codec_cases(od, golden):
    g = golden("codec_small.npz")
    for i in range(int(g["n_cases"])):
        codes = g[f"c{i}_codes"]
        cw, ro = O.encode_codes(codes, od)
        assert np.array_equal(cw, g[f"c{i}_cw"]) and np.array_equal(ro, g[f"c{i}_row_off"]), i
        r, c = codes.shape
        back = O.decompress(r, c, cw, ro, g[f"c{i}_minmax"], od.hash64, od)
        assert np.array_equal(back, codes)
        if c:
            y = O.fused_matvec(r, c, cw, ro, g[f"c{i}_minmax"], od.hash64, g[f"c{i}_x"], od)
            assert np.array_equal(y, g[f"c{i}_y"])  # same algorithm, same machine class
            y0 = g[f"c{i}_y0"].copy()
            O.fused_matvec(r, c, cw, ro, g[f"c{i}_minmax"], od.hash64, g[f"c{i}_x"], od, y=y0)
            assert np.array_equal(y0, g[f"c{i}_y_acc"])


def test_realistic_shapes(od, golden):
    g = golden("shapes.npz")
    for name, (rows, cols) in {"wo": (768, 3072), "wi": (3072, 768)}.items():
        y = O.fused_matvec(rows, cols, g[f"{name}_cw"], g[f"{name}_row_off"], g[f"{name}_minmax"], od.hash64,
                           g[f"{name}_x"], od, workers=4)
        assert np.array_equal(y, g[f"{name}_y"])


def test_rtn(golden):
    g = golden("shapes.npz")
    mm = O.make_grid_bits(g["rtn_w"])
    assert np.array_equal(mm, g["rtn_minmax"])
    assert np.array_equal(O.rtn_codes(g["rtn_w"], mm), g["rtn_codes"])


def test_moe_composition(od, golden):
    g = golden("moe_tiny.npz")
    E = int(g["E"])
    assign = O.router_argmax(g["x"], E, seed=0)
    assert np.array_equal(assign, g["assign"])
    experts = []
    for e in range(E):
        pair = []
        for m in range(2):
            ro = g[f"e{e}_m{m}_row_off"]
            rows = len(ro) - 1
            cols = int(g["d_model"]) if m == 0 else int(g["d_ff"])
            pair.append((rows, cols, g[f"e{e}_m{m}_cw"], ro, g[f"e{e}_m{m}_minmax"]))
        experts.append(tuple(pair))
    y = O.moe_layer(g["x"], assign, experts, od)
    assert np.array_equal(y, g["y"])


def test_warp_trace(od):
    with open(os.path.join(GOLDEN, "trace.json")) as fh:
        g = json.load(fh)
    codes = np.array(g["codes"], np.uint8)
    cw, ro = O.encode_codes(codes, od)
    for r, want in enumerate(g["rows"]):
        tr = O.warp_trace(codes.shape[1], cw, ro, od, r)
        assert tr["fetch_sizes"] == want["fetch_sizes"]
        assert tr["codewords"] == want["codewords"]
        assert tr["offsets"] == want["offsets"]
        assert tr["extract_counts"].tolist() == want["extract_counts"]


def test_rate_accounting():
    with open(os.path.join(GOLDEN, "misc.json")) as fh:
        g = json.load(fh)
    r = g["rate_1x28"]
    assert (r["payload_bits"] + r["metadata_bits"]) // 8 == O.compressed_bytes(1, 1)
    w = g["rate_wo"]
    assert (w["payload_bits"] + w["metadata_bits"]) // 8 == O.compressed_bytes(w["rows"], w["codeword_count"])


def test_bf16_known_answers():
    # RNE halfway cases (reference tests/test_bf16.py)
    u = np.array([0x3F808000, 0x3F818000, 0x3F80FFFF, 0x7F7FFFFF, 0x00000000, 0x80000000], np.uint32)
    bits = O.f32_to_bf16_bits(u.view(np.float32))
    assert bits.tolist() == [0x3F80, 0x3F82, 0x3F81, 0x7F80, 0x0000, 0x8000]


def _routing_cases(golden):
    g = golden("routing.npz")
    for i in range(int(g["n"])):
        E, d, T, seed = (int(v) for v in g[f"c{i}_meta"])
        x = (g[f"c{i}_xbits"].astype(np.uint32) << 16).view(np.float32)
        yield str(g[f"c{i}_rule"]), E, d, T, seed, float(g[f"c{i}_skew"]), x, g[f"c{i}_assign"]


def test_routersim_mirror_matches_reference_routing(golden):
    """The package's host RouterSim (the ids the GPU path and the oracle see)
    reproduces the reference's RouterSim.assign (pipeline.py:164-182) on the
    golden vectors, both rules."""
    from paper_2310_16795_b200.pipeline import RouterSim

    n = 0
    for rule, E, d, T, seed, skew, x, want in _routing_cases(golden):
        got = RouterSim(E, rule=rule, seed=seed, skew=skew).assign(x)
        assert np.array_equal(got, want), (rule, E, d)
        n += 1
    assert n == 5
