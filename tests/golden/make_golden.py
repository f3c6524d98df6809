"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (`moepack`, /root/reference/pkg/src) in this container.

This script is the only thing in the repo that imports the reference. It is
run by hand (``python tests/golden/make_golden.py``) where /root/reference
exists; its outputs are committed so that the oracle (oracle/) and the CUDA
path can be pinned on boxes where the reference is absent.

Every fixture records what reference call produced it:
  dict.npz          generate_dictionary(PairDistribution(p)) for p in (0.885, 0.7)
                    (dictionary.py:234-279), hash64 (:227-231), sampled entries
  codec_small.npz   encode / decompress / fused_matvec on small random cases
                    (codec.py:126-244), incl. edge shapes from test_codec.py
  shapes.npz        RTN(N(0, 0.02^2)) 768x3072 and 3072x768 (quantize.py:91-126,
                    219-235) encoded + one fused_matvec (SURVEY 8(d) recipe)
  moe_tiny.npz      composed MoE oracle: RouterSim argmax (pipeline.py:164-182),
                    gather order (:86-90), wi -> relu -> wo via fused_matvec
  trace.json        simulate_warp_row traces (codec.py:293-338)
  checkpoint.bin    write_checkpoint bytes (codec.py:341-351)
  misc.json         compression_rate (stats.py:103-114), theoretical_limit
  routing.npz       RouterSim.assign hash / argmax (+skew) (pipeline.py:164-182)
                    on bf16 tokens (the GPU router's parity vectors)
  stacked_wi.bin,   a stacked multi-expert MoE layer as the reference CLI writes
  stacked_wo.bin,   one (cli.py:150-153 _stack_quantized, :194-201 encode +
  stacked.npz       write_checkpoint; rows_per_expert in the report): all
                    experts' wi stacked by rows in one QMOE0001 file, the wo
                    likewise; stacked.npz = tokens, routing and the composed
                    fused_matvec outputs

`python tests/golden/make_golden.py routing|stacked` regenerates one fixture.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from moepack.bf16 import bf16_round, f32_to_bf16_bits  # noqa: E402
from moepack.codec import (  # noqa: E402
    decompress,
    encode,
    fused_matvec,
    simulate_warp_row,
    write_checkpoint,
)
from moepack.dictionary import PairDistribution, generate_dictionary  # noqa: E402
from moepack.pipeline import RouterSim  # noqa: E402
from moepack.quantize import TernaryMatrix, make_grid, rtn_quantize  # noqa: E402
from moepack.stats import compression_rate, theoretical_limit  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def make_ternary(codes, row_min=-1.0, row_max=1.0):
    codes = np.asarray(codes, dtype=np.uint8)
    mm = np.tile(
        f32_to_bf16_bits(np.array([row_min, row_max], dtype=np.float32)),
        (codes.shape[0], 1),
    ).astype(np.uint16)
    return TernaryMatrix(codes=codes, row_minmax=mm)


def random_codes(rng, rows, cols, p0):
    u = rng.random(size=(rows, cols))
    q = (1.0 - p0) / 2.0
    return np.where(u < p0, 0, np.where(u < p0 + q, 1, 2)).astype(np.uint8)


def rtn_matrix(seed_words, rows, cols):
    rng = np.random.default_rng(np.random.SeedSequence(seed_words))
    w = (rng.normal(size=(rows, cols)) * 0.02).astype(np.float32)
    return rtn_quantize(w, make_grid(w, "ternary"))


def main() -> None:
    dic = generate_dictionary(PairDistribution(0.885))
    dic_low = generate_dictionary(PairDistribution(0.7))

    # ---------------- dictionary ----------------
    sample_idx = np.concatenate([np.arange(64), np.arange(64, 65536, 257), [65535]])
    nz = np.count_nonzero(dic.values, axis=1)
    np.savez_compressed(
        os.path.join(HERE, "dict.npz"),
        hash_885=np.uint64(dic.hash64),
        hash_07=np.uint64(dic_low.hash64),
        sample_idx=sample_idx,
        words_885=dic.decode_words[sample_idx],
        words_07=dic_low.decode_words[sample_idx],
        pair_hist_885=np.bincount(dic.pair_counts, minlength=15),
        nz_hist_885=np.bincount(nz, minlength=29),
        max_nz_07=np.int64(np.count_nonzero(dic_low.values, axis=1).max()),
        next_node_root=dic.trie.next_node[0],
    )

    # ---------------- small codec cases ----------------
    rng = np.random.default_rng(20231025)
    cases = []
    fixed = [
        np.zeros((1, 28), np.uint8),
        np.array([[0, 0], [1, 2]], np.uint8),
        np.zeros((1, 30), np.uint8),
        np.zeros((1, 160), np.uint8),
        np.zeros((3, 0), np.uint8),
        np.array([[1, 2]], np.uint8),
    ]
    for codes in fixed:
        cases.append((codes, -1.0, 1.0))
    for p0 in (0.0, 0.3, 0.6, 0.885, 0.97, 1.0):
        for _ in range(3):
            rows = int(rng.integers(1, 65))
            cols = 2 * int(rng.integers(1, 300))
            cases.append((random_codes(rng, rows, cols, p0), -0.37, 0.81))
    # a wider case with a long row (> 512 codewords per row at p0 = 0)
    cases.append((random_codes(rng, 5, 2 * 1100, 0.0), -0.5, 0.25))
    out = {}
    for i, (codes, mn, mx) in enumerate(cases):
        t = make_ternary(codes, mn, mx)
        c = encode(t, dic)
        out[f"c{i}_codes"] = codes
        out[f"c{i}_minmax"] = t.row_minmax
        out[f"c{i}_cw"] = c.codewords
        out[f"c{i}_row_off"] = c.row_off
        if codes.shape[1] > 0:
            x = (rng.normal(size=codes.shape[1]) / np.sqrt(codes.shape[1])).astype(np.float32)
            y0 = rng.normal(size=codes.shape[0]).astype(np.float32)
            out[f"c{i}_xbits"] = f32_to_bf16_bits(x)  # exact: x is bf16-valued
            out[f"c{i}_y"] = fused_matvec(c, x, dic)
            out[f"c{i}_y0"] = y0
            out[f"c{i}_y_acc"] = fused_matvec(c, x, dic, y=y0.copy())
        assert np.array_equal(decompress(c, dic).codes, codes)
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "codec_small.npz"), **out)

    # ---------------- realistic shapes ----------------
    shp = {}
    for name, (rows, cols, m) in {"wo": (768, 3072, 1), "wi": (3072, 768, 0)}.items():
        t = rtn_matrix([0, 0, 0, m], rows, cols)
        c = encode(t, dic, workers=8)
        x = bf16_round(np.random.default_rng(np.random.SeedSequence([1, m])).normal(size=cols).astype(np.float32))
        shp[f"{name}_minmax"] = c.row_minmax
        shp[f"{name}_cw"] = c.codewords
        shp[f"{name}_row_off"] = c.row_off
        shp[f"{name}_x"] = x
        shp[f"{name}_y"] = fused_matvec(c, x, dic, workers=8)
        shp[f"{name}_codes_sha"] = np.frombuffer(
            __import__("hashlib").sha256(t.codes.tobytes()).digest(), np.uint8
        )
        shp[f"{name}_codes_row0"] = t.codes[0]
        shp[f"{name}_nonzero_count"] = np.int64(np.count_nonzero(t.codes))
        # a small RTN case with its float weights, to pin the quantizer
    w_rng = np.random.default_rng(np.random.SeedSequence([9, 9]))
    w = (w_rng.normal(size=(16, 40)) * 0.02).astype(np.float32)
    w[3, :] = 0.0
    w[5, 7] = w[5, 8]  # duplicate values
    q = rtn_quantize(w, make_grid(w, "ternary"))
    shp["rtn_w"] = w
    shp["rtn_codes"] = q.codes
    shp["rtn_minmax"] = q.row_minmax
    np.savez_compressed(os.path.join(HERE, "shapes.npz"), **shp)

    # ---------------- tiny MoE layer (composed reference oracle) ----------------
    E, d_model, d_ff, T = 4, 64, 256, 16
    moe = {}
    mats = {}
    for e in range(E):
        for m, (rows, cols) in enumerate([(d_ff, d_model), (d_model, d_ff)]):
            t = rtn_matrix([7, 0, e, m], rows, cols)
            c = encode(t, dic)
            mats[(e, m)] = c
            moe[f"e{e}_m{m}_cw"] = c.codewords
            moe[f"e{e}_m{m}_row_off"] = c.row_off
            moe[f"e{e}_m{m}_minmax"] = c.row_minmax
    x = bf16_round(np.random.default_rng(11).normal(size=(T, d_model)).astype(np.float32))
    assign = RouterSim(num_experts=E, rule="argmax", seed=0).assign(x)
    y = np.zeros((T, d_model), np.float32)
    order = []
    for e in range(E):
        pos = np.flatnonzero(assign == e)
        order.extend(pos.tolist())
        for p in pos:
            h = np.maximum(fused_matvec(mats[(e, 0)], x[p], dic), 0.0)
            y[p] = fused_matvec(mats[(e, 1)], h, dic)
    moe.update(x=x, assign=assign, y=y, order=np.array(order, np.int64),
               E=np.int64(E), d_model=np.int64(d_model), d_ff=np.int64(d_ff))
    np.savez_compressed(os.path.join(HERE, "moe_tiny.npz"), **moe)

    # ---------------- warp traces ----------------
    tr_rng = np.random.default_rng(90)
    t = make_ternary(random_codes(tr_rng, 4, 200, 0.3))
    c = encode(t, dic)
    traces = {"codes": t.codes.tolist(), "rows": []}
    for r in range(t.rows):
        tr = simulate_warp_row(c, r, dic)
        traces["rows"].append(
            {
                "fetch_sizes": tr.fetch_sizes,
                "codewords": [s.codeword for s in tr.symbols],
                "pair_counts": [s.pair_count for s in tr.symbols],
                "offsets": [s.offset for s in tr.symbols],
                "extract_counts": tr.extract_counts.tolist(),
                "lane_values_first": tr.symbols[0].lane_values.tolist(),
            }
        )
    with open(os.path.join(HERE, "trace.json"), "w") as fh:
        json.dump(traces, fh)

    # ---------------- checkpoint + rates ----------------
    ck_rng = np.random.default_rng(95)
    t = make_ternary(random_codes(ck_rng, 9, 24, 0.885))
    c = encode(t, dic)
    write_checkpoint(c, os.path.join(HERE, "checkpoint.bin"))
    np.save(os.path.join(HERE, "checkpoint_codes.npy"), t.codes)
    misc = {
        "rate_1x28": compression_rate(encode(make_ternary(np.zeros((1, 28), np.uint8)), dic)).as_dict(),
        "rate_wo": compression_rate(mats[(0, 1)]).as_dict(),
        "theoretical_limit_885": theoretical_limit(0.885),
    }
    with open(os.path.join(HERE, "misc.json"), "w") as fh:
        json.dump(misc, fh, indent=1)
    print("golden fixtures written to", HERE)


def make_routing() -> None:
    out = {}
    cases = [("hash", 128, 768, 64, 0.0, 3), ("hash", 2048, 2080, 12, 0.0, 5), ("argmax", 128, 768, 64, 0.0, 1),
             ("argmax", 128, 768, 64, 0.5, 1), ("argmax", 2048, 2080, 12, 0.0, 2)]
    for i, (rule, E, d, T, skew, seed) in enumerate(cases):
        x = bf16_round(np.random.default_rng(100 + i).normal(size=(T, d)).astype(np.float32))
        out[f"c{i}_xbits"] = f32_to_bf16_bits(x)  # exact: x is bf16-valued
        out[f"c{i}_assign"] = RouterSim(num_experts=E, rule=rule, seed=seed, skew=skew).assign(x)
        out[f"c{i}_meta"] = np.array([E, d, T, seed], np.int64)
        out[f"c{i}_rule"] = np.array(rule)
        out[f"c{i}_skew"] = np.float64(skew)
    out["n"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "routing.npz"), **out)
    print("routing.npz written")


def make_stacked() -> None:
    dic = generate_dictionary(PairDistribution(0.885))
    E, d_model, d_ff, T = 6, 96, 224, 24
    quant = {0: [], 1: []}
    for e in range(E):
        for m, (rows, cols) in enumerate([(d_ff, d_model), (d_model, d_ff)]):
            quant[m].append(rtn_matrix([13, 0, e, m], rows, cols))
    stacked = {}
    for m, name in ((0, "wi"), (1, "wo")):  # cli.py:150-153, 194-201
        st = TernaryMatrix(codes=np.concatenate([t.codes for t in quant[m]], axis=0),
                           row_minmax=np.concatenate([t.row_minmax for t in quant[m]], axis=0))
        c = encode(st, dic, workers=2)
        write_checkpoint(c, os.path.join(HERE, f"stacked_{name}.bin"))
        stacked[m] = c
    x = bf16_round(np.random.default_rng(31).normal(size=(T, d_model)).astype(np.float32))
    assign = RouterSim(num_experts=E, rule="argmax", seed=0).assign(x)
    assign[5] = -1  # a token without an expert: zero output row
    per = {(e, m): encode(quant[m][e], dic) for e in range(E) for m in (0, 1)}
    y = np.zeros((T, d_model), np.float32)
    for e in range(E):
        for p in np.flatnonzero(assign == e):
            h = np.maximum(fused_matvec(per[(e, 0)], x[p], dic), 0.0)
            y[p] = fused_matvec(per[(e, 1)], h, dic)
    np.savez_compressed(os.path.join(HERE, "stacked.npz"), x=x, assign=assign, y=y, E=np.int64(E),
                        d_model=np.int64(d_model), d_ff=np.int64(d_ff))
    print("stacked_*.bin / stacked.npz written")


if __name__ == "__main__":
    if sys.argv[1:] == ["routing"]:
        make_routing()
    elif sys.argv[1:] == ["stacked"]:
        make_stacked()
    else:
        main()
        make_routing()
        make_stacked()
