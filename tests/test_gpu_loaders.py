"""Checkpoint loaders straight to the device: QMOE0001 files
(codec.py:341-391) read into pinned memory, checked like the reference's
read_checkpoint, copied to HBM once; stacked multi-expert checkpoints as the
reference CLI writes them (cli.py:150-153, :194-201) loaded into a MoE layer
and run against the reference's own composed outputs (tests/golden/stacked.npz,
made by tests/golden/make_golden.py from moepack)."""

import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, bf16_ulp_diff

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_2310_16795_b200")
torch = pytest.importorskip("torch")

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)


def test_read_checkpoint_device_matches_host_reader(dic):
    path = os.path.join(GOLDEN, "checkpoint.bin")
    c = q.read_checkpoint(path)
    dm = q.read_checkpoint_device(path, dic)
    assert (dm.rows, dm.cols, dm.dict_hash) == (c.rows, c.cols, c.dict_hash)
    assert np.array_equal(dm.cw.cpu().numpy().view(np.uint16), c.codewords)
    assert np.array_equal(dm.row_off.cpu().numpy(), c.row_off)
    assert np.array_equal(dm.row_minmax.cpu().numpy().view(np.uint16).reshape(-1, 2), c.row_minmax)
    assert dm.bad_rows == 0
    codes = np.load(os.path.join(GOLDEN, "checkpoint_codes.npy"))
    assert np.array_equal(q.decompress(dm, dic).codes, codes)


def test_read_checkpoint_device_errors(dic, dic_low, tmp_path):
    src = os.path.join(GOLDEN, "checkpoint.bin")
    blob = open(src, "rb").read()
    bad_magic = tmp_path / "magic.bin"
    bad_magic.write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(q.CorruptionError, match="bad magic"):
        q.read_checkpoint_device(str(bad_magic), dic)
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(blob[:-2])
    with pytest.raises(q.CorruptionError, match="size disagrees"):
        q.read_checkpoint_device(str(trunc), dic)
    with pytest.raises(q.DictionaryMismatchError):
        q.read_checkpoint_device(src, dic_low)
    # a codeword that decodes to the wrong number of values: row validation on the GPU
    c = q.read_checkpoint(src)
    cw = c.codewords.copy()
    cw[0] = 25 if dic.pair_counts[cw[0]] != 14 else 0  # a different pair count (test_codec.py:362-370)
    tampered = tmp_path / "tampered.bin"
    q.write_checkpoint(q.CompressedMatrix(c.rows, c.cols, cw, c.row_off, c.row_minmax, c.dict_hash), str(tampered))
    with pytest.raises(q.CorruptionError, match="wrong number of values"):
        q.read_checkpoint_device(str(tampered), dic)


def test_load_moe_layer_from_stacked_reference_checkpoints(dic, tmp_path):
    g = np.load(os.path.join(GOLDEN, "stacked.npz"))
    E, d_model, d_ff = int(g["E"]), int(g["d_model"]), int(g["d_ff"])
    wi_path, wo_path = os.path.join(GOLDEN, "stacked_wi.bin"), os.path.join(GOLDEN, "stacked_wo.bin")
    layer = q.load_moe_layer(wi_path, wo_path, dic, max_tokens=len(g["x"]), rows_per_expert=(d_ff, d_model))
    assert (layer.E, layer.d_model, layer.d_ff) == (E, d_model, d_ff)
    y = layer.forward(g["x"], g["assign"])
    d = bf16_ulp_diff(y, g["y"])
    assert d.max() <= 2 and np.mean(d == 0) >= 0.99, (d.max(), np.mean(d == 0))
    assert np.all(y[g["assign"] < 0] == 0)
    # each expert's rows equal the stacked file's row block (rows are independent)
    st = q.read_checkpoint(wi_path)
    r0, r1 = 2 * d_ff, 3 * d_ff
    s, e = int(st.row_off[r0]), int(st.row_off[r1])
    m = layer.wi[2]
    cw = m.cw.cpu().numpy().view(np.uint16)
    assert np.array_equal(layer.codebook.order[cw], st.codewords[s:e])
    assert np.array_equal(m.row_off.cpu().numpy(), st.row_off[r0:r1 + 1] - s)
    with pytest.raises(ValueError):
        q.load_moe_layer(wi_path, wo_path, dic, rows_per_expert=(d_ff + 2, d_model))
    with pytest.raises(ValueError):
        q.read_stacked_device(wi_path, dic, rows_per_expert=d_ff - 1)
    # a corrupt row in one expert's block fails the whole load
    c = q.read_checkpoint(wo_path)
    cw = c.codewords.copy()
    k = int(c.row_off[3 * d_model + 1])
    cw[k] = 0 if dic.pair_counts[cw[k]] != 1 else 25  # a different pair count: the row's length breaks
    bad = tmp_path / "bad_wo.bin"
    q.write_checkpoint(q.CompressedMatrix(c.rows, c.cols, cw, c.row_off, c.row_minmax, c.dict_hash), str(bad))
    with pytest.raises(q.CorruptionError):
        q.load_moe_layer(wi_path, str(bad), dic)
    shutil.rmtree(tmp_path, ignore_errors=True)
