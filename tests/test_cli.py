"""CLI drop-in: the reference's cli.py subcommands and exit
codes (cli.py:232-306; its tests test_cli.py:185-280 are the model)."""

import json
import os

import numpy as np
import pytest

from paper_2310_16795_b200.cli import main

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CKPT = os.path.join(GOLDEN, "checkpoint.bin")


@pytest.fixture(scope="module")
def dict_file(tmp_path_factory):
    p = tmp_path_factory.mktemp("d") / "dict.bin"
    assert main(["gen-dict", "--out", str(p)]) == 0
    return str(p)


@pytest.fixture(scope="module")
def low_dict_file(tmp_path_factory):
    p = tmp_path_factory.mktemp("d") / "dict07.bin"
    assert main(["gen-dict", "--p0", "0.7", "--out", str(p)]) == 0
    return str(p)


def test_gen_dict_reports_reference_hash(tmp_path, capsys):
    assert main(["gen-dict", "--out", str(tmp_path / "d.bin")]) == 0
    out = capsys.readouterr().out
    assert "entries = 65536" in out
    assert "hash = 0x81f83180ef6b1a92" in out


def test_rates_text_and_json(dict_file, capsys):
    assert main(["rates", "--in", CKPT, "--dict", dict_file]) == 0
    assert "moe_only_rate = " in capsys.readouterr().out
    assert main(["rates", "--in", CKPT, "--dict", dict_file, "--json"]) == 0
    d = json.loads(capsys.readouterr().out)
    assert d["dictionary_excluded"] is True
    assert d["rows"] == 9 and d["cols"] == 24


def test_dictionary_mismatch_exit_code(low_dict_file, capsys):
    assert main(["rates", "--in", CKPT, "--dict", low_dict_file]) == 2
    assert "dictionary mismatch:" in capsys.readouterr().err


def test_corrupt_checkpoint_exit_code(dict_file, tmp_path, capsys):
    bad = tmp_path / "bad.bin"
    with open(CKPT, "rb") as fh:
        blob = fh.read()
    bad.write_bytes(blob[: len(blob) // 2])
    assert main(["rates", "--in", str(bad), "--dict", dict_file]) == 2
    assert "corrupt data:" in capsys.readouterr().err


def test_missing_file_and_usage_exit_codes(dict_file, tmp_path, capsys):
    assert main(["decompress", "--in", str(tmp_path / "nope.bin"), "--dict", dict_file,
                 "--out", str(tmp_path / "o.npz")]) == 1
    assert main(["matvec", "--in", CKPT]) == 1
    assert main(["compress"]) == 1
    x = tmp_path / "x.npy"
    np.save(str(x), np.zeros((2, 24), np.float32))
    assert main(["matvec", "--in", CKPT, "--dict", dict_file, "--x", str(x), "--y", str(tmp_path / "y.npy")]) == 1
    assert "1-d" in capsys.readouterr().err


def test_sample_matches_reference(tmp_path, capsys):
    out = tmp_path / "s.npz"
    assert main(["sample", "--rows", "4", "--cols", "28", "--seed", "1", "--out", str(out)]) == 0
    assert "sparsity = 0.901786" in capsys.readouterr().out  # reference cli, same args
    assert np.load(str(out))["codes"].shape == (4, 28)


@pytest.mark.gpu
def test_decompress_and_matvec_on_gpu(dict_file, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2310_16795_b200 as q

    out = tmp_path / "codes.npz"
    assert main(["decompress", "--in", CKPT, "--dict", dict_file, "--out", str(out)]) == 0
    assert np.array_equal(np.load(str(out))["codes"], np.load(os.path.join(GOLDEN, "checkpoint_codes.npy")))
    x = (np.random.default_rng(300).normal(size=24) / 8.0).astype(np.float32)
    xp, yp = tmp_path / "x.npy", tmp_path / "y.npy"
    np.save(str(xp), x)
    assert main(["matvec", "--in", CKPT, "--dict", dict_file, "--x", str(xp), "--y", str(yp), "--workers", "3"]) == 0
    y = np.load(str(yp))
    c = q.read_checkpoint(CKPT)
    dic = q.load_dictionary(dict_file)
    assert np.array_equal(y, q.fused_matvec(c, x, dic))  # library path, itself pinned to the oracle
