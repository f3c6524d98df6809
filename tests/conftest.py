"""Shared fixtures. `gpu`-marked tests need a B200 (run on the GPU box);
everything else runs on CPU. The oracle under oracle/ is imported here only
as the checker."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def dic():
    import paper_2310_16795_b200 as q

    return q.generate_dictionary(q.PairDistribution(0.885))


@pytest.fixture(scope="session")
def dic_low():
    import paper_2310_16795_b200 as q

    return q.generate_dictionary(q.PairDistribution(0.7))


@pytest.fixture(scope="session")
def odic(dic):
    from oracle import qmoe_oracle as O

    return O.OracleDictionary(0.885, dic.decode_words)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))

    return load


def make_ternary(codes, row_min=-1.0, row_max=1.0):
    """tests/helpers.py:9-22 of the reference."""
    import paper_2310_16795_b200 as q

    codes = np.asarray(codes, dtype=np.uint8)
    mm = np.tile(q.f32_to_bf16_bits(np.array([row_min, row_max], np.float32)), (codes.shape[0], 1)).astype(np.uint16)
    return q.TernaryMatrix(codes=codes, row_minmax=mm)


def random_codes(rng, rows, cols, p0):
    """tests/helpers.py:25-29 of the reference."""
    u = rng.random(size=(rows, cols))
    q = (1.0 - p0) / 2.0
    return np.where(u < p0, 0, np.where(u < p0 + q, 1, 2)).astype(np.uint8)


def bf16_ulp_diff(a, b):
    """|a - b| in units of the bf16 ulp, on the float32 bit patterns (both
    operands are bf16-valued sums y = 0 + bf16(dot))."""
    ai = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    bi = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    # map sign-magnitude to a monotone integer line
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi) >> 16
