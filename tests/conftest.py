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


def matvec_tolerance_ok(y, y_ref, abs_terms=None, nnz=None, min_identical=0.999):
    """Matvec parity: per row |y - y_ref| <= 1 bf16 ulp of y_ref
    plus the fp32 accumulation bound nnz * 2^-24 * sum_j |w_j x_j| (the
    reference's own sgemv order is unspecified, so rows whose sum cancels can
    legitimately round to a different bf16 value); >= min_identical of the
    rows bit-identical. Returns (ok, message)."""
    y = np.asarray(y, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    ulp = np.ldexp(1.0, np.floor(np.log2(np.maximum(np.abs(y_ref), 1e-38))).astype(int) - 7)
    bound = ulp.copy()
    if abs_terms is not None:
        bound += np.asarray(nnz, np.float64) * 2.0**-24 * np.asarray(abs_terms, np.float64)
    err = np.abs(y - y_ref)
    bad = ~(err <= bound)
    same = np.mean(y == y_ref) if len(y) else 1.0
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        return False, f"{bad.sum()} rows out of tolerance, e.g. row {i}: {y[i]!r} vs {y_ref[i]!r} (bound {bound[i]:.3g})"
    if same < min_identical:
        return False, f"only {same:.4f} rows identical"
    return True, ""
