"""Host cube/truth-table helpers (paper_2302_10083_b200.ternary): known answers
from the reference's tests, round trips, and — where the read-only reference
package is importable in this container — equality with its functions on
random inputs (ternary.py:63-264)."""

import os
import sys

import numpy as np
import pytest

from paper_2302_10083_b200 import ternary as T

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref_ternary():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF_SRC)
    try:
        from implicants import ternary as R
    finally:
        sys.path.remove(REF_SRC)
    return R


def test_known_answers():
    # tests/test_oracle.py:51-54 / test_dense.py:202-205: points {12, 14} at n=5 -> "0*110", rank 42
    assert T.rank("0*110") == 42 and T.unrank(42, 5) == "0*110"
    # Maj3 primes (test_dense.py:187-189)
    assert T.unrank_many([14, 16, 22], 3) == ["*11", "1*1", "11*"]
    assert T.index_to_rank(np.array([12, 14]), 5).tolist() == [T.rank("00110"), T.rank("01110")]
    assert T.rank_weights(np.array([42, 0, 3**5 - 1]), 5).tolist() == [1, 0, 5]
    assert T.ranks_to_text(np.array([42]), 5, "-") == "0-110\n"
    assert T.ranks_to_text(np.array([], dtype=np.int64), 5) == ""


def test_round_trips():
    rng = np.random.default_rng(1)
    for n in (1, 5, 13, 20, 31):
        r = rng.integers(0, 3**n, size=200, dtype=np.uint64)
        strs = T.unrank_many(r, n)
        assert [T.rank(s) for s in strs] == r.tolist()
        d = T.rank_digits(r, n)
        assert np.array_equal((d.astype(np.uint64) * np.array([3**i for i in range(n)], dtype=np.uint64)).sum(1), r)
    x = rng.integers(0, 2**31, size=500, dtype=np.uint64)
    ranks = T.index_to_rank(x, 31)
    assert all(set(s) <= {"0", "1"} for s in T.unrank_many(ranks, 31))


def test_truth_table_roundtrip_and_validation():
    rng = np.random.default_rng(2)
    for n in (1, 3, 6, 7, 12):
        v = rng.random(1 << n) < 0.4
        tt = T.TruthTable.from_bools(n, v)
        assert np.array_equal(tt.bools(), v)
        assert tt.popcount() == int(v.sum())
        assert np.array_equal(tt.support_indices(), np.flatnonzero(v))
        assert tt == T.TruthTable.from_indices(n, np.flatnonzero(v))
        assert hash(tt) == hash(T.TruthTable(n, tt.words))
        assert not tt.words.flags.writeable
    assert T.TruthTable.full(3).words.tolist() == [255] and T.TruthTable.empty(7).popcount() == 0
    with pytest.raises(ValueError):
        T.TruthTable(0, [0])
    with pytest.raises(ValueError):
        T.TruthTable(3, [256])  # a bit beyond 2^3
    with pytest.raises(ValueError):
        T.TruthTable(7, [0])  # 2 words expected
    with pytest.raises(ValueError):
        T.TruthTable.from_indices(4, [16])
    with pytest.raises(ValueError):
        T.unrank(3**4, 4)


def test_matches_reference_helpers(ref_ternary):
    R = ref_ternary
    rng = np.random.default_rng(3)
    for n in (1, 4, 9, 17, 26):
        r = rng.integers(0, 3**n, size=300, dtype=np.uint64)
        assert np.array_equal(T.rank_digits(r, n), R.rank_digits(r, n))
        assert np.array_equal(T.rank_weights(r, n), R.rank_weights(r, n))
        assert T.unrank_many(r, n) == R.unrank_many(r, n)
        assert T.ranks_to_text(r, n, "-") == R.ranks_to_text(r, n, "-")
        x = rng.integers(0, 2**n, size=300, dtype=np.uint64)
        assert np.array_equal(T.index_to_rank(x, n), R.index_to_rank(x, n))
        v = rng.random(1 << min(n, 16)) < 0.5
        m = min(n, 16)
        a, b = T.TruthTable.from_bools(m, v), R.TruthTable.from_bools(m, v)
        assert np.array_equal(a.words, b.words)
        assert np.array_equal(a.support_indices(), b.support_indices())
