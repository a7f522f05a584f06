"""Host-side logic of the Python mirror of the reference interface that runs
without a GPU: SparseCsrMatrix.from_triplets normalisation (sparse.hpp:24-53)
and argument validation that happens before any device call. CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle.oracle import Reference, reference_available
from paper_2601_20174_b200.nlsp import SparseCsrMatrix, ValidationError


def test_triplets_deduplicated_and_sorted():
    # SparseCsr.TripletsDeduplicatedAndSorted (test_linalg.cpp:94-101)
    a = SparseCsrMatrix.from_triplets(2, [(0, 1, 1.0), (0, 0, 2.0), (0, 1, 0.5)])
    g = golden("kat")
    assert a.nnz() == 2
    assert list(a.row_ptr()) == list(g["dedup_rp"])
    assert list(a.col_idx()) == list(g["dedup_ci"])
    assert list(a.values()) == list(g["dedup_v"])


def test_zeros_dropped_and_range_checked():
    a = SparseCsrMatrix.from_triplets(3, [(0, 0, 1.0), (1, 2, 2.0), (1, 2, -2.0), (2, 2, 0.0)])
    assert a.nnz() == 1 and list(a.row_ptr()) == [0, 1, 1, 1]
    with pytest.raises(ValidationError):
        SparseCsrMatrix.from_triplets(2, [(0, 2, 1.0)])
    with pytest.raises(ValidationError):
        SparseCsrMatrix(3, np.zeros(3, np.uint64), [], [])


def test_identity_and_dense():
    a = SparseCsrMatrix.identity(4)
    assert np.array_equal(a.to_dense(), np.eye(4))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built here")
def test_from_triplets_matches_reference_on_random_input():
    ref = Reference()
    rng = np.random.default_rng(3)
    n = 40
    i = rng.integers(0, n, 600)
    j = rng.integers(0, n, 600)
    v = rng.standard_normal(600)
    v[::17] = 0.0
    mine = SparseCsrMatrix.from_coo(n, i, j, v)
    theirs = ref.from_triplets(n, i, j, v)
    assert np.array_equal(mine.row_ptr(), theirs[1])
    assert np.array_equal(mine.col_idx(), theirs[2])
    assert np.allclose(mine.values(), theirs[3], rtol=1e-15, atol=0)
