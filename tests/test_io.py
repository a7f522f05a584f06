"""The on-disk input path without a GPU: libnlsp_io.so
(include/nlsp_io.h) against what the REFERENCE's own loaders produced on the
same files (tests/golden/io, made by tests/golden/make_io_golden.py):

* load_matrix_market (sparse.hpp:168-194) on 28 edge-case files — same status
  class and message, same CSR bits (ordering, duplicate sums, dropped zeros,
  symmetric mirroring, istream token rules: signs, exponents, split lines,
  CRLF/tabs, nan / overflow / garbage rejected);
* load_instance (instance_io.hpp:137-185) on instance directories of all three
  PDE families — every array bit-identical;
* save_matrix_market (sparse.hpp:148-166) reproduces the reference-written
  matrix.mtx byte for byte, and save -> load round-trips.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2601_20174_b200 import instance_io as io
from paper_2601_20174_b200 import nlsp

IO = os.path.join(GOLDEN, "io")
MTX = np.load(os.path.join(IO, "mtx_expected.npz"))
INST = np.load(os.path.join(IO, "instances.npz"))


@pytest.mark.parametrize("case", [str(c) for c in MTX["names"]])
def test_matrix_market_matches_reference(case):
    path = os.path.join(IO, "mtx", case + ".mtx")
    st = int(MTX[f"{case}__status"])
    if st == 0:
        a = io.load_matrix_market(path)
        assert a.dim() == int(MTX[f"{case}__n"])
        assert np.array_equal(a.row_ptr(), MTX[f"{case}__rp"])
        assert np.array_equal(a.col_idx(), MTX[f"{case}__ci"])
        assert np.array_equal(a.values().view(np.uint64), MTX[f"{case}__v"].view(np.uint64))
    else:
        exc = io.IoError if st == 8 else nlsp.ValidationError
        with pytest.raises(exc) as ei:
            io.load_matrix_market(path)
        msg = str(MTX[f"{case}__message"]).replace("<dir>", os.path.join(IO, "mtx"))
        assert str(ei.value) == msg


def test_missing_file_is_io_error():
    with pytest.raises(io.IoError, match="cannot open for read"):
        io.load_matrix_market(os.path.join(IO, "does_not_exist.mtx"))
    with pytest.raises(io.IoError, match="cannot open for read"):
        io.load_instance(os.path.join(IO, "no_such_instance"))


@pytest.mark.parametrize("name", [str(c) for c in INST["names"]])
def test_instance_matches_reference(name):
    inst = io.load_instance(os.path.join(IO, name))
    g = lambda k: INST[f"{name}__{k}"]  # noqa: E731
    assert io.FAMILIES.index(inst.family) == int(g("family"))
    assert inst.grid_n == int(g("grid_n")) and inst.seed == int(g("seed"))
    assert inst.jitter == float(g("jitter")) and inst.alpha == float(g("alpha"))
    a = inst.matrix
    assert a.dim() == int(g("n"))
    assert np.array_equal(a.row_ptr(), g("rp")) and np.array_equal(a.col_idx(), g("ci"))
    assert np.array_equal(a.values().view(np.uint64), g("v").view(np.uint64))
    assert np.array_equal(inst.rhs.view(np.uint64), g("rhs").view(np.uint64))
    assert np.array_equal(inst.boundary_mask, g("mask"))
    assert np.array_equal(inst.vertices, g("vertices"))
    assert np.array_equal(inst.triangles, g("triangles"))
    assert np.array_equal(inst.coefficients, g("coefficients"))
    # Dirichlet rows are identity rows (fem.hpp:184-200)
    rp = a.row_ptr().astype(np.int64)
    for i in np.flatnonzero(inst.boundary_mask)[:20]:
        assert rp[i + 1] - rp[i] == 1 and a.col_idx()[rp[i]] == i and a.values()[rp[i]] == 1.0


def test_save_reproduces_reference_file(tmp_path):
    src = os.path.join(IO, "inst_diffusion_n8", "matrix.mtx")
    a = io.load_matrix_market(src)
    out = tmp_path / "m.mtx"
    io.save_matrix_market(a, str(out))
    assert out.read_bytes() == open(src, "rb").read()
    b = io.load_matrix_market(str(out))
    assert np.array_equal(a.values(), b.values()) and np.array_equal(a.col_idx(), b.col_idx())


def test_round_trip_random_symmetric(tmp_path):
    rng = np.random.default_rng(3)
    n = 200
    i = rng.integers(0, n, 900)
    j = rng.integers(0, n, 900)
    v = rng.standard_normal(900) * 10.0 ** rng.integers(-300, 300, 900)
    ii, jj = np.concatenate([i, j, np.arange(n)]), np.concatenate([j, i, np.arange(n)])
    vv = np.concatenate([v, v, np.full(n, 5.0)])
    a = nlsp.SparseCsrMatrix.from_coo(n, ii, jj, vv)
    out = tmp_path / "r.mtx"
    io.save_matrix_market(a, str(out))
    b = io.load_matrix_market(str(out))
    assert np.array_equal(a.row_ptr(), b.row_ptr()) and np.array_equal(a.col_idx(), b.col_idx())
    assert np.array_equal(a.values().view(np.uint64), b.values().view(np.uint64))


def test_bad_manifest(tmp_path):
    import shutil
    d = tmp_path / "inst"
    shutil.copytree(os.path.join(IO, "inst_diffusion_n8"), d)
    (d / "manifest.txt").write_text("family = diffusion\nN = 8\n")
    with pytest.raises(nlsp.ValidationError, match="manifest: missing key seed"):
        io.load_instance(str(d))
    (d / "manifest.txt").write_text("family = elasticity\nN = 8\nseed = 1\njitter = 0\n")
    with pytest.raises(nlsp.ValidationError, match="unknown PDE family: elasticity"):
        io.load_instance(str(d))
    (d / "manifest.txt").write_text("no equals sign here\n")
    with pytest.raises(nlsp.ValidationError, match="manifest: bad line"):
        io.load_instance(str(d))


def test_wrapping_dimension_rejected_before_allocation(tmp_path):
    """A size line of -1 (istream >> size_t wraps it to 2^64 - 1) or any
    dimension past the device limit is a ValidationError, not a wrapped
    row_ptr size (heap corruption in a naive from_triplets)."""
    for line in ("-1 -1 0", "18446744073709551615 18446744073709551615 0", "2147483648 2147483648 1\n1 1 1.0"):
        p = tmp_path / "big.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real symmetric\n" + line + "\n")
        with pytest.raises(nlsp.ValidationError, match="dimension"):
            io.load_matrix_market(str(p))
