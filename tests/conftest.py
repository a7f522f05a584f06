"""Shared fixtures. `-m gpu` tests need a B200 and call the product through the
C-ABI (libnlsp_gpu.so); everything else runs on the CPU."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs through the C-ABI")
    config.addinivalue_line("markers", "slow: full BASELINE.json sizes")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def nlsp():
    """The product package with a live CUDA context (gpu tests only)."""
    from paper_2601_20174_b200 import nlsp as N
    N.default_context()
    return N


def csr_from_golden(d, prefix=""):
    from paper_2601_20174_b200.nlsp import SparseCsrMatrix
    n = int(d[prefix + "n"])
    return SparseCsrMatrix(n, d[prefix + "row_ptr"] if prefix == "" else d[prefix + "rp"],
                           d[prefix + "col_idx"] if prefix == "" else d[prefix + "ci"],
                           d[prefix + "values"] if prefix == "" else d[prefix + "v"])


def random_spd_sparse(n, rng, density=0.08, shift=6.0):
    """test_two_level.cpp:17-28 shape: symmetric random off-diagonals, diagonal
    shift + U[0,1) (numpy RNG; the matrix is the input, both sides see it)."""
    from paper_2601_20174_b200.nlsp import SparseCsrMatrix
    dense = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    pick = rng.random(iu[0].size) < density
    dense[iu[0][pick], iu[1][pick]] = rng.standard_normal(pick.sum())
    dense = dense + dense.T + np.diag(shift + rng.random(n))
    ii, jj = np.nonzero(dense)
    return SparseCsrMatrix.from_coo(n, ii, jj, dense[ii, jj]), dense


def col_match(p_gpu, p_ref):
    """max over columns of min_s ||p_gpu[:, j] - s p_ref[:, j]||_inf / ||p_ref[:, j]||_inf
    (SURVEY §8c P metric) and the per-column signs."""
    errs, signs = [], []
    for j in range(p_ref.shape[1]):
        den = np.abs(p_ref[:, j]).max()
        e_pos = np.abs(p_gpu[:, j] - p_ref[:, j]).max() / den
        e_neg = np.abs(p_gpu[:, j] + p_ref[:, j]).max() / den
        errs.append(min(e_pos, e_neg))
        signs.append(1.0 if e_pos <= e_neg else -1.0)
    return np.array(errs), np.array(signs)


def gap_bounds(sigma, k):
    """Per-column P bound of SURVEY §8c: 1e-10, or the gap-limited
    1e-13 lambda_0 / gap_j where lambda = sigma^2 (eigenvalues of the Gram)."""
    lam = np.asarray(sigma, np.float64) ** 2
    gaps = np.array([min(lam[j - 1] - lam[j] if j > 0 else np.inf,
                         lam[j] - lam[j + 1] if j + 1 < lam.size else np.inf) for j in range(k)])
    return np.maximum(1e-10, 1e-13 * lam[0] / gaps), np.maximum(1e-10, 1e-13 * lam[0] / gaps.min())


def check_basis_coarse_sketch(d, basis, coarse, k):
    """P (up to column sign) and A_c against a golden holding only sketches of
    the reference's basis_ (tests/golden/sketch.py): its row sample entrywise
    (relative to the column's largest |entry|) and its Gaussian sketch (2-norm
    relative; the JL factor is covered by 2x). Returns the per-column errors."""
    import sys
    sys.path.insert(0, GOLDEN)
    from sketch import sketch
    bound, sub = gap_bounds(d["sigma"], k)
    idx, val = d["basis_argmax_idx"], d["basis_argmax_val"]
    signs = np.sign(basis[idx, np.arange(k)]) * np.sign(val)
    signs[signs == 0] = 1.0
    rows = d["rows"]
    err_rows = np.abs(basis[rows] * signs - d["basis_rows"]).max(axis=0) / np.abs(val)
    sk = sketch(basis * signs)
    ref_sk = d["basis_sketch"]
    err_sk = np.linalg.norm(sk - ref_sk, axis=0) / np.linalg.norm(ref_sk, axis=0)
    assert np.all(err_rows <= bound), (err_rows, bound)
    assert np.all(err_sk <= 2 * bound), (err_sk, bound)
    dac = np.diag(signs)
    ac = dac @ coarse @ dac
    ac_ref = d["coarse"]
    err_ac = np.abs(ac - ac_ref).max() / np.abs(ac_ref).max()
    assert err_ac <= sub, (err_ac, sub)
    return err_rows, err_sk, err_ac
