"""GPU parity of the building blocks through the C-ABI: SpMV, Jacobi sweeps,
block smoothing, the SVD basis, QR/Galerkin/Cholesky of the two-level build.
Mirrors the reference's test_linalg.cpp / test_smoothing.cpp cases and compares
with the CPU oracle (pinned to the reference) and the golden fixtures."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import col_match, csr_from_golden, golden, random_spd_sparse

pytestmark = pytest.mark.gpu


# --------------------------------------------------------------- sparse.hpp --
def test_spmv_identity_passes_through(nlsp):
    a = nlsp.SparseCsrMatrix.identity(3)
    x = np.array([1.0, 2.0, 3.0])
    assert np.array_equal(nlsp.spmv(a, x), x)


def test_spmv_stencil_on_constant_vector(nlsp):
    a = nlsp.SparseCsrMatrix.from_triplets(2, [(0, 0, 2.0), (0, 1, -1.0), (1, 0, -1.0), (1, 1, 2.0)])
    assert np.array_equal(nlsp.spmv(a, np.ones(2)), golden("kat")["stencil_y"])


def test_spmv_matches_dense_and_oracle(nlsp, oracle):
    # Spmv.MatchesDenseOracle: rel < 1e-14 (test_linalg.cpp:73-86)
    rng = np.random.default_rng(42)
    n = 50
    mask = rng.random((n, n)) < 0.15
    ii, jj = np.nonzero(mask)
    a = nlsp.SparseCsrMatrix.from_coo(n, ii, jj, rng.standard_normal(ii.size))
    x = rng.standard_normal(n)
    y = nlsp.spmv(a, x)
    ref = a.to_dense() @ x
    assert np.linalg.norm(y - ref) < 1e-14 * np.linalg.norm(ref) + 1e-300
    yo = oracle.spmv((n, a.row_ptr(), a.col_idx(), a.values()), x)
    assert np.linalg.norm(y - yo) < 1e-14 * np.linalg.norm(yo)


def test_spmv_dimension_mismatch(nlsp):
    with pytest.raises(nlsp.ValidationError):
        nlsp.spmv(nlsp.SparseCsrMatrix.identity(3), np.array([1.0, 2.0]))


def test_spmv_long_and_empty_rows(nlsp, oracle):
    # rows longer than one 8-lane pass, empty rows, a dense row
    rng = np.random.default_rng(9)
    n = 300
    rows, cols = [], []
    for i in range(n):
        ln = [0, 1, 7, 8, 9, 17, 40, 299][i % 8]
        c = rng.choice(n, size=ln, replace=False) if ln else []
        rows += [i] * len(c)
        cols += list(c)
    a = nlsp.SparseCsrMatrix.from_coo(n, rows, cols, rng.standard_normal(len(rows)))
    x = rng.standard_normal(n)
    y = nlsp.spmv(a, x)
    yo = oracle.spmv((n, a.row_ptr(), a.col_idx(), a.values()), x)
    assert np.abs(y - yo).max() <= 1e-13 * np.abs(yo).max()


def test_csr_upload_rejects_broken_invariants(nlsp):
    from paper_2601_20174_b200 import _lib as L
    import ctypes as C
    ctx = nlsp.default_context()
    lib = L.gpu_lib()
    h = C.c_void_p()
    rp = np.array([0, 2, 3], np.uint64)
    for ci in (np.array([1, 0, 1], np.uint64), np.array([0, 5, 1], np.uint64),
               np.array([0, 0, 1], np.uint64)):
        v = np.ones(3)
        st = lib.nlsp_csr_upload(ctx.handle, 2, 3, L.u64ptr(rp), L.u64ptr(ci), L.dptr(v), C.byref(h))
        assert st == L.NLSP_E_VALIDATION


# ------------------------------------------------------------ smoothing.hpp --
def test_jacobi_identity_contracts(nlsp):
    a = nlsp.SparseCsrMatrix.identity(5)
    sm = nlsp.JacobiSmoother(a, 0.3)
    x = np.array([1.0, -2.0, 3.0, 0.5, -1.5])
    sm.sweep(a, x, np.zeros(5))
    assert np.allclose(x, 0.7 * np.array([1.0, -2.0, 3.0, 0.5, -1.5]), atol=1e-15)
    assert np.array_equal(x, golden("kat")["jacobi_eye_x"])


def test_jacobi_full_omega_solves_identity(nlsp):
    a = nlsp.SparseCsrMatrix.identity(4)
    sm = nlsp.JacobiSmoother(a, 1.0)
    x = np.zeros(4)
    target = np.array([2.0, -1.0, 0.0, 5.0])
    sm.sweep(a, x, target)
    assert np.array_equal(x, target)


def test_jacobi_error_decreases_in_d_norm(nlsp):
    rng = np.random.default_rng(77)
    a, dense = random_spd_sparse(30, rng, density=0.1)
    sm = nlsp.JacobiSmoother(a, 0.66)
    x_star = rng.standard_normal(30)
    b = dense @ x_star
    x = np.zeros(30)
    d = np.diag(dense)
    prev = np.sqrt(np.sum(d * (x - x_star) ** 2))
    for _ in range(50):
        sm.sweep(a, x, b)
        cur = np.sqrt(np.sum(d * (x - x_star) ** 2))
        assert cur <= prev * (1 + 1e-12)
        prev = cur
    assert prev < 1e-2


def test_jacobi_rejects(nlsp):
    a = nlsp.SparseCsrMatrix.from_triplets(2, [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0)])
    with pytest.raises(nlsp.NumericError):
        nlsp.JacobiSmoother(a, 0.66)
    with pytest.raises(nlsp.ValidationError):
        nlsp.JacobiSmoother(nlsp.SparseCsrMatrix.identity(2), 1.5)


def test_jacobi_sweeps_match_oracle(nlsp, oracle):
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    rng = np.random.default_rng(4)
    x0 = rng.standard_normal(a.dim())
    b = rng.standard_normal(a.dim())
    x = x0.copy()
    nlsp.JacobiSmoother(a, 0.66).sweep(a, x, b, sweeps=7)
    xo = oracle.jacobi_sweep((a.dim(), a.row_ptr(), a.col_idx(), a.values()), 0.66, 7, x0, b)
    assert np.abs(x - xo).max() <= 1e-13 * np.abs(xo).max()


@pytest.mark.parametrize("name", ["c1_default", "scaled_C2", "scaled_C3", "scaled_C4", "scaled_C5"])
def test_smoothed_vectors_match_reference(nlsp, name):
    d = golden(name)
    a = csr_from_golden(d)
    mask = d["mask"] if d["mask"].any() else None
    sv = nlsp.generate_smoothed_vectors(a, mask, int(d["m"]), int(d["s1"]), float(d["omega"]),
                                        int(d["s0_seed"]))
    s = sv.s.numpy()
    # S^(0) is bit-identical (same Rng stream); the sweeps round like the
    # contracted reference build
    assert np.abs(s - d["S"]).max() <= 1e-13 * np.abs(d["S"]).max()
    if mask is not None:
        assert np.all(s[mask.astype(bool)] == 0.0)  # SmoothedVectors.BoundaryRowsStayExactlyZero


@pytest.mark.parametrize("name,m", [("scaled_C4", 128), ("scaled_C3", 96), ("c1_default", 80)])
def test_wide_smoothing_diagonal_form_matches_csr_and_reference(nlsp, oracle, name, m):
    """m > 64 on a constant-coefficient stencil runs the diagonal-form block
    sweep (k_block_sweep_dia): bitwise the CSR block sweep (upload with
    NLSP_DIA=0), and within rounding of the reference's smoothing."""
    import os
    d = golden(name)
    a = csr_from_golden(d)
    assert a.device().format()[0] == 1
    os.environ["NLSP_DIA"] = "0"
    try:
        a_csr = csr_from_golden(d)
        assert a_csr.device().format()[0] == 0
    finally:
        os.environ.pop("NLSP_DIA", None)
    s_dia = nlsp.generate_smoothed_vectors(a, None, m, 10, 2 / 3, 11).s.numpy()
    s_csr = nlsp.generate_smoothed_vectors(a_csr, None, m, 10, 2 / 3, 11).s.numpy()
    assert np.array_equal(s_dia, s_csr)
    so = oracle.generate_smoothed_vectors((a.dim(), a.row_ptr(), a.col_idx(), a.values()), None,
                                          m, 10, 2 / 3, 11)
    assert np.abs(s_dia - so).max() <= 1e-13 * np.abs(so).max()


def test_zero_sweeps_returns_raw_gaussians(nlsp, oracle):
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    s1 = nlsp.generate_smoothed_vectors(a, d["mask"], 8, 0, 0.66, 5).s.numpy()
    s2 = nlsp.generate_smoothed_vectors(a, d["mask"], 8, 0, 0.66, 5).s.numpy()
    so = oracle.generate_smoothed_vectors((a.dim(), a.row_ptr(), a.col_idx(), a.values()), d["mask"],
                                          8, 0, 0.66, 5)
    assert np.array_equal(s1, s2) and np.array_equal(s1, so)


# ------------------------------------------------------------------ svd.hpp --
def test_svd_basis_diagonal_case(nlsp):
    s = np.zeros((3, 2))
    s[0, 0], s[1, 1] = 3.0, 2.0
    p, sig, _ = nlsp.svd_basis(s, 2)
    assert np.allclose(sig, [3.0, 2.0], atol=1e-12)
    pu = p.numpy()
    assert abs(abs(pu[0, 0]) - 1.0) < 1e-10 and pu[0, 0] >= 0.0


def test_svd_basis_random_matches_oracle(nlsp, oracle):
    rng = np.random.default_rng(5)
    s = rng.standard_normal((400, 12))
    p, sig, _ = nlsp.svd_basis(s, 6)
    u, sig_o, _, _ = oracle.svd(s)
    assert np.abs(sig - sig_o).max() <= 1e-12 * sig_o[0]
    errs, signs = col_match(p.numpy(), u[:, :6])
    assert errs.max() <= 1e-10 and np.all(signs == 1.0)  # same sign convention


def test_svd_basis_rejects_nonfinite_and_wide(nlsp):
    s = np.ones((10, 3))
    s[4, 1] = np.nan
    with pytest.raises(nlsp.ValidationError):
        nlsp.svd_basis(s, 2)
    with pytest.raises(nlsp.ValidationError):
        nlsp.svd_basis(np.ones((3, 10)), 2)
    with pytest.raises(nlsp.ValidationError):
        nlsp.svd_basis(np.random.default_rng(1).standard_normal((10, 3)), 4)


@pytest.mark.parametrize("name", ["c1_default", "scaled_C2", "scaled_C3", "scaled_C4", "scaled_C5"])
def test_svd_basis_matches_reference(nlsp, name):
    d = golden(name)
    k = int(d["k"])
    p, sig, _ = nlsp.svd_basis(d["S"], k)
    assert np.abs(sig - d["sigma"]).max() <= 1e-12 * d["sigma"][0]
    pg = p.numpy()
    errs, signs = col_match(pg, d["P"])
    # per column to 1e-10 where the singular gap allows it; the
    # subspace itself always (principal angles)
    lam = d["sigma"] ** 2
    gaps = np.array([min(lam[j - 1] - lam[j] if j > 0 else np.inf, lam[j] - lam[j + 1])
                     for j in range(k)])
    # first-order rotation of column j ~ (Gram rounding) / eigen-gap: columns
    # whose gap allows 1e-10 must meet it; the others are gap-limited
    bound = np.maximum(1e-10, 1e-13 * lam[0] / gaps)
    assert np.all(errs <= bound), (errs, bound)
    # largest principal angle via its sine, ||(I - P_g P_g^T) P_ref||_2 (arccos of
    # a cosine near 1 is ill-conditioned); the k-dimensional subspace is limited
    # only by the gap after column k
    sin_max = np.linalg.norm(d["P"] - pg @ (pg.T @ d["P"]), 2)
    assert sin_max <= max(1e-10, 1e-13 * lam[0] / (lam[k - 1] - lam[k]))


@pytest.mark.parametrize("m,k", [(200, 20), (256, 130)])
def test_svd_basis_wide_gram_blocks(nlsp, oracle, m, k):
    """m > 128: the Gram is tiled over 128-column blocks and the eigensolver
    works out of global scratch."""
    rng = np.random.default_rng(m)
    # a spread spectrum so every column is well separated
    s = rng.standard_normal((3000, m)) * np.geomspace(1.0, 1e-2, m)
    p, sig, sweeps = nlsp.svd_basis(s, k)
    u, sig_o, _, _ = oracle.svd(s)
    assert np.abs(sig - sig_o).max() <= 1e-11 * sig_o[0]
    errs, _ = col_match(p.numpy(), u[:, :k])
    assert errs.max() <= 1e-9
