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


@pytest.mark.parametrize("cfg,nx", [("C4", 64), ("C5", 320)])
def test_streamed_s0_matches_host_stream(nlsp, cfg, nx):
    """nlsp_generate_smoothed_vectors streams S^(0) to the device in 8 M-value
    chunks through pinned staging (several chunks here; C5's clamped edge
    takes the masked scatter path): with no sweeps the device holds exactly
    the reference's Rng stream (the host restatement, pinned to rng.npz)."""
    from paper_2601_20174_b200 import problems
    c = problems.CONFIGS[cfg].scaled(nx=nx)
    pb = problems.generate(c)
    a = pb.csr()
    mask = pb.mask if pb.mask.any() else None
    assert pb.n * c.m > 2 * (1 << 23) and (mask is not None) == (cfg == "C5")
    s = nlsp.generate_smoothed_vectors(a, mask, c.m, 0, c.omega, c.s0_seed).s.numpy()
    ref = problems.smoothed_s0(c.s0_seed, pb.n, c.m, mask)
    assert np.array_equal(s, ref)


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


def test_svd_basis_rejects_nonfinite_and_k_past_rank(nlsp):
    s = np.ones((10, 3))
    s[4, 1] = np.nan
    with pytest.raises(nlsp.ValidationError):
        nlsp.svd_basis(s, 2)
    with pytest.raises(nlsp.ValidationError):  # first_cols: k > min(n, m)
        nlsp.svd_basis(np.random.default_rng(1).standard_normal((10, 3)), 4)
    with pytest.raises(nlsp.ValidationError):
        nlsp.svd_basis(np.random.default_rng(1).standard_normal((3, 10)), 4)


def _svd_vs_oracle(nlsp, oracle, s, k, tol_orth=1e-12):
    p, sig, _ = nlsp.svd_basis(s, k)
    u, sig_o, _, _ = oracle.svd(s)
    r = min(s.shape)
    assert sig.shape == (r,)
    # sigma_j = sqrt(lambda_j) of the Gram: lambda to ~u lambda_0 on both sides
    assert np.abs(sig ** 2 - sig_o ** 2).max() <= 1e-13 * sig_o[0] ** 2
    pg = p.numpy()
    assert np.abs(pg.T @ pg - np.eye(k)).max() <= tol_orth
    return pg, u[:, :k], sig_o


def test_svd_basis_wide_s_matches_reference(nlsp, oracle):
    """m > n: svd_oracle eigensolves S S^T and U is its eigenvectors
    (svd.hpp:161-165, 186, 205), then the sign convention."""
    rng = np.random.default_rng(11)
    s = rng.standard_normal((12, 40)) * np.geomspace(1.0, 0.2, 12)[:, None]
    pg, pr, sig = _svd_vs_oracle(nlsp, oracle, s, 6)
    errs, signs = col_match(pg, pr)
    assert np.all(signs == 1.0)  # same sign convention
    lam = sig ** 2
    gaps = np.array([min(lam[j - 1] - lam[j] if j > 0 else np.inf, lam[j] - lam[j + 1]) for j in range(6)])
    assert np.all(errs <= np.maximum(1e-10, 1e-13 * lam[0] / gaps)), errs


def test_svd_basis_completes_rank_deficient_s(nlsp, oracle):
    """Numerical rank 3 < k = 5: columns past the sigma cutoff come from
    complete_orthonormal (svd.hpp:101-126, 185-203), coordinate vectors
    projected off the solid columns, as in the reference."""
    rng = np.random.default_rng(5)
    s = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 8))
    pg, pr, sig = _svd_vs_oracle(nlsp, oracle, s, 5)
    assert np.all(sig[3:] == 0.0)  # clamped below the Gram's rounding floor
    errs, _ = col_match(pg, pr)
    assert errs[:3].max() <= 1e-10 and errs[3:].max() <= 1e-10, errs


def test_svd_basis_polishes_lost_orthogonality(nlsp, oracle):
    """sigma spread over 1e5: U = S V / sigma loses orthogonality (~u
    sigma_0^2 / sigma_j^2), so the defect exceeds 1e-11 and the Gram-Schmidt
    polish runs (svd.hpp:128-145, :204) — U orthonormal to rounding again."""
    rng = np.random.default_rng(9)
    q = np.linalg.qr(rng.standard_normal((400, 6)))[0]
    v = np.linalg.qr(rng.standard_normal((6, 6)))[0]
    s = (q * np.geomspace(1.0, 1e-5, 6)) @ v.T
    pg, pr, sig = _svd_vs_oracle(nlsp, oracle, s, 6, tol_orth=1e-13)
    errs, _ = col_match(pg, pr)
    lam = sig ** 2
    gaps = np.array([min(lam[j - 1] - lam[j] if j > 0 else np.inf, lam[j] - lam[j + 1] if j < 5 else np.inf)
                     for j in range(6)])
    # columns are determined to ~u lambda_0 / gap_j (both sides alike)
    assert np.all(errs <= np.maximum(1e-10, 1e-12 * lam[0] / gaps)), errs


@pytest.mark.parametrize("cond", [1e4, 1e10, 1e13])
def test_qr_thin_ill_conditioned_basis_matches_reference(nlsp, oracle, cond):
    """qr_thin (qr.hpp:18-45) through the two-level build: CholeskyQR2 for a
    well-conditioned basis, shifted CholeskyQR3 once the Gram's pivots fall
    under 1e-6 ||B||_F (where CholeskyQR2 would lose orthogonality or report a
    spurious rank deficiency). Q matches the reference's two-pass MGS to
    ~u cond(B) per column, and the reference's rank test is kept."""
    from test_gpu_twolevel import tridiag
    rng = np.random.default_rng(int(np.log10(cond)))
    n, k = 300, 8
    u0 = np.linalg.qr(rng.standard_normal((n, k)))[0]
    v0 = np.linalg.qr(rng.standard_normal((k, k)))[0]
    b = (u0 * np.geomspace(1.0, 1.0 / cond, k)) @ v0.T
    a = tridiag(n, nlsp)
    try:
        qr, _ = oracle.qr_thin(b)
    except Exception:  # cond 1e13: the last post-elimination norm < 1e-12 ||B||_F
        with pytest.raises(nlsp.RankDeficiencyError):
            nlsp.TwoLevelPreconditioner(a, b, 2 / 3, 1, 1)
        return
    m = nlsp.TwoLevelPreconditioner(a, b, 2 / 3, 1, 1)
    q = m._export()[0]
    assert np.abs(q.T @ q - np.eye(k)).max() <= 1e-12
    errs, signs = col_match(q, qr)
    assert np.all(signs == 1.0)  # positive diagonal of R on both sides
    assert errs.max() <= max(1e-10, 1e-15 * cond), errs
    # the span: B = Q R exactly up to rounding
    rr = q.T @ b
    assert np.abs(q @ rr - b).max() <= 1e-13 * np.abs(b).max()


def test_qr_thin_rank_test_matches_reference(nlsp, oracle):
    """A column dependent to 1e-14 ||B||_F is rank-deficient for the reference
    (post-elimination norm < 1e-12 ||B||_F) and here; one at 1e-10 is not."""
    from test_gpu_twolevel import tridiag
    rng = np.random.default_rng(3)
    n = 200
    a = tridiag(n, nlsp)
    base = rng.standard_normal((n, 4))
    for eps, deficient in [(1e-14, True), (1e-10, False)]:
        b = np.hstack([base, (base @ [1.0, -2.0, 0.5, 0.25])[:, None] + eps * rng.standard_normal((n, 1))])
        try:
            oracle.qr_thin(b)
            ref_def = False
        except Exception:
            ref_def = True
        assert ref_def == deficient
        if deficient:
            with pytest.raises(nlsp.RankDeficiencyError):
                nlsp.TwoLevelPreconditioner(a, b, 2 / 3, 1, 1)
        else:
            m = nlsp.TwoLevelPreconditioner(a, b, 2 / 3, 1, 1)
            q = m._export()[0]
            assert np.abs(q.T @ q - np.eye(5)).max() <= 1e-12


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
