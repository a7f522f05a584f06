"""Pins the CPU oracle (oracle/nlsp_oracle.c) before it is trusted:
  * against the golden fixtures produced by the reference itself
    (tests/golden/make_golden.py over oracle/_ref): bitwise for the
    -ffp-contract=off build, within rounding for the default build;
  * against every hand-checked case of the reference's unit tests;
  * against the live reference build when /root/reference is present here.
CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle.oracle import Oracle, OracleError, Reference, reference_available


def csr(d):
    return (int(d["n"]), d["row_ptr"], d["col_idx"], d["values"])


# ------------------------------------------------------------------ rng.hpp --
def test_rng_streams_match_reference(oracle):
    g = golden("rng")
    mix = [oracle.mix_seed(s, t) for s, t in [(0, 0), (7, 0x736d6f6f), (2601, 0x726873),
                                              (2**64 - 1, 12345)]]
    assert np.array_equal(np.array(mix, dtype=np.uint64), g["mix"])
    assert np.array_equal(oracle.rng_u64(5, 700), g["u64_seed5"])
    assert np.array_equal(oracle.rng_normal(5, 1001), g["normal_seed5"])
    assert np.array_equal(oracle.rng_normal(oracle.mix_seed(7, 0x736d6f6f), 4097), g["normal_seed_smoo7"])
    assert np.array_equal(oracle.rng_uniform(9, 513, -1.0, 1.0), g["uniform_seed9"])


# ------------------------------------------------------- hand-checked cases --
def test_cholesky_hand_checked(oracle):
    # Cholesky.HandChecked2x2 (test_linalg.cpp:276-285)
    x = oracle.cholesky_solve(np.array([[4.0, 2.0], [2.0, 3.0]]), np.array([4.0, 2.0]))
    assert np.allclose(x, [1.0, 0.0], atol=1e-14)
    assert np.array_equal(x, golden("kat")["chol_2x2_x"])


def test_cholesky_rejects(oracle):
    with pytest.raises(OracleError) as e:
        oracle.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.kind == "not_spd"
    with pytest.raises(OracleError) as e:
        oracle.cholesky(np.array([[2.0, 1.0], [0.5, 2.0]]))
    assert e.value.kind == "not_spd"


def test_qr_hand_checked(oracle):
    q, r = oracle.qr_thin(np.array([[3.0], [4.0]]))
    assert np.allclose(q[:, 0], [0.6, 0.8], atol=1e-15) and abs(r[0, 0] - 5.0) < 1e-15
    g = golden("kat")
    assert np.array_equal(q, g["qr_3_4_q"]) and np.array_equal(r, g["qr_3_4_r"])


def test_qr_rank_deficiency(oracle):
    m = np.array([[i + 1.0, 2.0 * (i + 1)] for i in range(4)])
    with pytest.raises(OracleError) as e:
        oracle.qr_thin(m)
    assert e.value.kind == "rank_deficient"


def test_svd_diagonal(oracle):
    s = np.zeros((3, 2))
    s[0, 0], s[1, 1] = 3.0, 2.0
    u, sig, _, _ = oracle.svd(s)
    assert np.allclose(sig, [3.0, 2.0], atol=1e-12)
    assert u[0, 0] >= 0.0 and abs(abs(u[0, 0]) - 1.0) < 1e-10
    g = golden("kat")
    assert np.array_equal(u, g["svd_diag_u"]) and np.array_equal(sig, g["svd_diag_sigma"])


def test_svd_reconstructs(oracle):
    rng = np.random.default_rng(5)
    s = rng.standard_normal((20, 8))
    u, sig, v, _ = oracle.svd(s)
    assert np.linalg.norm(u * sig @ v.T - s) < 1e-9 * np.linalg.norm(s)
    assert oracle.orthonormality_defect(u) < 1e-10
    assert np.all(np.diff(sig) <= 0)
    wide = rng.standard_normal((8, 20))
    u, sig, v, _ = oracle.svd(wide)
    assert np.linalg.norm(u * sig @ v.T - wide) < 1e-9 * np.linalg.norm(wide)


def test_spmv_stencil_and_dedup(oracle):
    g = golden("kat")
    a = (2, np.array([0, 2, 4], np.uint64), np.array([0, 1, 0, 1], np.uint64),
         np.array([2.0, -1.0, -1.0, 2.0]))
    assert np.array_equal(oracle.spmv(a, np.ones(2)), g["stencil_y"])
    # SparseCsr.TripletsDeduplicatedAndSorted through the reference
    assert list(g["dedup_rp"]) == [0, 2, 2] and list(g["dedup_ci"]) == [0, 1]
    assert list(g["dedup_v"]) == [2.0, 1.5]


def test_jacobi_identity_contracts(oracle):
    eye = (5, np.arange(6, dtype=np.uint64), np.arange(5, dtype=np.uint64), np.ones(5))
    x = oracle.jacobi_sweep(eye, 0.3, 1, np.array([1.0, -2.0, 3.0, 0.5, -1.5]), np.zeros(5))
    assert np.allclose(x, 0.7 * np.array([1.0, -2.0, 3.0, 0.5, -1.5]), atol=1e-15)
    assert np.array_equal(x, golden("kat")["jacobi_eye_x"])


def test_jacobi_rejects(oracle):
    a = (2, np.array([0, 2, 3], np.uint64), np.array([0, 1, 0], np.uint64), np.array([1.0, 1.0, 1.0]))
    with pytest.raises(OracleError) as e:
        oracle.inv_diag(a, 0.66)
    assert e.value.kind == "numeric"
    eye = (2, np.arange(3, dtype=np.uint64), np.arange(2, dtype=np.uint64), np.ones(2))
    with pytest.raises(OracleError) as e:
        oracle.inv_diag(eye, 1.5)
    assert e.value.kind == "validation"


def test_pcg_identity_one_iteration(oracle):
    eye = (10, np.arange(11, dtype=np.uint64), np.arange(10, dtype=np.uint64), np.ones(10))
    r = oracle.pcg(eye, np.full(10, 2.5), 0, None, 1e-10, 100)
    assert r.converged and r.iterations == 1 and np.allclose(r.x, 2.5, atol=1e-12)
    with pytest.raises(OracleError) as e:
        oracle.pcg(eye, np.zeros(10), 0, None, 1e-6, 10)
    assert e.value.kind == "validation"


# ------------------------------------------------------- golden pipelines ---
@pytest.mark.parametrize("name", ["c1_strict", "c1_default", "scaled_C2", "scaled_C3",
                                  "scaled_C4", "scaled_C5"])
def test_pipeline_against_reference(oracle, name):
    d = golden(name)
    a = csr(d)
    mask = d["mask"] if d["mask"].any() else None
    k, m = int(d["k"]), int(d["m"])
    s = oracle.generate_smoothed_vectors(a, mask, m, int(d["s1"]), float(d["omega"]), int(d["s0_seed"]))
    u, sig, _, sweeps = oracle.svd(s)
    p = np.ascontiguousarray(u[:, :k])
    t = oracle.twolevel(a, p, float(d["omega"]), int(d["nu1"]), int(d["nu2"]))
    basis, chol, coarse = t.export()
    res = oracle.pcg(a, d["rhs"], 2, t, float(d["delta"]), 10 * int(d["n"]))
    z = t.apply(d["r_probe"])
    if name.endswith("strict"):
        # sequential-rounding reference build: bitwise everywhere
        for mine, theirs in [(s, d["S"]), (sig, d["sigma"]), (p, d["P"]), (basis, d["basis"]),
                             (chol, d["chol"]), (coarse, d["coarse"]), (res.x, d["x"]),
                             (res.history, d["history"]), (z, d["z_probe"])]:
            assert np.array_equal(mine, theirs)
        assert res.iterations == int(d["iterations"]) and sweeps == int(d["eigh_sweeps"])
        return
    # default (-O3 -march) reference build: same algorithm, contracted rounding
    assert np.abs(s - d["S"]).max() <= 1e-13 * np.abs(d["S"]).max()
    assert np.abs(sig - d["sigma"]).max() <= 1e-12 * sig[0]
    assert np.abs(coarse - d["coarse"]).max() <= 1e-10 * np.abs(d["coarse"]).max()
    assert abs(res.iterations - int(d["iterations"])) <= 2
    assert res.converged and bool(d["converged"])
    assert np.linalg.norm(res.x - d["x"]) <= 1e-9 * np.linalg.norm(d["x"])
    assert np.linalg.norm(z - d["z_probe"]) <= 1e-12 * np.linalg.norm(d["z_probe"])


def test_fem_instance_against_reference(oracle):
    d = golden("fem_diffusion")
    a = csr(d)
    s = oracle.generate_smoothed_vectors(a, d["mask"], 16, 10, 0.66, 29)
    assert np.abs(s - d["S"]).max() <= 1e-13 * np.abs(d["S"]).max()
    u = np.ascontiguousarray(oracle.svd(s)[0][:, :8])
    t = oracle.twolevel(a, u, 0.66, 5, 5)
    two = oracle.pcg(a, d["rhs"], 2, t, 1e-6, 10 * int(d["n"]))
    plain = oracle.pcg(a, d["rhs"], 0, None, 1e-6, 10 * int(d["n"]))
    # fixtures come from the default (contracted) build: iteration counts +-2
    assert abs(two.iterations - int(d["iterations"])) <= 2
    assert abs(plain.iterations - int(d["plain_iterations"])) <= 2
    assert two.iterations < plain.iterations and two.true_relative_residual <= 1e-5
    jac = oracle.pcg(a, d["rhs"], 1, None, 1e-8, 5000)
    assert abs(jac.iterations - int(d["jacobi_iterations"])) <= 2
    assert len(jac.history) == jac.iterations and jac.history[-1] < 1e-8


def test_random_spd_against_reference(oracle):
    d = golden("random_spd")
    for t in range(int(d["trials"])):
        a = (int(d[f"t{t}_n"]), d[f"t{t}_rp"], d[f"t{t}_ci"], d[f"t{t}_v"])
        m0 = oracle.twolevel(a, d[f"t{t}_basis_in"], 0.66, 0, 0)
        m2 = oracle.twolevel(a, d[f"t{t}_basis_in"], 0.66, 2, 2)
        b0, _, c0 = m0.export()
        assert np.abs(b0 - d[f"t{t}_basis"]).max() <= 1e-13
        assert np.abs(c0 - d[f"t{t}_coarse"]).max() <= 1e-12 * np.abs(c0).max()
        assert np.allclose(m0.apply(d[f"t{t}_r"]), d[f"t{t}_z0"], rtol=1e-12, atol=1e-13)
        assert np.allclose(m2.apply(d[f"t{t}_r"]), d[f"t{t}_z2"], rtol=1e-12, atol=1e-13)


# ----------------------------------------- live reference (where it exists) --
@pytest.mark.skipif(not reference_available(strict=True), reason="oracle/_ref not built here")
def test_oracle_bitwise_equals_strict_reference_on_random_cases():
    o, r = Oracle(), Reference(strict=True)
    rng = np.random.default_rng(77)
    for trial in range(5):
        n = int(rng.integers(30, 90))
        dense = np.zeros((n, n))
        iu = np.triu_indices(n, 1)
        pick = rng.random(iu[0].size) < 0.1
        dense[iu[0][pick], iu[1][pick]] = rng.standard_normal(pick.sum())
        dense = dense + dense.T + np.diag(6.0 + rng.random(n))
        ii, jj = np.nonzero(dense)
        a = r.from_triplets(n, ii, jj, dense[ii, jj])
        s_o = o.generate_smoothed_vectors(a, None, 12, 5, 0.66, trial)
        s_r = r.generate_smoothed_vectors(a, None, 12, 5, 0.66, trial)
        assert np.array_equal(s_o, s_r)
        p = np.ascontiguousarray(o.svd(s_o)[0][:, :5])
        t_o, t_r = o.twolevel(a, p, 0.66, 1, 2), r.twolevel(a, p, 0.66, 1, 2)
        (b_o, l_o, c_o), (b_r, l_r, _) = t_o.export(), t_r.export()
        assert np.array_equal(b_o, b_r) and np.array_equal(l_o, l_r)
        assert np.array_equal(c_o, r.galerkin(t_r))
        b = rng.standard_normal(n)
        ro, rr = o.pcg(a, b, 2, t_o, 1e-10, 500), r.pcg(a, b, 2, t_r, 1e-10, 500)
        assert ro.iterations == rr.iterations and np.array_equal(ro.x, rr.x)
