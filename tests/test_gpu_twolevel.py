"""GPU parity of the two-level operator and the PCG loop through the C-ABI.
Mirrors tests/unit/test_two_level.cpp and acceptance C05/C06 of the reference,
and compares every configuration family with the reference's own outputs
(golden fixtures) and the CPU oracle: iterations +-2, true residual,
||x - x_ref|| / ||x_ref|| <= 1e-9, P and A_c to 1e-10."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import col_match, csr_from_golden, golden, random_spd_sparse

pytestmark = pytest.mark.gpu


def orthonormal(n, k, rng):
    return np.linalg.qr(rng.standard_normal((n, k)))[0]


def tridiag(n, nlsp):
    t = []
    for i in range(n):
        t.append((i, i, 2.0))
        if i + 1 < n:
            t += [(i, i + 1, -1.0), (i + 1, i, -1.0)]
    return nlsp.SparseCsrMatrix.from_triplets(n, t)


# ------------------------------------------------------ test_two_level.cpp --
def test_identity_basis_gives_principal_submatrix(nlsp):
    rng = np.random.default_rng(3)
    a, dense = random_spd_sparse(12, rng)
    e = np.zeros((12, 4))
    e[np.arange(4), np.arange(4)] = 1.0
    m = nlsp.TwoLevelPreconditioner(a, e, 0.66, 0, 0)
    y = np.array([1.0, -2.0, 0.5, 3.0])
    uy = np.zeros(12)
    uy[:4] = y
    rhs = nlsp.spmv(a, uy)
    expect = np.linalg.solve(dense[:4, :4], rhs[:4])
    z = m.apply(a, rhs)
    assert np.allclose(z[:4], expect, atol=1e-10)
    assert np.allclose(z[4:], 0.0, atol=1e-12)


def test_empty_coarse_space_rejected(nlsp):
    rng = np.random.default_rng(5)
    a, _ = random_spd_sparse(8, rng)
    with pytest.raises(nlsp.ValidationError):
        nlsp.TwoLevelPreconditioner(a, np.zeros((8, 0)), 0.66, 1, 1)
    with pytest.raises(nlsp.ValidationError):
        nlsp.TwoLevelPreconditioner(a, np.zeros((7, 2)), 0.66, 1, 1)


def test_rank_deficient_basis_rejected(nlsp):
    a = tridiag(4, nlsp)
    m = np.array([[i + 1.0, 2.0 * (i + 1)] for i in range(4)])
    with pytest.raises(nlsp.RankDeficiencyError):
        nlsp.TwoLevelPreconditioner(a, m, 0.66, 1, 1)


@pytest.mark.parametrize("trials,nmax,seed", [(20, 80, 7), (100, 200, 505)])
def test_coarse_exactness_without_smoothing(nlsp, trials, nmax, seed):
    # TwoLevel.CoarseExactnessWithoutSmoothing / acceptance C05 (<= 1e-10)
    rng = np.random.default_rng(seed)
    for _ in range(trials):
        n = int(rng.integers(20, nmax + 1))
        nc = int(rng.integers(1, 9 if nmax < 100 else 13))
        a, dense = random_spd_sparse(n, rng, density=0.08 if nmax < 100 else 0.05,
                                     shift=6.0 if nmax < 100 else 8.0)
        u = orthonormal(n, nc, rng)
        m = nlsp.build_preconditioner(a, u, 0.66, 0, 0)
        y = rng.standard_normal(nc)
        uy = m.basis() @ y
        z = nlsp.apply_two_level(m, a, dense @ uy)
        assert np.abs(z - uy).max() <= 1e-10


def test_apply_is_linear(nlsp):
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    rng = np.random.default_rng(9)
    m = nlsp.TwoLevelPreconditioner(a, orthonormal(a.dim(), 6, rng), 0.66, 2, 2)
    r = rng.standard_normal(a.dim())
    z1 = m.apply(a, r)
    z2 = m.apply(a, -3.75 * r)
    assert np.all(np.abs(z2 + 3.75 * z1) <= 1e-12 * np.maximum(1.0, np.abs(z1)))


def test_preconditioned_operator_self_adjoint(nlsp):
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    dense = a.to_dense()
    rng = np.random.default_rng(13)
    m = nlsp.TwoLevelPreconditioner(a, orthonormal(a.dim(), 8, rng), 0.66, 5, 5)
    for _ in range(20):
        x, y = rng.standard_normal(a.dim()), rng.standard_normal(a.dim())
        ax, ay = dense @ x, dense @ y
        lhs = (dense @ m.apply(a, ax)) @ y
        rhs = ax @ m.apply(a, ay)
        nx, ny = np.linalg.norm(x), np.linalg.norm(y)
        assert abs(lhs - rhs) <= 1e-8 * nx * ny
        assert abs(m.apply(a, x) @ y - x @ m.apply(a, y)) <= 1e-10 * nx * ny
    for _ in range(100):
        r = rng.standard_normal(a.dim())
        assert m.apply(a, r) @ r > 0.0


def test_apply_matches_reference_on_random_systems(nlsp):
    d = golden("random_spd")
    for t in range(int(d["trials"])):
        a = nlsp.SparseCsrMatrix(int(d[f"t{t}_n"]), d[f"t{t}_rp"], d[f"t{t}_ci"], d[f"t{t}_v"])
        for nu, key in [(0, "z0"), (2, "z2")]:
            m = nlsp.TwoLevelPreconditioner(a, d[f"t{t}_basis_in"], 0.66, nu, nu)
            z = m.apply(a, d[f"t{t}_r"])
            ref = d[f"t{t}_{key}"]
            assert np.linalg.norm(z - ref) <= 1e-12 * np.linalg.norm(ref)
        m = nlsp.TwoLevelPreconditioner(a, d[f"t{t}_basis_in"], 0.66, 0, 0)
        basis, chol, coarse = m._export()
        assert np.abs(basis - d[f"t{t}_basis"]).max() <= 1e-12
        assert np.abs(coarse - d[f"t{t}_coarse"]).max() <= 1e-10 * np.abs(d[f"t{t}_coarse"]).max()
        assert np.allclose(chol @ chol.T, coarse, rtol=1e-12, atol=1e-12 * np.abs(coarse).max())


# ------------------------------------------------------------------- pcg ---
def test_pcg_identity_converges_in_one_iteration(nlsp):
    a = nlsp.SparseCsrMatrix.identity(10)
    res = nlsp.pcg(a, np.full(10, 2.5), nlsp.IdentityPreconditioner(), 1e-10, 100)
    assert res.report.converged and res.report.iterations == 1
    assert np.allclose(res.solution, 2.5, atol=1e-12)


def test_pcg_zero_rhs_rejected(nlsp):
    a = nlsp.SparseCsrMatrix.identity(4)
    with pytest.raises(nlsp.ValidationError):
        nlsp.pcg(a, np.zeros(4), nlsp.IdentityPreconditioner(), 1e-6, 10)
    with pytest.raises(nlsp.ValidationError):
        nlsp.pcg(a, np.ones(3), nlsp.IdentityPreconditioner(), 1e-6, 10)


def test_pcg_error_order_matches_reference(nlsp):
    """pcg checks the right-hand side before the preconditioner is applied
    (two_level.hpp:148 then :152): a zero rhs under a Jacobi preconditioner
    with a non-positive diagonal is a ValidationError, a nonzero one the
    JacobiPreconditioner's NumericError (:112-113)."""
    a = nlsp.SparseCsrMatrix.from_triplets(2, [(0, 0, 1.0), (1, 1, -1.0)])
    with pytest.raises(nlsp.ValidationError):
        nlsp.pcg(a, np.zeros(2), nlsp.JacobiPreconditioner(), 1e-8, 10)
    with pytest.raises(nlsp.NumericError):
        nlsp.pcg(a, np.ones(2), nlsp.JacobiPreconditioner(), 1e-8, 10)


def test_pcg_history_sized_by_iterations(nlsp):
    """The history is read after the solve (nlsp_pcg_history), sized by the
    iterations run: a reference-style max_iters = 10 n, or SIZE_MAX, allocates
    nothing proportional to it."""
    import ctypes as C
    from paper_2601_20174_b200 import _lib as L
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    for mx in (10 * a.dim(), 2**64 - 1):
        res = nlsp.pcg(a, d["rhs"], nlsp.IdentityPreconditioner(), 1e-8, mx)
        assert res.report.converged and len(res.report.residual_history) == res.report.iterations
    ctx = nlsp.default_context()
    cnt = C.c_uint64(0)
    assert L.gpu_lib().nlsp_pcg_history(ctx.handle, None, 0, C.byref(cnt)) == 0
    assert cnt.value == res.report.iterations
    part = np.empty(3)
    assert L.gpu_lib().nlsp_pcg_history(ctx.handle, L.dptr(part), 3, C.byref(cnt)) == 0
    assert np.array_equal(part, res.report.residual_history[:3])


def test_pcg_not_spd_detected(nlsp):
    a = nlsp.SparseCsrMatrix.from_triplets(2, [(0, 0, 1.0), (1, 1, -1.0)])
    with pytest.raises(nlsp.NotSpdError):
        nlsp.pcg(a, np.array([0.0, 1.0]), nlsp.IdentityPreconditioner(), 1e-8, 10)


def test_pcg_max_iters_and_zero_iters(nlsp):
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    res = nlsp.pcg(a, d["rhs"], nlsp.IdentityPreconditioner(), 1e-12, 5)
    assert not res.report.converged and res.report.iterations == 5
    assert len(res.report.residual_history) == 5
    res = nlsp.pcg(a, d["rhs"], nlsp.IdentityPreconditioner(), 1e-12, 0)
    assert res.report.iterations == 0 and not res.report.converged
    assert np.all(res.solution == 0.0) and abs(res.report.true_relative_residual - 1.0) < 1e-15


def test_pcg_unpreconditioned_and_jacobi_match_reference(nlsp, oracle):
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    n = a.dim()
    plain = nlsp.pcg(a, d["rhs"], nlsp.IdentityPreconditioner(), 1e-6, 10 * n)
    assert plain.report.converged and plain.report.iterations <= 2 * n
    assert plain.report.true_relative_residual <= 10 * 1e-6
    assert abs(plain.report.iterations - int(d["plain_iterations"])) <= 2
    jac = nlsp.pcg(a, d["rhs"], nlsp.JacobiPreconditioner(), 1e-8, 5000)
    assert jac.report.converged
    assert len(jac.report.residual_history) == jac.report.iterations
    assert jac.report.residual_history[-1] < 1e-8
    assert abs(jac.report.iterations - int(d["jacobi_iterations"])) <= 2
    assert np.linalg.norm(jac.solution - d["jacobi_x"]) <= 1e-9 * np.linalg.norm(d["jacobi_x"])


def test_two_level_beats_unpreconditioned_on_diffusion(nlsp):
    # Pcg.TwoLevelBeatsUnpreconditionedOnDiffusion with the reference's own S
    d = golden("fem_diffusion")
    a = csr_from_golden(d)
    sv = nlsp.generate_smoothed_vectors(a, d["mask"], 16, 10, 0.66, 29)
    p, _, _ = nlsp.svd_basis(sv.s, 8)
    m = nlsp.TwoLevelPreconditioner(a, p, 0.66, 5, 5)
    two = nlsp.pcg(a, d["rhs"], m, 1e-6, 10 * a.dim())
    plain = nlsp.pcg(a, d["rhs"], nlsp.IdentityPreconditioner(), 1e-6, 10 * a.dim())
    assert two.report.converged and plain.report.converged
    assert two.report.iterations < plain.report.iterations
    assert two.report.true_relative_residual <= 10 * 1e-6
    assert abs(two.report.iterations - int(d["iterations"])) <= 2
    assert np.linalg.norm(two.solution - d["x"]) <= 1e-9 * np.linalg.norm(d["x"])


@pytest.mark.parametrize("name", ["c1_default", "c1_strict", "scaled_C2", "scaled_C3",
                                  "scaled_C4", "scaled_C5"])
def test_full_pipeline_matches_reference(nlsp, name):
    """bench_single's SVD row (pipeline.hpp:303-346) end to end on the GPU vs the
    reference's outputs for the same seeded inputs."""
    d = golden(name)
    a = csr_from_golden(d)
    mask = d["mask"] if d["mask"].any() else None
    k = int(d["k"])
    sv = nlsp.generate_smoothed_vectors(a, mask, int(d["m"]), int(d["s1"]), float(d["omega"]),
                                        int(d["s0_seed"]))
    p, sig, _ = nlsp.svd_basis(sv.s, k)
    m = nlsp.TwoLevelPreconditioner(a, p, float(d["omega"]), int(d["nu1"]), int(d["nu2"]))
    basis, chol, coarse = m._export()
    # P and A_c to 1e-10 (norm-relative per column, up to column sign)
    errs, signs = col_match(basis, d["basis"])
    lam = d["sigma"] ** 2
    gaps = np.array([min(lam[j - 1] - lam[j] if j > 0 else np.inf, lam[j] - lam[j + 1])
                     for j in range(k)])
    assert np.all(errs <= np.maximum(1e-10, 1e-13 * lam[0] / gaps)), errs
    dac = np.diag(signs)
    ac_ref = dac @ d["coarse"] @ dac
    sub = np.maximum(1e-10, 1e-13 * lam[0] / gaps.min())
    assert np.abs(coarse - ac_ref).max() <= sub * np.abs(ac_ref).max()
    # PCG: iterations +-2, same stopping tolerance, solution to 1e-9
    res = nlsp.pcg(a, d["rhs"], m, float(d["delta"]), 10 * a.dim())
    rep = res.report
    assert rep.converged and bool(d["converged"])
    assert abs(rep.iterations - int(d["iterations"])) <= 2
    assert rep.residual_history[-1] < float(d["delta"])
    assert rep.true_relative_residual < 10 * float(d["delta"])
    assert np.linalg.norm(res.solution - d["x"]) <= 1e-9 * np.linalg.norm(d["x"])
    # apply on a random r to ~1e-12 (SURVEY §8c unit-level check)
    z = m.apply(a, d["r_probe"])
    assert np.linalg.norm(z - d["z_probe"]) <= 1e-11 * np.linalg.norm(d["z_probe"])


def test_nu_variants_match_oracle(nlsp, oracle):
    d = golden("scaled_C3")
    a = csr_from_golden(d)
    ao = (a.dim(), a.row_ptr(), a.col_idx(), a.values())
    p = d["P"]
    for nu1, nu2 in [(0, 0), (0, 1), (1, 0), (2, 2), (3, 1)]:
        m = nlsp.TwoLevelPreconditioner(a, p, 2 / 3, nu1, nu2)
        t = oracle.twolevel(ao, p, 2 / 3, nu1, nu2)
        r = np.random.default_rng(nu1 * 10 + nu2).standard_normal(a.dim())
        z, zo = m.apply(a, r), t.apply(r)
        assert np.linalg.norm(z - zo) <= 1e-12 * np.linalg.norm(zo), (nu1, nu2)
        res = nlsp.pcg(a, d["rhs"], m, 1e-8, 10 * a.dim())
        ro = oracle.pcg(ao, d["rhs"], 2, t, 1e-8, 10 * a.dim())
        assert abs(res.report.iterations - ro.iterations) <= 2, (nu1, nu2)
        assert np.linalg.norm(res.solution - ro.x) <= 1e-9 * np.linalg.norm(ro.x)


def test_odd_coarse_dimension_and_repeat_solves_are_deterministic(nlsp):
    d = golden("scaled_C4")
    a = csr_from_golden(d)
    p = d["P"][:, :7]
    m = nlsp.TwoLevelPreconditioner(a, p, 2 / 3, 1, 1)
    r1 = nlsp.pcg(a, d["rhs"], m, 1e-8, 10 * a.dim())
    r2 = nlsp.pcg(a, d["rhs"], m, 1e-8, 10 * a.dim())
    assert r1.report.converged and np.array_equal(r1.solution, r2.solution)
    assert np.array_equal(r1.report.residual_history, r2.report.residual_history)


_LOOP_SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
from paper_2601_20174_b200 import nlsp
d = np.load({path!r})
a = nlsp.SparseCsrMatrix(int(d["n"]), d["row_ptr"], d["col_idx"], d["values"])
m = nlsp.TwoLevelPreconditioner(a, d["P"], float(d["omega"]), int(d["nu1"]), int(d["nu2"]))
r = nlsp.pcg(a, d["rhs"], m, float(d["delta"]), 10 * a.dim())
np.save({out!r}, r.solution)
print(json.dumps({{"iterations": r.report.iterations, "launches": r.report.kernel_launches}}))
"""


@pytest.mark.parametrize("cycle", ["folded", "literal"])
def test_graph_and_stream_loops_agree(tmp_path, cycle):
    """The CUDA-graph WHILE loop and the stream-ordered loop (NLSP_LOOP=host, used
    under ncu) run the same kernels: identical iterations and bitwise x, for the
    folded and the literal cycle."""
    import json
    import subprocess
    import sys
    from conftest import GOLDEN, ROOT
    res = {}
    for loop in ["graph", "host"]:
        out = str(tmp_path / f"x_{loop}.npy")
        code = _LOOP_SCRIPT.format(root=ROOT, path=f"{GOLDEN}/scaled_C3.npz", out=out)
        env = dict(os.environ, NLSP_LOOP=loop, NLSP_CYCLE=cycle)
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        res[loop] = (json.loads(p.stdout.strip().splitlines()[-1]), np.load(out))
    assert res["graph"][0]["iterations"] == res["host"][0]["iterations"]
    assert np.array_equal(res["graph"][1], res["host"][1])
    assert res["graph"][0]["launches"] > 0


@pytest.mark.parametrize("k", [65, 128, 200])
def test_large_coarse_dimension(nlsp, oracle, k):
    """k beyond the configs' 64 (the reference has no limit): wider basis rows,
    2-stage or direct-load fallbacks of the staged kernels."""
    d = golden("scaled_C4")
    a = csr_from_golden(d)
    ao = (a.dim(), a.row_ptr(), a.col_idx(), a.values())
    basis = np.linalg.qr(np.random.default_rng(k).standard_normal((a.dim(), k)))[0]
    m = nlsp.TwoLevelPreconditioner(a, basis, 2 / 3, 1, 1)
    t = oracle.twolevel(ao, basis, 2 / 3, 1, 1)
    r = np.random.default_rng(1).standard_normal(a.dim())
    z, zo = m.apply(a, r), t.apply(r)
    assert np.linalg.norm(z - zo) <= 1e-11 * np.linalg.norm(zo)
    res = nlsp.pcg(a, d["rhs"], m, 1e-8, 10 * a.dim())
    ro = oracle.pcg(ao, d["rhs"], 2, t, 1e-8, 10 * a.dim())
    assert abs(res.report.iterations - ro.iterations) <= 2
    assert np.linalg.norm(res.solution - ro.x) <= 1e-9 * np.linalg.norm(ro.x)


def test_long_rows_fall_back_from_staged_tiles(nlsp, oracle):
    """An SPD matrix with a few dense rows/columns: staged tiles would exceed
    shared memory, the direct-load kernels take over; results unchanged."""
    rng = np.random.default_rng(21)
    n = 3000
    dense = np.zeros((n, n))
    for i in range(n):
        for dj in (-1, 1):
            if 0 <= i + dj < n:
                dense[i, i + dj] = -1.0
    hub = [5, 1700]
    for h in hub:
        cols = rng.choice(n, size=2500, replace=False)
        vals = 0.01 * rng.standard_normal(2500)
        dense[h, cols] += vals
        dense[cols, h] += vals
    dense += np.diag(np.abs(dense).sum(axis=1) + 1.0)
    ii, jj = np.nonzero(dense)
    a = nlsp.SparseCsrMatrix.from_coo(n, ii, jj, dense[ii, jj])
    ao = (n, a.row_ptr(), a.col_idx(), a.values())
    x = rng.standard_normal(n)
    assert np.abs(nlsp.spmv(a, x) - dense @ x).max() <= 1e-12 * np.abs(dense @ x).max()
    basis = np.linalg.qr(rng.standard_normal((n, 6)))[0]
    m = nlsp.TwoLevelPreconditioner(a, basis, 2 / 3, 1, 1)
    t = oracle.twolevel(ao, basis, 2 / 3, 1, 1)
    b = rng.standard_normal(n)
    res = nlsp.pcg(a, b, m, 1e-10, 10 * n)
    ro = oracle.pcg(ao, b, 2, t, 1e-10, 10 * n)
    assert abs(res.report.iterations - ro.iterations) <= 2
    assert np.linalg.norm(res.solution - ro.x) <= 1e-9 * np.linalg.norm(ro.x)
