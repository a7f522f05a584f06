"""The SA coarse space against the reference's own sa.hpp
(tests/golden/sa/sa.npz, tests/golden/make_sa_golden.py): aggregate ids
bit-exact on the host; on the GPU the dense prolongator, and bench_single's SA
row (TwoLevelPreconditioner(A, sa_prolongator(A)), nu 5/5, delta 1e-6) — the
N = 32 instance has n_c = 551, so it runs the wide (k > 256) kernels."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2601_20174_b200 import instance_io as io
from paper_2601_20174_b200 import sa
from paper_2601_20174_b200.nlsp import SparseCsrMatrix

G = np.load(os.path.join(GOLDEN, "sa", "sa.npz"))
NAMES = [str(x) for x in G["names"]]


def case(name):
    if name.startswith("inst_"):
        inst = io.load_instance(os.path.join(GOLDEN, "io", name))
        return inst.matrix, inst.rhs
    a = SparseCsrMatrix(int(G[f"{name}__n"]), G[f"{name}__rp"], G[f"{name}__ci"], G[f"{name}__v"])
    return a, G[f"{name}__rhs"]


@pytest.mark.parametrize("name", NAMES)
def test_aggregates_match_reference(name):
    a, _ = case(name)
    agg, nc = sa.aggregate_nodes(a, 0.25)
    assert nc == int(G[f"{name}__nc"])
    assert np.array_equal(agg, G[f"{name}__agg"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_sa_row_matches_reference(nlsp, name):
    a, rhs = case(name)
    p = sa.sa_prolongator(a, 0.25, 0.66)
    assert (p.rows, p.cols) == (a.dim(), int(G[f"{name}__nc"]))
    if f"{name}__P" in G.files:
        pr = G[f"{name}__P"]
        assert np.abs(p.numpy() - pr).max() <= 1e-15 * np.abs(pr).max()
    m = nlsp.TwoLevelPreconditioner(a, p, 0.66, 5, 5)
    res = nlsp.pcg(a, rhs, m, 1e-6, 10 * a.dim())
    assert res.report.converged and bool(G[f"{name}__converged"])
    assert abs(res.report.iterations - int(G[f"{name}__iterations"])) <= 2
    x_ref = G[f"{name}__x"]
    assert np.linalg.norm(res.solution - x_ref) <= 1e-9 * np.linalg.norm(x_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("k,nu", [(300, (1, 1)), (700, (2, 2)), (1100, (1, 1)), (2048, (1, 1))])
def test_wide_coarse_space_apply_and_pcg(nlsp, k, nu):
    """k > 256: the wide restriction / A_c^-1 mat-vec / prolongation kernels,
    against the cycle of two_level.hpp:60-81 evaluated densely in numpy."""
    rng = np.random.default_rng(k)
    n = max(1800, k + 600)
    # 1D Laplacian-plus-random-couplings SPD system
    ii, jj, vv = [], [], []
    for i in range(n):
        ii += [i]
        jj += [i]
        vv += [4.0 + rng.random()]
        for d in (1, 7, 31):
            if i + d < n:
                w = -0.3 - 0.4 * rng.random()
                ii += [i, i + d]
                jj += [i + d, i]
                vv += [w, w]
    a = SparseCsrMatrix.from_coo(n, ii, jj, vv)
    basis = rng.standard_normal((n, k))
    m = nlsp.TwoLevelPreconditioner(a, basis, 0.66, nu[0], nu[1])
    assert m.coarse_dim() == k
    A = a.to_dense()
    P = m.basis()
    assert np.abs(P.T @ P - np.eye(k)).max() < 1e-11
    Ac = P.T @ A @ P
    dinv = 0.66 / np.diag(A)
    r = rng.standard_normal(n)
    z = np.zeros(n)
    for _ in range(nu[0]):
        z = z + dinv * (r - A @ z)
    z = z + P @ np.linalg.solve(Ac, P.T @ (r - A @ z))
    for _ in range(nu[1]):
        z = z + dinv * (r - A @ z)
    zg = m.apply(a, r)
    assert np.abs(zg - z).max() <= 1e-9 * np.abs(z).max()
    b = rng.standard_normal(n)
    res = nlsp.pcg(a, b, m, 1e-8, 10 * n)
    assert res.report.converged
    assert np.linalg.norm(b - A @ res.solution) <= 1e-7 * np.linalg.norm(b)


G64 = np.load(os.path.join(GOLDEN, "sa", "sa_n64.npz"))


def test_aggregates_n64_match_reference():
    inst = io.load_instance(os.path.join(GOLDEN, "io", "inst_diffusion_n64"))
    agg, nc = sa.aggregate_nodes(inst.matrix, 0.25)
    assert nc == int(G64["nc"]) == 2009
    assert np.array_equal(agg, G64["agg"])


@pytest.mark.gpu
def test_sa_row_n64_matches_reference(nlsp):
    """The paper's N = 64 SA row: n_c = 2 009 (the reference's constructor
    took 575 s on one core to make this golden)."""
    inst = io.load_instance(os.path.join(GOLDEN, "io", "inst_diffusion_n64"))
    p = sa.sa_prolongator(inst.matrix, 0.25, 0.66)
    m = nlsp.TwoLevelPreconditioner(inst.matrix, p, 0.66, 5, 5)
    assert m.coarse_dim() == 2009
    res = nlsp.pcg(inst.matrix, inst.rhs, m, 1e-6, 10 * inst.matrix.dim())
    assert res.report.converged
    assert abs(res.report.iterations - int(G64["iterations"])) <= 2
    assert np.linalg.norm(res.solution - G64["x"]) <= 1e-9 * np.linalg.norm(G64["x"])
