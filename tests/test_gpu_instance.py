"""bench_single's SVD row (pipeline.hpp:303-346) end to end on an instance
directory read by libnlsp_io.so: load_instance -> generate_smoothed_vectors
with the instance's Dirichlet mask and ExperimentConfig::smoothing_seed ->
svd_basis -> TwoLevelPreconditioner(nu1 = nu2 = 5) -> pcg(delta = 1e-6), at
the reference's default ranks 4/8/16/32, plus the plain-CG column. Compared
with the reference's own run of the same pipeline (tests/golden/io/n32_svd.npz,
tests/golden/make_io_golden.py)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, col_match
from paper_2601_20174_b200 import instance_io as io

pytestmark = pytest.mark.gpu

IO = os.path.join(GOLDEN, "io")


@pytest.fixture(scope="module")
def case(nlsp):
    inst = io.load_instance(os.path.join(IO, "inst_diffusion_n32"))
    g = np.load(os.path.join(IO, "n32_svd.npz"))
    sv = nlsp.generate_smoothed_vectors(inst.matrix, inst.boundary_mask, int(g["K"]), int(g["s1"]),
                                        float(g["omega"]), int(g["smoothing_seed"]))
    return inst, g, sv


def test_smoothed_vectors_on_instance(case):
    inst, g, sv = case
    s = sv.s.numpy()
    assert np.abs(s - g["S"]).max() <= 1e-13 * np.abs(g["S"]).max()
    assert np.all(s[inst.boundary_mask.astype(bool)] == 0.0)


@pytest.mark.parametrize("rank", [4, 8, 16, 32])
def test_svd_row(nlsp, case, rank):
    inst, g, sv = case
    p, sig, _ = nlsp.svd_basis(sv.s, rank)
    lam = g["sigma"] ** 2
    assert np.abs(sig - g["sigma"]).max() <= 1e-12 * g["sigma"][0]
    errs, _ = col_match(p.numpy(), g[f"r{rank}_P"])
    gaps = np.array([min(lam[j - 1] - lam[j] if j > 0 else np.inf,
                         lam[j] - lam[j + 1] if j + 1 < lam.size else np.inf) for j in range(rank)])
    assert np.all(errs <= np.maximum(1e-10, 1e-13 * lam[0] / gaps))
    omega, nu, delta = float(g["omega"]), int(g["nu"]), float(g["delta"])
    m = nlsp.TwoLevelPreconditioner(inst.matrix, p, omega, nu, nu)
    res = nlsp.pcg(inst.matrix, inst.rhs, m, delta, 10 * inst.matrix.dim())
    rep = res.report
    assert rep.converged and bool(g[f"r{rank}_converged"])
    assert abs(rep.iterations - int(g[f"r{rank}_iterations"])) <= 2
    assert rep.true_relative_residual < 10 * delta
    x_ref = g[f"r{rank}_x"]
    assert np.linalg.norm(res.solution - x_ref) <= 1e-9 * np.linalg.norm(x_ref)


def test_plain_cg_column(nlsp, case):
    inst, g, _ = case
    res = nlsp.pcg(inst.matrix, inst.rhs, nlsp.IdentityPreconditioner(), float(g["delta"]),
                   10 * inst.matrix.dim())
    assert abs(res.report.iterations - int(g["plain_iterations"])) <= 2
