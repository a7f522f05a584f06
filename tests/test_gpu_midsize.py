"""bench_single's SVD row at mid size against the reference's own run
(tests/golden/make_mid_golden.py): the C2–C5 families beyond the
single-cluster solver (n = 74 498 to 262 144, the BASELINE k, m, nu), so the
whole pipeline — smoothing, SVD basis, two-level build, and PCG on the graph
loop with the one-pass schedule — is checked against the reference's outputs
with the north-star tolerances."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import check_basis_coarse_sketch, golden
from paper_2601_20174_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["mid_C4", "mid_C3", "mid_C2", "mid_C5"])
def test_midsize_pipeline_matches_reference(nlsp, name):
    d = golden(name)
    cfg = problems.CONFIGS[name[4:]].scaled(nx=int(d["nx"]))
    pb = problems.generate(cfg)
    assert pb.n == int(d["n"]) and pb.n > 65536
    a = pb.csr()
    mask = pb.mask if pb.mask.any() else None
    sv = nlsp.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
    p, sig, _ = nlsp.svd_basis(sv.s, cfg.k)
    sref = np.asarray(d["sigma"])
    assert np.abs(np.asarray(sig) - sref[: len(sig)]).max() <= 1e-10 * sref[0]
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    assert m.cycle() in ("onepass", "lean")
    # P and A_c at the BASELINE k / m (north star: 1e-10 up to column sign,
    # gap-limited where the singular values cluster)
    basis, _, coarse = m._export()
    er, es, ea = check_basis_coarse_sketch(d, basis, coarse, cfg.k)
    print(f"{name}: P rows {er.max():.2e} sketch {es.max():.2e} A_c {ea:.2e}")
    res = nlsp.pcg(a, pb.rhs, m, cfg.delta, 10 * pb.n)
    rep = res.report
    assert rep.converged and rep.kernel_launches > 2  # the graph loop, not the cluster solver
    assert abs(rep.iterations - int(d["iterations"])) <= 2, (rep.iterations, int(d["iterations"]))
    assert rep.residual_history[-1] < cfg.delta and rep.true_relative_residual < 10 * cfg.delta
    x = np.asarray(d["x"])
    assert np.linalg.norm(res.solution - x) <= 1e-9 * np.linalg.norm(x)
