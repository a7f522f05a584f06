"""The synthetic BASELINE.json inputs (csrc/inputs.cpp): sizes, CSR invariants,
symmetry / definiteness, and that the random streams are the reference's own
(Rng / mix_seed / generate_smoothed_vectors). CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden
from paper_2601_20174_b200 import problems as P


def dense(pb):
    d = np.zeros((pb.n, pb.n))
    rows = np.repeat(np.arange(pb.n), np.diff(pb.row_ptr.astype(np.int64)))
    d[rows, pb.col_idx.astype(np.int64)] = pb.values
    return d


def check_csr(pb):
    rp = pb.row_ptr.astype(np.int64)
    assert rp[0] == 0 and rp[-1] == pb.nnz and np.all(np.diff(rp) >= 0)
    ci = pb.col_idx.astype(np.int64)
    assert ci.min() >= 0 and ci.max() < pb.n
    for i in range(pb.n):
        seg = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(seg) > 0)  # sorted, no duplicates (sparse.hpp:17-18)
    assert np.all(pb.values != 0.0)      # zeros kept out (sparse.hpp:45)


@pytest.mark.parametrize("cfg,n,nnz", [
    (P.C1, 4096, 20224),
    (P.C2, 1048576, 5238784),
    (P.C3, 4194304, 37724164),
    (P.C4, 4096000, 28518400),
])
def test_full_size_counts(cfg, n, nnz):
    # SURVEY §8a sizes (Dirichlet eliminated for C1-C4)
    pb = P.generate(cfg)
    assert pb.n == n and pb.nnz == nnz
    assert not pb.mask.any()


def test_c5_counts_and_clamp():
    pb = P.generate(P.C5)
    assert pb.n == 2 * 513 * 513
    # 18 structural couplings per row (~9.45M), minus the couplings
    # that cancel exactly inside equal-E blocks, which from_triplets drops
    # (sparse.hpp:45): ~13 stored per row
    assert 6.5e6 < pb.nnz < 9.5e6
    assert pb.nnz < 18 * pb.n
    clamped = np.flatnonzero(pb.mask)
    assert clamped.size == 2 * 513
    # clamped dofs are identity rows with zero rhs (fem.hpp:184-200)
    rp = pb.row_ptr.astype(np.int64)
    for i in clamped[:20]:
        assert rp[i + 1] - rp[i] == 1 and pb.col_idx[rp[i]] == i and pb.values[rp[i]] == 1.0
    assert np.all(pb.rhs[clamped] == 0.0)


@pytest.mark.parametrize("name,cfg", [
    ("C1", P.C1.scaled(nx=9)),
    ("C2", P.C2.scaled(nx=12)),
    ("C3", P.C3.scaled(nx=11)),
    ("C4", P.C4.scaled(nx=6)),
    ("C5", P.C5.scaled(nx=6, blocks=2)),
])
def test_small_operators_are_spd(name, cfg):
    pb = P.generate(cfg)
    check_csr(pb)
    a = dense(pb)
    assert np.abs(a - a.T).max() <= 1e-12 * np.abs(a).max()
    assert np.linalg.eigvalsh(a).min() > 0.0
    assert np.all(np.diag(a) > 0.0)


def test_c1_stencil_values():
    pb = P.generate(P.C1.scaled(nx=5))
    a = dense(pb)
    assert np.all(np.diag(a) == 4.0)
    off = a - np.diag(np.diag(a))
    assert set(np.unique(off)) <= {-1.0, 0.0}


def test_c3_rotated_tensor_coefficients():
    pb = P.generate(P.C3.scaled(nx=7))
    a = dense(pb)
    eps, th = 1e-3, math.pi / 6
    c, s = math.cos(th), math.sin(th)
    k11, k22, k12 = c * c + eps * s * s, s * s + eps * c * c, (1 - eps) * c * s
    i = 3 * 7 + 3  # interior point
    assert math.isclose(a[i, i], 2 * k11 + 2 * k22, rel_tol=1e-15)
    assert math.isclose(a[i, i + 1], -k11, rel_tol=1e-15)
    assert math.isclose(a[i, i + 7], -k22, rel_tol=1e-15)
    assert math.isclose(a[i, i + 8], -0.5 * k12, rel_tol=1e-15)
    assert math.isclose(a[i, i + 6], 0.5 * k12, rel_tol=1e-15)


def test_c2_grf_statistics():
    pb = P.generate(P.C2.scaled(nx=256))
    g = np.log(pb.coef).reshape(256, 256)
    # variance 1 and correlation length 0.1 of the domain (SE covariance)
    assert 0.3 < g.var() < 2.5
    lag = int(round(0.1 * 256))
    c_lag = np.mean((g[:, :-lag] - g.mean()) * (g[:, lag:] - g.mean())) / g.var()
    assert 0.3 < c_lag < 0.9  # exp(-1/2) ~= 0.61 in expectation
    # harmonic face means: row sums of the off-diagonals vs the diagonal
    a = pb.csr()
    assert pb.nnz == 5 * 256 * 256 - 4 * 256


def test_c5_young_modulus_range():
    pb = P.generate(P.C5.scaled(nx=64, blocks=16))
    e = np.unique(pb.coef)
    assert e.size <= 256 and e.min() >= 1.0 and e.max() <= 1e3


def test_streams_are_the_reference_rng():
    g = golden("rng")
    assert np.array_equal(P.rng_normal(5, 1001), g["normal_seed5"])
    assert P.mix_seed(7, 0x736d6f6f) == int(g["mix"][1])
    # S^(0) of generate_smoothed_vectors = Rng(mix_seed(seed, "smoo")) i-major
    s0 = P.smoothed_s0(7, 1024, 4)
    assert np.array_equal(s0.ravel(), g["normal_seed_smoo7"][:4096])


def test_s0_matches_reference_fill_with_mask(oracle):
    pb = P.generate(P.C5.scaled(nx=4, blocks=2))
    a = (pb.n, pb.row_ptr, pb.col_idx, pb.values)
    s_ref = oracle.generate_smoothed_vectors(a, pb.mask, 5, 0, 0.66, 11)
    assert np.array_equal(P.smoothed_s0(11, pb.n, 5, pb.mask), s_ref)


def test_rhs_uniform_for_c3():
    pb = P.generate(P.C3.scaled(nx=16))
    assert pb.rhs.min() >= -1.0 and pb.rhs.max() < 1.0 and abs(pb.rhs.mean()) < 0.2


def test_bad_spec_rejected():
    with pytest.raises(ValueError):
        P.generate(P.C1.scaled(nx=0))
    with pytest.raises(ValueError):
        P.generate(P.C5.scaled(young_lo=-1.0))
