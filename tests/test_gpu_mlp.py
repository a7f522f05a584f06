"""MLP inference on the device against the reference: the
forward pass (mlp.hpp:113-161), infer_basis (train.hpp:52-62) and
bench_single's NLSS row (pipeline.hpp:303-346) at rank 8 on the N = 32
instance (tests/golden/mlp, made by tests/golden/make_mlp_golden.py)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2601_20174_b200 import instance_io as io
from paper_2601_20174_b200 import mlp

pytestmark = pytest.mark.gpu

D = os.path.join(GOLDEN, "mlp")


def test_forward_matches_reference(nlsp):
    g = np.load(os.path.join(D, "small.npz"))
    m = mlp.MlpModel.load(os.path.join(D, "small.ckpt"))
    y = m.forward(g["x"])
    assert np.abs(y - g["y"]).max() <= 1e-12 * np.abs(g["y"]).max()


def test_wide_forward_splitk_matches_numpy(nlsp):
    # fan-in above the split-K threshold, hidden LayerNorm + GELU, plain output
    from math import erf, sqrt
    rng = np.random.default_rng(8)
    m = mlp.MlpModel.init([9000, 64, 300], 3)
    m.params[:] = m.params + 0.01 * rng.standard_normal(m.params.size)  # non-trivial bias/gain/offset
    x = rng.standard_normal(9000)
    w = m.widths
    o = 0
    a = x
    for l in range(len(w) - 1):
        fi, fo = w[l], w[l + 1]
        W = m.params[o:o + fi * fo].reshape(fo, fi)
        o += fi * fo
        b = m.params[o:o + fo]
        o += fo
        z = W @ a + b
        if l + 2 < len(w):
            gain, off = m.params[o:o + fo], m.params[o + fo:o + 2 * fo]
            o += 2 * fo
            xh = (z - z.mean()) / np.sqrt(z.var() + 1e-5)
            yv = gain * xh + off
            a = np.array([0.5 * t * (1.0 + erf(t / sqrt(2.0))) for t in yv])
        else:
            a = z
    y = m.forward(x)
    assert np.abs(y - a).max() <= 1e-11 * np.abs(a).max()


@pytest.fixture(scope="module")
def n32(nlsp):
    g = np.load(os.path.join(D, "n32_nlss.npz"))
    s = np.load(os.path.join(GOLDEN, "io", "n32_svd.npz"))["S"]
    model = mlp.MlpModel.init(g["widths"], int(g["seed"]))
    return g, s, model


def test_infer_basis_matches_reference(nlsp, n32):
    g, s, model = n32
    q = mlp.infer_basis(model, s).numpy()
    assert q.shape == g["Q"].shape
    # CholeskyQR2 vs two-pass MGS: the same Q (positive R diagonal) to rounding
    err = np.abs(q - g["Q"]).max(axis=0) / np.abs(g["Q"]).max(axis=0)
    assert err.max() <= 1e-10, err.max()
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-13


def test_nlss_row_matches_reference(nlsp, n32):
    g, s, model = n32
    inst = io.load_instance(os.path.join(GOLDEN, "io", "inst_diffusion_n32"))
    rank = int(g["rank"])
    q = mlp.infer_basis(model, s).numpy()
    m = nlsp.TwoLevelPreconditioner(inst.matrix, np.ascontiguousarray(q[:, :rank]), 0.66, 5, 5)
    res = nlsp.pcg(inst.matrix, inst.rhs, m, 1e-6, 10 * inst.matrix.dim())
    assert res.report.converged and bool(g["converged"])
    assert abs(res.report.iterations - int(g["iterations"])) <= 2
    assert np.linalg.norm(res.solution - g["x"]) <= 1e-9 * np.linalg.norm(g["x"])


def test_infer_basis_errors(nlsp, n32):
    g, s, model = n32
    with pytest.raises(nlsp.ValidationError, match="width mismatch"):
        mlp.infer_basis(model, s[:, :16])
    with pytest.raises(nlsp.ValidationError, match="zero vector set"):
        mlp.infer_basis(model, np.zeros_like(s))
