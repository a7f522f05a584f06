"""MLP checkpoints and initialisation without a GPU: the host
side of libnlsp_io.so against the reference's own MlpModel
(tests/golden/mlp, tests/golden/make_mlp_golden.py)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2601_20174_b200 import mlp
from paper_2601_20174_b200.instance_io import IoError
from paper_2601_20174_b200.nlsp import ValidationError

D = os.path.join(GOLDEN, "mlp")
SMALL = np.load(os.path.join(D, "small.npz"))


def test_load_reference_checkpoint():
    m = mlp.MlpModel.load(os.path.join(D, "small.ckpt"))
    assert m.widths == [40, 16, 8, 24]
    assert np.array_equal(m.params.view(np.uint64), SMALL["params"].view(np.uint64))
    assert m.manifest == "created by oracle/ref_driver.cpp"


def test_seeded_init_is_the_reference_init():
    # MlpModel(widths, seed): Rng(mix_seed(seed, 0x6d6c70)) He weights, gains 1
    m = mlp.MlpModel.init([40, 16, 8, 24], 5)
    assert np.array_equal(m.params.view(np.uint64), SMALL["params"].view(np.uint64))


def test_default_widths_init_matches_golden_run():
    # the N = 32 NLSS golden was produced by MlpModel(default widths, 77); its
    # widths and parameter count are reproduced
    g = np.load(os.path.join(D, "n32_nlss.npz"))
    m = mlp.MlpModel.init(g["widths"], int(g["seed"]))
    n = 1089
    assert list(g["widths"][1:-1]) == mlp.default_hidden_widths(n)
    w = m.widths
    expect = sum(w[i] * w[i + 1] + w[i + 1] + (2 * w[i + 1] if i + 2 < len(w) else 0)
                 for i in range(len(w) - 1))
    assert m.params.size == expect


def test_save_load_round_trip(tmp_path):
    m = mlp.MlpModel.init([7, 5, 3], 11)
    p = tmp_path / "m.ckpt"
    m.save(str(p), "hello = 1\n")
    r = mlp.MlpModel.load(str(p))
    assert r.widths == m.widths and np.array_equal(r.params, m.params) and r.manifest == "hello = 1\n"


def test_checkpoint_errors(tmp_path):
    with pytest.raises(IoError, match="cannot open for read"):
        mlp.MlpModel.load(str(tmp_path / "none.ckpt"))
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"NOTMAGIC" + bytes(64))
    with pytest.raises(IoError, match="bad checkpoint magic"):
        mlp.MlpModel.load(str(bad))
    src = open(os.path.join(D, "small.ckpt"), "rb").read()
    (tmp_path / "trunc.ckpt").write_bytes(src[: len(src) // 2])
    with pytest.raises(IoError, match="truncated checkpoint"):
        mlp.MlpModel.load(str(tmp_path / "trunc.ckpt"))
    # parameter count that does not match the widths
    hdr = bytearray(src)
    np_off = 8 + 8 + 4 * 8
    hdr[np_off:np_off + 8] = (12345).to_bytes(8, "little")
    (tmp_path / "count.ckpt").write_bytes(bytes(hdr))
    with pytest.raises(IoError, match="parameter count mismatch"):
        mlp.MlpModel.load(str(tmp_path / "count.ckpt"))
    with pytest.raises(ValidationError, match="at least input and output"):
        mlp.MlpModel.init([5], 1)
