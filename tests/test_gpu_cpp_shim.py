"""The C++ drop-in shim (include/nlsp_gpu.hpp): a reference-style program
(bench_single's SVD row) built against it — once with local types, once with
the reference's own nlsp::SparseCsrMatrix / exceptions — solves config C1 and
agrees with the reference's golden outputs."""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu
BUILD = os.path.join(ROOT, "tests", "cpp", "build")


def save(path, arr):
    arr = np.ascontiguousarray(arr, dtype=np.float64).reshape(len(arr), -1)
    with open(path, "wb") as f:
        np.array(arr.shape, dtype=np.uint64).tofile(f)
        arr.tofile(f)


def load(path):
    with open(path, "rb") as f:
        rows, cols = np.fromfile(f, dtype=np.uint64, count=2)
        return np.fromfile(f, dtype=np.float64, count=int(rows * cols))


@pytest.mark.parametrize("binary", ["shim_demo", "shim_demo_ref"])
def test_shim_program_matches_reference(tmp_path, binary):
    exe = os.path.join(BUILD, binary)
    if binary == "shim_demo_ref" and not os.path.exists(exe):
        pytest.skip("built only where /root/reference exists")
    assert os.path.exists(exe), "run __graft_entry__.build() first"
    d = golden("c1_default")
    save(tmp_path / "csr_rp.bin", d["row_ptr"].astype(np.float64))
    save(tmp_path / "csr_ci.bin", d["col_idx"].astype(np.float64))
    save(tmp_path / "csr_v.bin", d["values"])
    save(tmp_path / "rhs.bin", d["rhs"])
    save(tmp_path / "params.bin", np.array([d["k"], d["m"], d["s1"], d["nu1"], d["nu2"], d["omega"],
                                            d["delta"], d["s0_seed"]], dtype=np.float64))
    p = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["converged"] == 1 and out["zero_rhs_rejected"] == 1
    assert abs(out["iterations"] - int(d["iterations"])) <= 2
    assert abs(out["plain_iterations"] - int(d["plain_iterations"])) <= 2
    assert out["history_len"] == out["iterations"]
    # the reference-signature call site (build_preconditioner / unqualified pcg /
    # apply_two_level / M.apply(a, r) on the reference's matrix type): same solve
    assert out["ref_style_iterations"] == out["iterations"]
    assert out["ref_style_history_len"] == out["iterations"] and out["ref_style_method"] == "two_level"
    assert out["ref_style_x_maxdiff"] <= 1e-12 * np.abs(d["x"]).max()
    assert out["apply_rel_diff"] <= 1e-12
    # generate_smoothed_vectors / svd_first_cols with the reference's arguments:
    # the same (deterministic) basis
    assert out["ref_style_basis_maxdiff"] == 0.0
    x = load(tmp_path / "x.bin")
    assert np.linalg.norm(x - d["x"]) <= 1e-9 * np.linalg.norm(d["x"])
