"""CPU check of the lean cycle's scalar recurrences (DESIGN.md §3 "Lean cycle"):
the numpy prototype runs PCG with beta formed before the pass over W
(r.z = r.s + c.e) and alpha predicted after it (p.Ap = z.Az - beta r.z / alpha_prev)
beside the plain folded schedule, on scaled instances of the BASELINE families.
The GPU kernels implement exactly these formulas (solve_kernels.cu, OpSpmvUpd /
OpSweepLean / k_prolong_onepass_tma lean)."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _proto():
    spec = importlib.util.spec_from_file_location("lean_prototype", os.path.join(ROOT, "scripts", "lean_prototype.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("case", [("C3", 64, 12, 2), ("C4", 16, 12, 1), ("C2", 64, 8, 1), ("C5", 24, 12, 1)])
def test_lean_scalars_track_plain_pcg(case):
    r = _proto().main(*case)
    # same iteration count, x to rounding, the predicted p.Ap within 1e-12 of
    # the direct one, and no cancellation to speak of in z.Az - beta r.z / alpha
    assert r["lean"] == r["folded"]
    assert r["x_diff"] <= 1e-12
    assert r["pap_dev"] <= 1e-12
    assert r["cancellation"] <= 8.0
    assert r["hist_dev"] <= 1e-8
