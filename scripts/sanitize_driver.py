"""Small end-to-end runs of the product path for compute-sanitizer
(scripts/gpu_sanitize.sh): smoothing, SVD basis, two-level build and a few
PCG iterations, sized so every TMA/mbarrier ring of the solve kernels cycles
many times while the instrumented run stays within minutes.

  python scripts/sanitize_driver.py C1|C4|C5|C3 [max_iters]
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_20174_b200 import nlsp, problems  # noqa: E402

CASES = {
    "C1": problems.C1,                                   # n = 4 096: the single-cluster solver
    "C4": problems.C4.scaled(nx=40, m=64, s1=2),          # n = 64 000, k = 64: graph/stream loop, TMA rings
    "C3": problems.C3.scaled(nx=256, m=96, s1=2),         # n = 65 536, nu = 2/2, k = 48
    "C5": problems.C5.scaled(nx=128, m=96, s1=2),         # n = 33 282: CSR row tiles (no diagonal form)
}


def main():
    name = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    cfg = CASES[name]
    pb = problems.generate(cfg)
    a = pb.csr()
    mask = pb.mask if pb.mask.any() else None
    sv = nlsp.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
    p, sig, _ = nlsp.svd_basis(sv.s, cfg.k)
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    mx = 10 * pb.n if name == "C1" else iters
    res = nlsp.pcg(a, pb.rhs, m, cfg.delta, mx)
    z = m.apply(a, pb.rhs)
    y = nlsp.spmv(a, pb.rhs)
    print(f"{name}: n={pb.n} k={cfg.k} iterations={res.report.iterations} converged={res.report.converged} "
          f"cycle={m.cycle()} |z|={np.linalg.norm(z):.6e} launches={res.report.kernel_launches} "
          f"|Ab|={np.linalg.norm(y):.6e}", flush=True)


if __name__ == "__main__":
    main()
