"""tests/golden/make_mid_golden.py — mid-size goldens produced by the REFERENCE
ITSELF (oracle/_ref/libnlsp_ref.so, the reference's headers): the C4 and C3
families at sizes beyond the single-cluster solver (n > 65 536), where the GPU
runs its multi-kernel graph loop with the one-pass schedule. Each is
bench_single's SVD row end to end (generate_smoothed_vectors -> svd_oracle ->
first_cols -> TwoLevelPreconditioner -> pcg, pipeline.hpp:303-346) at the
BASELINE k, m, nu. Only the outputs are stored (the inputs are regenerated
bit-identically from the seeded generators).

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_mid_golden.py
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2601_20174_b200 import problems  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sketch import col_argmax, sample_rows, sketch  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

MID = {
    "mid_C4": problems.C4.scaled(nx=64),    # n = 262 144, k = 64, m = 128, nu = 1/1
    "mid_C3": problems.C3.scaled(nx=320),   # n = 102 400, k = 48, m = 96, nu = 2/2
    "mid_C2": problems.C2.scaled(nx=320),   # n = 102 400, k = 32, m = 64, s1 = 20 (per-row values)
    "mid_C5": problems.C5.scaled(nx=192),   # n = 74 498, k = 64, m = 128 (CSR, clamped edge)
}


def main(names=None):
    ref = Reference(strict=False)
    for name, cfg in MID.items():
        if names and name not in names:
            continue
        t0 = time.perf_counter()
        pb = problems.generate(cfg)
        a = (pb.n, pb.row_ptr, pb.col_idx, pb.values)
        mask = pb.mask if pb.mask.any() else None
        s = ref.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
        u, sig, _, sweeps = ref.svd(s)
        p = np.ascontiguousarray(u[:, : cfg.k])
        t = ref.twolevel(a, p, cfg.omega, cfg.nu1, cfg.nu2)
        res = ref.pcg(a, pb.rhs, 2, t, cfg.delta, 10 * pb.n)
        # the reference's basis_ (after qr_thin) as sketches, its Galerkin A_c
        # (the constructor's own loops) and Cholesky factor: the north star's
        # P / A_c rule at the BASELINE k and m
        basis, chol, _ = t.export()
        coarse = ref.galerkin(t)
        rows = sample_rows(pb.n)
        amax_i, amax_v = col_argmax(basis)
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), config=name, nx=cfg.nx, n=pb.n, k=cfg.k, m=cfg.m,
            sigma=sig, eigh_sweeps=sweeps, x=res.x, iterations=res.iterations, converged=res.converged,
            history=res.history, true_res=res.true_relative_residual,
            basis_sketch=sketch(basis), basis_rows=basis[rows], rows=rows, basis_argmax_idx=amax_i,
            basis_argmax_val=amax_v, svd_p_sketch=sketch(p), coarse=coarse, chol=chol)
        print(f"{name}: n={pb.n} iterations={res.iterations} true_res={res.true_relative_residual:.3e} "
              f"({time.perf_counter() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
