"""tests/golden/make_full_golden.py — FULL-SIZE goldens for BASELINE.json's
configurations C2–C5, produced by the REFERENCE ITSELF (oracle/_ref/libnlsp_ref.so,
the reference's unmodified headers; TEST INFRASTRUCTURE).

Each run is bench_single's SVD row end to end at the benchmarked size
(pipeline.hpp:303-346):

    generate_smoothed_vectors(A, mask, m, s1, omega, seed)   smoothing.hpp:81-100
    svd_oracle(S) -> first_cols(U, k)                        svd.hpp:155-227
    TwoLevelPreconditioner(A, P, omega, nu1, nu2)            two_level.hpp:24-53
    pcg(A, b, M, 1e-8, 10 n)                                 two_level.hpp:141-191

The inputs are regenerated bit-identically from the seeded generators, so only
outputs are stored: iterations, the whole residual history, the true residual,
sigma, the reference's basis_ as sketches (tests/golden/sketch.py), its
Galerkin A_c (recomputed by the constructor's own loops, ref_twolevel_galerkin)
and Cholesky factor L, and x (in full for C2/C5, as a sketch + row sample for
C3/C4). The wall time of every reference phase (one core) is kept as well.

Run here (where /root/reference exists), one process per config, e.g.
    make -C oracle ref
    for c in C2 C3 C4 C5; do python tests/golden/make_full_golden.py $c & done
C4 takes about 40 min, C3 about 2 h on one core.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle.oracle import Reference  # noqa: E402
from paper_2601_20174_b200 import problems  # noqa: E402
from sketch import col_argmax, sample_rows, sketch  # noqa: E402

FULL_X = {"C2", "C5"}


def run(name: str) -> None:
    cfg = problems.CONFIGS[name]
    ref = Reference(strict=False)
    times = {}
    t0 = time.perf_counter()
    pb = problems.generate(cfg)
    a = (pb.n, pb.row_ptr, pb.col_idx, pb.values)
    mask = pb.mask if pb.mask.any() else None
    t = time.perf_counter()
    s = ref.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
    times["smooth_s"] = time.perf_counter() - t
    print(f"{name}: smoothed ({times['smooth_s']:.0f} s)", flush=True)
    t = time.perf_counter()
    u, sig, _, sweeps = ref.svd(s)
    times["svd_s"] = time.perf_counter() - t
    del s
    p = np.ascontiguousarray(u[:, : cfg.k])
    del u
    print(f"{name}: svd ({times['svd_s']:.0f} s)", flush=True)
    t = time.perf_counter()
    tl = ref.twolevel(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    times["build_s"] = time.perf_counter() - t
    print(f"{name}: build ({times['build_s']:.0f} s)", flush=True)
    basis, chol, _ = tl.export()
    t = time.perf_counter()
    coarse = ref.galerkin(tl)
    times["galerkin_s"] = time.perf_counter() - t
    t = time.perf_counter()
    res = ref.pcg(a, pb.rhs, 2, tl, cfg.delta, 10 * pb.n)
    times["pcg_s"] = time.perf_counter() - t
    print(f"{name}: pcg {res.iterations} iterations ({times['pcg_s']:.0f} s)", flush=True)

    rows = sample_rows(pb.n)
    amax_i, amax_v = col_argmax(basis)
    out = dict(
        config=name, n=pb.n, nnz=pb.nnz, k=cfg.k, m=cfg.m, s1=cfg.s1, nu1=cfg.nu1, nu2=cfg.nu2,
        sigma=sig, eigh_sweeps=sweeps,
        svd_p_sketch=sketch(p), svd_p_rows=p[rows],
        basis_sketch=sketch(basis), basis_rows=basis[rows], basis_argmax_idx=amax_i,
        basis_argmax_val=amax_v, coarse=coarse, chol=chol,
        iterations=res.iterations, converged=res.converged, history=res.history,
        true_res=res.true_relative_residual, x_norm=np.linalg.norm(res.x),
        x_sketch=sketch(res.x), x_rows=res.x[rows], rows=rows,
        ref_times=np.array([times[k] for k in ("smooth_s", "svd_s", "build_s", "galerkin_s", "pcg_s")]),
        ref_time_keys=np.array(["smooth_s", "svd_s", "build_s", "galerkin_s", "pcg_s"]),
        pcg_ms=res.solve_ms)
    if name in FULL_X:
        out["x"] = res.x
    np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), **out)
    print(f"{name}: n={pb.n} iterations={res.iterations} true_res={res.true_relative_residual:.3e} "
          f"total {time.perf_counter() - t0:.0f} s  {times}", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
        run(nm)
