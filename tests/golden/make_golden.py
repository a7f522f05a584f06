"""tests/golden/make_golden.py — regenerates the committed golden fixtures from
the REFERENCE ITSELF (oracle/_ref/libnlsp_ref*.so: the reference's own headers
under /root/reference/proj/include, compiled by oracle/Makefile).

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py

Outputs (small, compressed .npz, committed):
  rng.npz            Rng/mix_seed streams (rng.hpp)
  kat.npz            the hand-checked cases of the reference's unit tests
  c1_default.npz     config C1 end to end through the default build
  c1_strict.npz      the same through the -ffp-contract=off build
  scaled_<Cx>.npz    scaled-down C2..C5 families end to end (default build)
  fem_diffusion.npz  make_instance(Diffusion, 16, 0.25, 23) + the two-level
                     PCG of Pcg.TwoLevelBeatsUnpreconditionedOnDiffusion
  random_spd.npz     random sparse SPD systems with random orthonormal bases
                     (TwoLevel.CoarseExactnessWithoutSmoothing style)
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2601_20174_b200 import problems  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# scaled-down families: the same generators at sizes the reference solves in seconds
SCALED = {
    "C2": problems.C2.scaled(nx=48, k=8, m=16, s1=20),
    "C3": problems.C3.scaled(nx=40, k=8, m=16, s1=10),
    "C4": problems.C4.scaled(nx=14, k=12, m=24, s1=10),
    "C5": problems.C5.scaled(nx=16, k=12, m=24, s1=10, blocks=4),
}


def csr_tuple(pb):
    return (pb.n, pb.row_ptr, pb.col_idx, pb.values)


def pipeline(ref, cfg, pb, mask=None):
    """generate_smoothed_vectors -> svd_oracle -> first_cols -> TwoLevel -> pcg,
    exactly bench_single's SVD row (pipeline.hpp:303-346)."""
    a = csr_tuple(pb)
    s = ref.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
    u, sig, v, sweeps = ref.svd(s)
    p = np.ascontiguousarray(u[:, : cfg.k])
    t = ref.twolevel(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    basis, chol, coarse_llt = t.export()
    coarse = ref.galerkin(t)
    res = ref.pcg(a, pb.rhs, 2, t, cfg.delta, 10 * pb.n)
    plain = ref.pcg(a, pb.rhs, 0, None, cfg.delta, 10 * pb.n)
    rng = np.random.default_rng(1234)
    r_probe = rng.standard_normal(pb.n)
    z_probe = t.apply(r_probe)
    return dict(
        n=pb.n, row_ptr=pb.row_ptr, col_idx=pb.col_idx, values=pb.values, rhs=pb.rhs,
        mask=pb.mask, k=cfg.k, m=cfg.m, s1=cfg.s1, nu1=cfg.nu1, nu2=cfg.nu2, omega=cfg.omega,
        delta=cfg.delta, s0_seed=cfg.s0_seed, S=s, sigma=sig, eigh_sweeps=sweeps, P=p,
        basis=basis, chol=chol, coarse=coarse, x=res.x, iterations=res.iterations,
        converged=res.converged, history=res.history, true_res=res.true_relative_residual,
        plain_iterations=plain.iterations, r_probe=r_probe, z_probe=z_probe,
    )


def main():
    ref = Reference(strict=False)
    strict = Reference(strict=True)

    # rng.hpp streams
    np.savez_compressed(
        os.path.join(OUT, "rng.npz"),
        mix=np.array([ref.mix_seed(s, t) for s, t in [(0, 0), (7, 0x736d6f6f), (2601, 0x726873),
                                                       (2**64 - 1, 12345)]], dtype=np.uint64),
        u64_seed5=ref.rng_u64(5, 700),
        normal_seed5=ref.rng_normal(5, 1001),
        normal_seed_smoo7=ref.rng_normal(ref.mix_seed(7, 0x736d6f6f), 4097),
        uniform_seed9=ref.rng_uniform(9, 513, -1.0, 1.0),
    )

    # hand-checked cases (test_linalg.cpp / test_smoothing.cpp / test_two_level.cpp)
    kat = {}
    kat["chol_2x2_x"] = ref.cholesky_solve(np.array([[4.0, 2.0], [2.0, 3.0]]), np.array([4.0, 2.0]))
    q, r = ref.qr_thin(np.array([[3.0], [4.0]]))
    kat["qr_3_4_q"], kat["qr_3_4_r"] = q, r
    s = np.zeros((3, 2))
    s[0, 0], s[1, 1] = 3.0, 2.0
    u, sig, v, _ = ref.svd(s)
    kat["svd_diag_u"], kat["svd_diag_sigma"] = u, sig
    a = ref.from_triplets(2, [0, 0, 1, 1], [0, 1, 0, 1], [2.0, -1.0, -1.0, 2.0])
    kat["stencil_y"] = ref.spmv(a, np.ones(2))
    dd = ref.from_triplets(2, [0, 0, 0], [1, 0, 1], [1.0, 2.0, 0.5])
    kat["dedup_rp"], kat["dedup_ci"], kat["dedup_v"] = dd[1], dd[2], dd[3]
    eye5 = ref.from_triplets(5, range(5), range(5), [1.0] * 5)
    kat["jacobi_eye_x"] = ref.jacobi_sweep(eye5, 0.3, 1, np.array([1.0, -2.0, 3.0, 0.5, -1.5]), np.zeros(5))
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **kat)

    # C1 end to end, both reference builds
    pb = problems.generate(problems.C1)
    np.savez_compressed(os.path.join(OUT, "c1_default.npz"), **pipeline(ref, problems.C1, pb))
    np.savez_compressed(os.path.join(OUT, "c1_strict.npz"), **pipeline(strict, problems.C1, pb))

    # scaled families
    for name, cfg in SCALED.items():
        pbs = problems.generate(cfg)
        mask = pbs.mask if pbs.mask.any() else None
        np.savez_compressed(os.path.join(OUT, f"scaled_{name}.npz"), **pipeline(ref, cfg, pbs, mask))

    # P1 FEM diffusion instance (fem.hpp:223-236) and the reference test's solve
    (n, rp, ci, v), rhs, mask = ref.fem_instance(0, 16, 0.25, 23)
    a = (n, rp, ci, v)
    s = ref.generate_smoothed_vectors(a, mask, 16, 10, 0.66, 29)
    u = ref.svd(s)[0][:, :8]
    t = ref.twolevel(a, np.ascontiguousarray(u), 0.66, 5, 5)
    two = ref.pcg(a, rhs, 2, t, 1e-6, 10 * n)
    plain = ref.pcg(a, rhs, 0, None, 1e-6, 10 * n)
    jac = ref.pcg(a, rhs, 1, None, 1e-8, 5000)
    np.savez_compressed(
        os.path.join(OUT, "fem_diffusion.npz"), n=n, row_ptr=rp, col_idx=ci, values=v, rhs=rhs,
        mask=mask, S=s, P=u, basis=t.export()[0], coarse=ref.galerkin(t), x=two.x,
        iterations=two.iterations, true_res=two.true_relative_residual, history=two.history,
        plain_iterations=plain.iterations, plain_x=plain.x, jacobi_iterations=jac.iterations,
        jacobi_x=jac.x)

    # random sparse SPD + random orthonormal bases (nu = 0 coarse exactness, apply)
    rng = np.random.default_rng(505)
    cases = {}
    for trial in range(6):
        n = int(rng.integers(20, 120))
        nc = int(rng.integers(1, 9))
        dense = np.zeros((n, n))
        iu = np.triu_indices(n, 1)
        pick = rng.random(iu[0].size) < 0.08
        vals = rng.standard_normal(pick.sum())
        dense[iu[0][pick], iu[1][pick]] = vals
        dense = dense + dense.T + np.diag(6.0 + rng.random(n))
        ii, jj = np.nonzero(dense)
        a = ref.from_triplets(n, ii, jj, dense[ii, jj])
        basis = np.linalg.qr(rng.standard_normal((n, nc)))[0]
        t = ref.twolevel(a, basis, 0.66, 0, 0)
        t2 = ref.twolevel(a, basis, 0.66, 2, 2)
        r = rng.standard_normal(n)
        cases[f"t{trial}_n"] = n
        cases[f"t{trial}_rp"], cases[f"t{trial}_ci"], cases[f"t{trial}_v"] = a[1], a[2], a[3]
        cases[f"t{trial}_basis_in"] = basis
        cases[f"t{trial}_basis"] = t.export()[0]
        cases[f"t{trial}_coarse"] = ref.galerkin(t)
        cases[f"t{trial}_r"] = r
        cases[f"t{trial}_z0"] = t.apply(r)
        cases[f"t{trial}_z2"] = t2.apply(r)
    np.savez_compressed(os.path.join(OUT, "random_spd.npz"), trials=6, **cases)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
