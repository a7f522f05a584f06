"""numpy prototype of the one-pass PCG schedule, used to check
its numerics before the CUDA kernels were written: PCG with the folded
two-level operator z = S_T(r) + W A_c^-1 W^T r against the same PCG with the
restriction carried by its recurrence

    c_{i+1} = u_i - alpha_i (v_i + M e_i + beta_i (u_{i-1} - u_i) / alpha_{i-1}),
    u_i = W^T r_i,  v_i = W^T A s_i,  M = W^T A W,

on a scaled instance of a BASELINE configuration. Prints both iteration counts,
the relative difference of the solutions and the largest relative deviation of
the recurrence c from the direct W^T r.

usage: python scripts/onepass_prototype.py C3 256 48 2     (config, nx, k, nu)
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20174_b200 import problems  # noqa: E402


def main(name="C3", nx=256, k=48, nu=2):
    cfg = problems.CONFIGS[name].scaled(nx=nx, k=k, nu1=nu, nu2=nu)
    pb = problems.generate(cfg)
    A = sp.csr_matrix((pb.values, pb.col_idx.astype(np.int64), pb.row_ptr.astype(np.int64)), shape=(pb.n, pb.n))
    n = pb.n
    rng = np.random.default_rng(0)
    wd = (2 / 3) / A.diagonal()
    S = rng.standard_normal((n, 2 * k))
    for _ in range(10):
        S = S - wd[:, None] * (A @ S)
    P = np.linalg.svd(S, full_matrices=False)[0][:, :k]
    Ac = P.T @ (A @ P)
    Ainv = np.linalg.inv(0.5 * (Ac + Ac.T))
    W = P.copy()
    for _ in range(nu):
        W = W - wd[:, None] * (A @ W)
    M = W.T @ (A @ W)

    def smooth(r):
        s = wd * r
        for _ in range(2 * nu - 1):
            s = s + wd * (r - A @ s)
        return s

    b = pb.rhs
    bn = np.linalg.norm(b)

    def folded():
        x, r = np.zeros(n), b.copy()
        z = smooth(r) + W @ (Ainv @ (W.T @ r))
        p, rz = z.copy(), r @ z
        for it in range(10 * n):
            q = A @ p
            a = rz / (p @ q)
            x += a * p
            r -= a * q
            if np.linalg.norm(r) / bn < cfg.delta:
                return x, it + 1
            z = smooth(r) + W @ (Ainv @ (W.T @ r))
            rzn = r @ z
            p = z + (rzn / rz) * p
            rz = rzn

    def onepass():
        x, r = np.zeros(n), b.copy()
        e = Ainv @ (W.T @ r)
        s = smooth(r)
        z = s + W @ e
        u, v = W.T @ r, W.T @ (A @ s)
        p, rz, beta, dev = z.copy(), r @ z, 0.0, 0.0
        uprev = aprev = None
        for it in range(10 * n):
            q = A @ p
            a = rz / (p @ q)
            x += a * p
            r -= a * q
            if np.linalg.norm(r) / bn < cfg.delta:
                return x, it + 1, dev
            g = v + M @ e + (beta * (uprev - u) / aprev if it > 0 else 0.0)
            c = u - a * g
            ct = W.T @ r
            dev = max(dev, np.linalg.norm(c - ct) / np.linalg.norm(ct))
            uprev, aprev = u, a
            e = Ainv @ c
            s = smooth(r)
            z = s + W @ e
            u, v = W.T @ r, W.T @ (A @ s)
            rzn = r @ z
            beta = rzn / rz
            p = z + beta * p
            rz = rzn

    x1, i1 = folded()
    x2, i2, dev = onepass()
    print(f"{name} n={n} iterations folded={i1} onepass={i2} "
          f"rel x diff={np.linalg.norm(x2 - x1) / np.linalg.norm(x1):.2e} max rel dev of c={dev:.2e}")


if __name__ == "__main__":
    args = sys.argv[1:]
    main(args[0] if args else "C3", *(int(v) for v in args[1:4]))
