"""numpy prototype of the lean one-pass PCG schedule ("lean
cycle"): on top of the one-pass restriction recurrence, beta is known BEFORE
the pass over W (r.z = r.s + c.e), so the pass writes p directly, and alpha is
known right AFTER it (p.Ap = z.Az - beta * rz / alpha_prev with
z.Az = s.As + 2 e.v + e.Me), so q = A p never has to be stored and the smoother
gathers r_new alone.  Compared against the folded schedule: iteration counts,
relative x difference, and the largest relative deviation of the predicted
p.Ap from the direct one.

usage: python scripts/lean_prototype.py C3 256 48 2     (config, nx, k, nu)
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
        hist = []
        for it in range(10 * n):
            q = A @ p
            a = rz / (p @ q)
            x += a * p
            r -= a * q
            hist.append(np.linalg.norm(r) / bn)
            if hist[-1] < cfg.delta:
                return x, it + 1, np.array(hist)
            z = smooth(r) + W @ (Ainv @ (W.T @ r))
            rzn = r @ z
            p = z + (rzn / rz) * p
            rz = rzn

    def lean():
        x, r = np.zeros(n), b.copy()
        c = W.T @ r
        e = Ainv @ c
        s = smooth(r)
        gam = r @ s + c @ e
        beta = 0.0
        p = s + W @ e
        As = A @ s
        u, v, sig = W.T @ r, W.T @ As, s @ As
        pap = sig + 2 * (e @ v) + e @ (M @ e)
        a = gam / pap
        dev = 0.0
        canc = 0.0
        hist = []
        uprev = aprev = None
        for it in range(10 * n):
            q = A @ p
            direct = p @ q
            dev = max(dev, abs(direct - pap) / direct)
            x += a * p
            r -= a * q
            hist.append(np.linalg.norm(r) / bn)
            if hist[-1] < cfg.delta:
                return x, it + 1, np.array(hist), dev, canc
            g = v + M @ e + (beta * (uprev - u) / aprev if it > 0 else 0.0)
            c = u - a * g
            uprev, aprev = u, a
            e = Ainv @ c
            s = smooth(r)
            gnew = r @ s + c @ e
            beta = gnew / gam
            gam = gnew
            p = s + W @ e + beta * p
            As = A @ s
            u, v, sig = W.T @ r, W.T @ As, s @ As
            delta = sig + 2 * (e @ v) + e @ (M @ e)
            pap = delta - beta * gam / aprev
            canc = max(canc, delta / pap)
            a = gam / pap

    x1, i1, h1 = folded()
    x2, i2, h2, dev, canc = lean()
    m = min(len(h1), len(h2))
    out = {"n": n, "folded": i1, "lean": i2, "x_diff": float(np.linalg.norm(x2 - x1) / np.linalg.norm(x1)),
           "hist_dev": float(np.max(np.abs(h2[:m] - h1[:m]) / h1[:m])), "pap_dev": float(dev), "cancellation": float(canc)}
    print(f"{name} n={n} iterations folded={i1} lean={i2} "
          f"rel x diff={np.linalg.norm(x2 - x1) / np.linalg.norm(x1):.2e} "
          f"history dev={np.max(np.abs(h2[:m] - h1[:m]) / h1[:m]):.2e} "
          f"max rel dev of p.Ap={dev:.2e} max cancellation={canc:.1f}")
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    main(args[0] if args else "C3", *(int(v) for v in args[1:4]))
