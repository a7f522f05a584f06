"""tests/golden/make_sa_golden.py — golden fixtures for the SA coarse space
(SURVEY §8f.3), produced by the REFERENCE ITSELF (oracle/_ref: aggregate_nodes,
sa_prolongator, TwoLevelPreconditioner, pcg from the reference headers).

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_sa_golden.py

Outputs: tests/golden/sa/sa.npz with, per case (the io instances of all three
families at N = 8, a diffusion instance at N = 16, and inst_diffusion_n32):
aggregate ids and count, P (not for n32: 1089 x 551), and bench_single's SA
row (pipeline.hpp:316-317: theta 0.25, omega 0.66, nu 5/5, delta 1e-6):
iterations, converged, x.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402

GOLDEN = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(GOLDEN, "sa")


def main():
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)
    cases = {}
    for name in ("inst_diffusion_n8", "inst_anisotropic_n8", "inst_screened_poisson_n8", "inst_diffusion_n32"):
        inst = ref.load_instance(os.path.join(GOLDEN, "io", name))
        cases[name] = (inst["matrix"], inst["rhs"])
    a16, rhs16, _ = ref.fem_instance(0, 16, 0.25, 41)
    cases["fem_diffusion_n16"] = (a16, rhs16)
    out = {"names": np.array(list(cases))}
    for name, (a, rhs) in cases.items():
        agg, nc = ref.aggregate_nodes(a, 0.25)
        p = ref.sa_prolongator(a, 0.25, 0.66)
        t = ref.twolevel(a, p, 0.66, 5, 5)
        res = ref.pcg(a, rhs, 2, t, 1e-6, 10 * a[0])
        out[f"{name}__agg"], out[f"{name}__nc"] = agg, nc
        if name != "inst_diffusion_n32":
            out[f"{name}__P"] = p
        out[f"{name}__iterations"] = res.iterations
        out[f"{name}__converged"] = res.converged
        out[f"{name}__x"] = res.x
        if name == "fem_diffusion_n16":
            n, rp, ci, v = a
            out[f"{name}__n"], out[f"{name}__rp"], out[f"{name}__ci"], out[f"{name}__v"] = n, rp, ci, v
            out[f"{name}__rhs"] = rhs
        print(name, "n", a[0], "nc", nc, "iters", res.iterations)
    np.savez_compressed(os.path.join(OUT, "sa.npz"), **out)


if __name__ == "__main__":
    main()
