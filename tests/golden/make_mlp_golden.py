"""tests/golden/make_mlp_golden.py — golden fixtures for MLP inference (SURVEY
§8f.4), produced by the REFERENCE ITSELF (oracle/_ref: MlpModel, save/load,
forward, infer_basis, TwoLevelPreconditioner, pcg from the reference headers).

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_mlp_golden.py

Outputs under tests/golden/mlp/ (committed):
  small.ckpt        MlpModel([40, 16, 8, 24], seed 5).save(...) by the reference
  small.npz         its parameters as the reference loads them, a random input
                    and the reference's forward output
  n32_nlss.npz      bench_single's NLSS row (pipeline.hpp:303-346) on
                    tests/golden/io/inst_diffusion_n32 with an untrained model of
                    the default widths (train.hpp:28-32) from seed 77: the
                    reference's infer_basis Q (n x K), the rank-8 two-level PCG
                    (nu 5/5, delta 1e-6) iterations and solution
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mlp")


def main():
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)
    small = os.path.join(OUT, "small.ckpt")
    ref.mlp_create_save([40, 16, 8, 24], 5, small)
    x = np.random.default_rng(3).standard_normal(40)
    np.savez_compressed(os.path.join(OUT, "small.npz"), widths=np.array([40, 16, 8, 24]), seed=5,
                        params=ref.mlp_params(small), x=x, y=ref.mlp_forward(small, x, 24))

    io = np.load(os.path.join(os.path.dirname(OUT), "io", "n32_svd.npz"))
    inst = ref.load_instance(os.path.join(os.path.dirname(OUT), "io", "inst_diffusion_n32"))
    a = inst["matrix"]
    n, K = io["S"].shape
    widths = [n * K, 128, 256, 256, 128, n * K]
    seed = 77
    with tempfile.TemporaryDirectory() as d:
        ck = os.path.join(d, "m.ckpt")
        ref.mlp_create_save(widths, seed, ck)
        q, ms = ref.infer_basis(ck, io["S"], K)
    rank = 8
    t = ref.twolevel(a, np.ascontiguousarray(q[:, :rank]), 0.66, 5, 5)
    res = ref.pcg(a, inst["rhs"], 2, t, 1e-6, 10 * n)
    np.savez_compressed(os.path.join(OUT, "n32_nlss.npz"), widths=np.array(widths), seed=seed, Q=q,
                        rank=rank, iterations=res.iterations, x=res.x, converged=res.converged,
                        ref_infer_ms=ms)
    print("mlp golden fixtures written to", OUT, "ref infer_basis ms", ms, "iters", res.iterations)


if __name__ == "__main__":
    main()
