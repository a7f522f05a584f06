"""tests/golden/make_io_golden.py — golden fixtures for the on-disk input path
(SURVEY §8f.2), produced by the REFERENCE ITSELF (oracle/_ref/libnlsp_ref.so:
the reference headers' make_instance / save_instance / load_instance /
load_matrix_market and the bench_single SVD pipeline, compiled by
oracle/Makefile).

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_io_golden.py

Outputs under tests/golden/io/ (committed):
  inst_<family>_n8/         instance directories written by save_instance
  inst_diffusion_n32/       (instance_io.hpp:99-135), family x N as named
  inst_diffusion_n64/
  instances.npz             load_instance of each directory (reference arrays)
  mtx/<case>.mtx            MatrixMarket edge cases (text written here)
  mtx_expected.npz          load_matrix_market outcome per case: status code
                            (0 ok, 1 ValidationError, 8 IoError) + CSR arrays
  n32_svd.npz               bench_single's SVD row on inst_diffusion_n32
                            (pipeline.hpp:303-346 with the ExperimentConfig
                            defaults: K=32, s1=10, omega=0.66, nu=5/5,
                            delta=1e-6) at ranks 4/8/16/32, plus plain CG
"""
from __future__ import annotations

import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import OracleError, Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")

INSTANCES = {
    # dir name: (family, N, jitter, seed)
    "inst_diffusion_n8": (0, 8, 0.25, 101),
    "inst_anisotropic_n8": (1, 8, 0.25, 102),
    "inst_screened_poisson_n8": (2, 8, 0.25, 103),
    "inst_diffusion_n32": (0, 32, 0.25, None),  # seed: test_seed(0) of the default config
    "inst_diffusion_n64": (0, 64, 0.25, None),  # the paper's Tables 1-3 size (bench_instance.py)
}

H = "%%MatrixMarket matrix coordinate real "
MTX = {
    "general": H + "general\n3 3 4\n1 1 2.0\n2 2 3.5\n3 1 -1e-3\n3 3 4\n",
    "symmetric_comments": H + "symmetric\n% a comment\n%another\n3 3 4\n1 1 4\n2 1 -1\n2 2 4\n3 2 -1.25\n",
    "duplicates2": H + "general\n2 2 3\n1 1 1.5\n1 1 2.25\n2 2 1\n",
    "duplicates3_order": H + "general\n2 2 4\n2 1 1e16\n2 1 1.0\n2 1 -1e16\n1 1 1\n",
    "explicit_zeros": H + "general\n2 2 4\n1 1 0.0\n1 2 -0.0\n2 1 3\n2 2 1\n",
    "blank_size_line": H + "general\n\n1 1 1.0\n",
    "skew_symmetric": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 1.5\n3 2 -2\n",
    "bad_header": "%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n",
    "array_format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "nonsquare": H + "general\n2 3 1\n1 1 1\n",
    "truncated": H + "general\n3 3 3\n1 1 1\n2 2 2\n",
    "index_zero": H + "general\n2 2 1\n0 1 1.0\n",
    "index_too_big": H + "general\n3 3 1\n5 1 1.0\n",
    "index_negative": H + "general\n3 3 1\n-1 1 1.0\n",
    "number_forms": H + "general\n4 4 5\n1 1 +1.5E+02\n2 2 -.5\n3 3 5.\n4 4 1e-310\n4 1 +7\n",
    "exponent_without_digits": H + "general\n2 2 2\n1 1 2.5e\n2 2 1\n",
    "nan_value": H + "general\n2 2 1\n1 1 nan\n",
    "overflow_value": H + "general\n2 2 1\n1 1 1e999\n",
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n1 1\n2 1\n",
    "crlf_tabs": H + "symmetric\r\n3\t3\t2\r\n1\t1\t2.5\r\n3 1\t-1\r\n",
    "trailing_garbage": H + "general\n2 2 2\n1 1 1\n2 2 2\nthis is not read\n",
    "entry_split_across_lines": H + "general\n2 2 2\n1\n1\n2.0 2 2\n3.0\n",
    "garbage_in_entry": H + "general\n2 2 2\n1 1 1\n2x 2 2\n",
    "empty_file": "",
    "header_only": H + "general\n",
    "leading_plus": H + "general\n2 2 2\n+1 +1 +3.0\n+2 +2 1\n",
    "comments_then_eof": H + "general\n% only comments\n",
    "zero_dim": H + "general\n0 0 0\n",
}


def main():
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)
    # --- instance directories (save_instance) + their reference loads
    arrays = {}
    for name, (fam, n, jit, seed) in INSTANCES.items():
        if seed is None:
            seed = int(ref.lib.ref_mix_seed(1, 50))  # ExperimentConfig::test_seed(0), seed 1, 50 train
        d = os.path.join(OUT, name)
        shutil.rmtree(d, ignore_errors=True)
        ref.save_instance(fam, n, jit, seed, d)
        inst = ref.load_instance(d)
        dim, rp, ci, v = inst["matrix"]
        for key in ("family", "grid_n", "seed", "jitter", "alpha"):
            arrays[f"{name}__{key}"] = np.array(inst[key])
        arrays[f"{name}__n"] = np.array(dim)
        arrays[f"{name}__rp"], arrays[f"{name}__ci"], arrays[f"{name}__v"] = rp, ci, v
        for key in ("rhs", "mask", "vertices", "triangles", "coefficients"):
            arrays[f"{name}__{key}"] = inst[key]
    np.savez_compressed(os.path.join(OUT, "instances.npz"), names=np.array(list(INSTANCES)), **arrays)

    # --- MatrixMarket edge cases (load_matrix_market)
    mdir = os.path.join(OUT, "mtx")
    shutil.rmtree(mdir, ignore_errors=True)
    os.makedirs(mdir)
    exp = {}
    for name, text in MTX.items():
        path = os.path.join(mdir, name + ".mtx")
        with open(path, "w", newline="") as f:
            f.write(text)
        try:
            dim, rp, ci, v = ref.load_matrix_market(path)
            exp[f"{name}__status"] = np.array(0)
            exp[f"{name}__n"] = np.array(dim)
            exp[f"{name}__rp"], exp[f"{name}__ci"], exp[f"{name}__v"] = rp, ci, v
        except OracleError as e:
            exp[f"{name}__status"] = np.array(e.code)
            exp[f"{name}__message"] = np.array(e.message.replace(mdir, "<dir>"))
    np.savez_compressed(os.path.join(OUT, "mtx_expected.npz"), names=np.array(list(MTX)), **exp)

    # --- bench_single SVD rows on the N=32 instance (pipeline.hpp:303-346)
    d = os.path.join(OUT, "inst_diffusion_n32")
    inst = ref.load_instance(d)
    a = inst["matrix"]
    K, s1, omega, nu, delta = 32, 10, 0.66, 5, 1e-6
    sseed = int(ref.lib.ref_mix_seed(inst["seed"], 3))  # ExperimentConfig::smoothing_seed
    s = ref.generate_smoothed_vectors(a, inst["mask"], K, s1, omega, sseed)
    u, sig, _, _ = ref.svd(s)
    out = dict(K=K, s1=s1, omega=omega, nu=nu, delta=delta, smoothing_seed=sseed, S=s, sigma=sig,
               ranks=np.array([4, 8, 16, 32]))
    for r in (4, 8, 16, 32):
        p = u[:, :r].copy()
        t = ref.twolevel(a, p, omega, nu, nu)
        res = ref.pcg(a, inst["rhs"], 2, t, delta, 10 * a[0])
        out[f"r{r}_P"] = p
        out[f"r{r}_iterations"] = res.iterations
        out[f"r{r}_x"] = res.x
        out[f"r{r}_true"] = res.true_relative_residual
        out[f"r{r}_converged"] = res.converged
    plain = ref.pcg(a, inst["rhs"], 0, None, delta, 10 * a[0])
    out["plain_iterations"] = plain.iterations
    out["plain_x"] = plain.x
    np.savez_compressed(os.path.join(OUT, "n32_svd.npz"), **out)
    print("io golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
