"""Prints the GPU's bench_single SVD row against the reference's mid-size
goldens (tests/golden/mid_*.npz): iterations, solution error, singular values
(development helper; tests/test_gpu_midsize.py asserts the tolerances)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import golden
from paper_2601_20174_b200 import problems, nlsp
for name in ["mid_C4", "mid_C3", "mid_C2", "mid_C5"]:
    d = golden(name); cfg = problems.CONFIGS[name[4:]].scaled(nx=int(d["nx"])); pb = problems.generate(cfg); a = pb.csr()
    mask = pb.mask if pb.mask.any() else None
    sv = nlsp.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
    p, sig, _ = nlsp.svd_basis(sv.s, cfg.k)
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    r = nlsp.pcg(a, pb.rhs, m, cfg.delta, 10 * pb.n)
    x = d["x"]
    print(name, "n", pb.n, "iters gpu", r.report.iterations, "ref", int(d["iterations"]), "x rel err %.2e" % (np.linalg.norm(r.solution - x) / np.linalg.norm(x)),
          "sigma rel %.2e" % (np.abs(np.asarray(sig) - d["sigma"][:len(sig)]).max() / d["sigma"][0]), "true res %.2e" % r.report.true_relative_residual)
