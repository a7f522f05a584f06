"""Setup-phase probe (development helper): smoothing, svd_basis, two-level
build for one config, timed with host syncs; run under ncu for a kernel list."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20174_b200 import nlsp, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = problems.CONFIGS[name]
pb = problems.generate(cfg)
a = pb.csr()
ctx = nlsp.default_context()
a.device()
for r in range(reps):
    t0 = time.time()
    sv = nlsp.generate_smoothed_vectors(a, pb.mask if pb.mask.any() else None, cfg.m, cfg.s1, cfg.omega,
                                        cfg.s0_seed)
    ctx.synchronize()
    t1 = time.time()
    p, sig, sw = nlsp.svd_basis(sv.s, cfg.k)
    ctx.synchronize()
    t2 = time.time()
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    ctx.synchronize()
    t3 = time.time()
    print(f"{name} rep {r}: smooth(+host S0) {1e3*(t1-t0):.1f} ms  svd_basis {1e3*(t2-t1):.1f} ms "
          f"(sweeps {sw})  build {1e3*(t3-t2):.1f} ms", flush=True)
