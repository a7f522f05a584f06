"""Device time of the setup smoothing sweeps alone (development helper):
S^(0) uploaded once, then `reps` x nlsp_smooth_vectors(s1 sweeps), host-synced.
  python scripts/sweep_probe.py [C4] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20174_b200 import nlsp, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = problems.CONFIGS[name]
pb = problems.generate(cfg)
a = pb.csr()
ctx = nlsp.default_context()
s0 = problems.smoothed_s0(cfg.s0_seed, pb.n, cfg.m, pb.mask if pb.mask.any() else None)
s = nlsp.DeviceDense.upload(s0, ctx)
for r in range(reps):
    ctx.synchronize()
    t0 = time.perf_counter()
    nlsp.smooth_vectors(a, s, cfg.s1, cfg.omega)
    ctx.synchronize()
    print(f"{name}: {cfg.s1} sweeps of n={pb.n} x m={cfg.m}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
