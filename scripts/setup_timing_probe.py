"""Replicates bench.py's setup timing (events on the context stream) with host
times alongside (development helper)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20174_b200 import nlsp, problems  # noqa: E402

cfg = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ctx = nlsp.default_context()
pb = problems.generate(cfg)
a = pb.csr()
a.device(ctx)
mask = pb.mask if pb.mask.any() else None
s0 = problems.smoothed_s0(cfg.s0_seed, pb.n, cfg.m, mask)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
for rep in range(3):
    s = nlsp.DeviceDense.upload(s0, ctx)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ctx.synchronize()
    h = [time.perf_counter()]
    ev[0].record(stream)
    nlsp.smooth_vectors(a, s, cfg.s1, cfg.omega)
    h.append(time.perf_counter())
    ev[1].record(stream)
    p, sigma, sweeps = nlsp.svd_basis(s, cfg.k, ctx)
    h.append(time.perf_counter())
    ev[2].record(stream)
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    h.append(time.perf_counter())
    ev[3].record(stream)
    ctx.synchronize()
    h.append(time.perf_counter())
    print(f"rep {rep}: events smooth {ev[0].elapsed_time(ev[1]):.1f} svd {ev[1].elapsed_time(ev[2]):.1f} "
          f"build {ev[2].elapsed_time(ev[3]):.1f} ms | host smooth {1e3*(h[1]-h[0]):.1f} svd {1e3*(h[2]-h[1]):.1f} "
          f"build {1e3*(h[3]-h[2]):.1f} tail {1e3*(h[4]-h[3]):.1f} ms", flush=True)
    del s, p, m
