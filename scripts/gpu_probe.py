"""Quick GPU probe: one config end to end with timings (development helper)."""
import sys, time, json, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20174_b200 import nlsp, problems, _lib as L
import ctypes as C

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = problems.CONFIGS[name]
t0 = time.time(); pb = problems.generate(cfg); tg = time.time() - t0
print(f"{name}: n={pb.n} nnz={pb.nnz} gen {tg:.1f}s", flush=True)
a = pb.csr()
ctx = nlsp.default_context()
t0 = time.time(); dev = a.device(); print(f"upload {time.time()-t0:.2f}s", flush=True)
t0 = time.time()
sv = nlsp.generate_smoothed_vectors(a, pb.mask if pb.mask.any() else None, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
ctx.synchronize(); print(f"smooth (incl host S0) {time.time()-t0:.2f}s", flush=True)
t0 = time.time(); p, sig, sw = nlsp.svd_basis(sv.s, cfg.k); ctx.synchronize()
print(f"svd_basis {time.time()-t0:.3f}s sweeps={sw} sigma[k-1:k+1]={sig[cfg.k-1:cfg.k+1]}", flush=True)
t0 = time.time(); m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2); ctx.synchronize()
print(f"build {time.time()-t0:.3f}s", flush=True)
for r in range(reps):
    res = nlsp.pcg(a, pb.rhs, m, cfg.delta, 10 * pb.n)
    rep = res.report
    print(f"solve {r}: iters={rep.iterations} conv={rep.converged} true={rep.true_relative_residual:.3e} "
          f"solve_ms={rep.solve_ms:.2f} total_ms={rep.total_ms:.2f} ms/iter={rep.solve_ms/max(rep.iterations,1):.4f}", flush=True)
# per-kernel profile
bdev = C.c_void_p()
import ctypes
lib = L.gpu_lib()
# upload b via a dense handle
bd = nlsp.DeviceDense.upload(pb.rhs.reshape(-1, 1))
class _DD(ctypes.Structure): pass
stats = (L.KernelStatC * 8)()
# device pointer of bd: not exposed; use a profile through pcg_device API needs a device ptr
xd = nlsp.DeviceDense.upload(np.zeros((pb.n, 1)))
iters = 20
nk = lib.nlsp_pcg_profile(ctx.handle, dev.handle, 2, m.handle, bd.data_ptr, iters, stats, 8)
tot = 0.0
rows = []
for i in range(nk):
    s = stats[i]
    per = s.total_ms / s.launches
    tot += per
    gbs = s.bytes_per_launch / (per * 1e-3) / 1e9 if per > 0 else 0
    rows.append((s.name.decode(), per, s.bytes_per_launch / 1e6, gbs))
for r in rows:
    print(f"  {r[0]:12s} {r[1]*1e3:9.1f} us  {r[2]:9.1f} MB  {r[3]:8.1f} GB/s")
print(f"  sum {tot*1e3:.1f} us/iter (stepwise)")
rep = L.SolveReportC()
t0 = time.time()
st = lib.nlsp_pcg_device(ctx.handle, dev.handle, 2, m.handle, bd.data_ptr, cfg.delta, 10 * pb.n, xd.data_ptr, C.byref(rep), None)
print("pcg_device", st, rep.iterations, rep.solve_ms, rep.total_ms)
