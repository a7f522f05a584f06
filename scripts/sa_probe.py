"""SA build probe (development helper): sa_prolongator + TwoLevelPreconditioner
on an instance directory, timed; run under ncu for the kernel list."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20174_b200 import instance_io as io  # noqa: E402
from paper_2601_20174_b200 import nlsp, sa  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "tests/golden/io/inst_diffusion_n64"
inst = io.load_instance(path)
ctx = nlsp.default_context()
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    t0 = time.time()
    p = sa.sa_prolongator(inst.matrix, 0.25, 0.66)
    ctx.synchronize()
    t1 = time.time()
    m = nlsp.TwoLevelPreconditioner(inst.matrix, p, 0.66, 5, 5)
    ctx.synchronize()
    t2 = time.time()
    res = nlsp.pcg(inst.matrix, inst.rhs, m, 1e-6, 10 * inst.matrix.dim())
    t3 = time.time()
    print(f"nc={p.cols} sa {1e3*(t1-t0):.1f} ms build {1e3*(t2-t1):.1f} ms solve {1e3*(t3-t2):.1f} ms "
          f"iters {res.report.iterations}", flush=True)
