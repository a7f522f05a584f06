cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/t.py <<'PY'
import sys, time, numpy as np, ctypes as C
sys.path.insert(0, '.')
from paper_2601_20174_b200 import problems, nlsp, _lib as L
for name in sys.argv[1:]:
    cfg = problems.CONFIGS[name]; pb = problems.generate(cfg); a = pb.csr()
    rng = np.random.default_rng(0); p = np.linalg.qr(rng.standard_normal((pb.n, cfg.k)))[0]
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    for rep in range(2):
        r = nlsp.pcg(a, pb.rhs, m, 0.0, 300)  # fixed 300 iterations
    print(name, "us/iter %.2f" % (r.report.solve_ms * 1e3 / r.report.iterations))
PY
for V in base skip; do if [ $V = base ]; then LIB=""; else LIB=paper_2601_20174_b200/variants/libnlsp_gpu_$V.so; fi; echo $V; NLSP_GPU_LIB=$LIB python /tmp/t.py C4 C2 C5; done
