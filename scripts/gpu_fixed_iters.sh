# Fixed-iteration A/B helper: VARIANTS is a ';'-separated list of env settings,
# CFGS the configs; prints us per iteration (best of 4 x 300 iterations) and
# digests of x for each.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/t.py <<'PY'
import sys, os, numpy as np
sys.path.insert(0, '.')
from paper_2601_20174_b200 import problems, nlsp
tag = sys.argv[1]
for name in sys.argv[2:]:
    base, _, nx = name.partition(":")  # "C1:2048" = C1 scaled to nx = 2048
    cfg = problems.CONFIGS[base].scaled(nx=int(nx)) if nx else problems.CONFIGS[base]
    pb = problems.generate(cfg); a = pb.csr()
    rng = np.random.default_rng(0); p = np.linalg.qr(rng.standard_normal((pb.n, cfg.k)))[0]
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    best = 1e30
    for rep in range(4):
        r = nlsp.pcg(a, pb.rhs, m, 0.0, 300)  # fixed 300 iterations
        best = min(best, r.report.solve_ms * 1e3 / r.report.iterations)
    x = np.asarray(r.solution)
    print(name, "[%s]" % tag, "us/iter %.2f" % best, "|x| %.15e" % np.linalg.norm(x), "last %.6e" % r.report.residual_history[-1], flush=True)
PY
IFS=';' read -ra VS <<< "${VARIANTS:-NLSP_NONE=1}"
for V in "${VS[@]}"; do env $V python /tmp/t.py "$V" ${CFGS:-C4}; done 2>&1 | tee gpurun_out/fixed_iters.log
