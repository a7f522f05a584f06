#!/bin/bash
# Development helper under gpurun: C4 bench lines for one-pass prolongation
# ring shapes (NLSP_OP_BUDGET KB / NLSP_OP_S stages / NLSP_OP_P stencil pairs).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for spec in ${SPECS:-"200:0:0" "224:6:3" "224:6:2" "200:4:2" "224:6:6"}; do
  IFS=: read B S P <<< "$spec"
  env NLSP_OP_BUDGET=$B NLSP_OP_S=$S NLSP_OP_P=$P timeout 600 python bench.py --config ${CFG:-C4} --no-cpu-baseline --steps 5 \
    > gpurun_out/op_${S}_${P}_$B.json 2>/dev/null
  python - "$spec" <<'PY'
import json, sys
spec = sys.argv[1]
b, s, p = spec.split(":")
try:
    d = json.load(open(f"gpurun_out/op_{s}_{p}_{b}.json"))
except Exception:
    d = None
print(spec, d and (d["value"], d["clocks"]["sm_mhz"], {k: round(v["avg_us"], 1) for k, v in d["kernels"].items()}))
PY
done
