#!/bin/bash
# Development helper under gpurun: the one-pass prolongation's stage / stencil
# pair choices (NLSP_OP_S / NLSP_OP_P) per config; one short bench line each.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for C in ${CONFIGS:-C3 C4}; do
  for SP in ${VARIANTS:-0_0 4_4 4_2 4_1 6_3 6_2 8_4 8_2}; do
    set -- ${SP/_/ }
    NLSP_OP_S=$1 NLSP_OP_P=$2 timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_${C}_S$1_P$2.json 2>/dev/null
    python - "$C" "$1" "$2" <<'PY'
import json, sys
c, s, p = sys.argv[1:4]
try:
    d = json.load(open(f"gpurun_out/sweep_{c}_S{s}_P{p}.json"))
    k = d["kernels"]
    print(c, "S", s, "P", p, "iters/s", d["value"], "prolong_us", k["prolong_onepass"]["avg_us"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(c, s, p, "failed", e)
PY
  done
done
