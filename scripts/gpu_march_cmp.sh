#!/bin/bash
# Development helper under gpurun: bench lines with the plane-march kernels on
# (NLSP_MARCH=1) and off (0) per config, one summary line each.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in ${CONFIGS:-C4 C3 C2}; do for m in ${MODES:-1 0}; do
  NLSP_MARCH=$m timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/bm_${c}_$m.json 2>gpurun_out/bm_${c}_$m.err
  python - "$c" "$m" <<'PY'
import json, sys
c, m = sys.argv[1:3]
try:
    d = json.load(open(f"gpurun_out/bm_{c}_{m}.json"))
    print(c, "march" if m == "1" else "direct", d["value"], "clk", d["clocks"]["sm_mhz"],
          {k: round(v["avg_us"], 1) for k, v in d["kernels"].items()},
          {k: d["setup"].get(k) for k in ("smooth_ms", "svd_basis_ms", "twolevel_build_ms", "api_generate_smoothed_vectors_ms", "api_setup_total_ms")})
except Exception as e:
    print(c, m, "failed", e)
PY
done; done
