#!/bin/bash
# Development helper under gpurun: one bench line per (variant library, config).
# VARIANTS: tags of paper_2601_20174_b200/variants/libnlsp_gpu_<tag>.so ("base" = the main build)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for C in ${CONFIGS:-C4}; do
  for V in ${VARIANTS:-base}; do
    if [ "$V" = "base" ]; then LIB=""; else LIB=paper_2601_20174_b200/variants/libnlsp_gpu_$V.so; fi
    NLSP_GPU_LIB=$LIB timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_${C}_$V.json 2>/dev/null
    python - "$C" "$V" <<'PY'
import json, sys
c, v = sys.argv[1:3]
try:
    d = json.load(open(f"gpurun_out/var_{c}_{v}.json"))
    print(c, v, "iters/s", d["value"], "clk", d["clocks"]["sm_mhz"], {k: x["avg_us"] for k, x in d["kernels"].items()})
except Exception as e:
    print(c, v, "failed", e)
PY
  done
done
