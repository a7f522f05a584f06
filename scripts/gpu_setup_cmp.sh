#!/bin/bash
# Development helper under gpurun: setup timings (bench.py's "setup" object)
# with and without an env toggle, per config.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for C in ${CONFIGS:-C4 C3 C2}; do for B in 1 0; do
env ${TOGGLE:-NLSP_BSWEEP_DIA}=$B timeout 300 python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/setup_${C}_$B.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/setup_${C}_$B.json')); s=d['setup']; print('$C', '${TOGGLE:-NLSP_BSWEEP_DIA}=$B', {k: s[k] for k in ['smooth_ms','svd_basis_ms','twolevel_build_ms','total_ms']}, d['value'])"
done; done
