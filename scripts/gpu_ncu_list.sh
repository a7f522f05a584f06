#!/bin/bash
# Development helper under gpurun: the ncu launch list (gpu__time_duration) of a
# short stream-ordered bench run, for each ';'-separated env setting in VARIANTS.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${CFG:-C4}
IFS=';' read -ra VS <<< "${VARIANTS:-NLSP_NONE=1}"
i=0
for V in "${VS[@]}"; do
  SHORT="env NLSP_LOOP=host $V python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --profile-iters 1"
  timeout 300 $SHORT > gpurun_out/short_plain_$i.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_${CFG}_$i.csv $SHORT > gpurun_out/ncu_list_$i.log 2>&1
  echo "$V -> launches_${CFG}_$i.csv exit=$?"
  i=$((i+1))
done
