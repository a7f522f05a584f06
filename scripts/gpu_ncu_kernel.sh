#!/bin/bash
# Development helper under gpurun: one ncu --set full capture of the kernels
# matching $K in the stream-ordered C4 (or $CFG) bench loop, after the same
# command has exited 0 without ncu. Output: gpurun_out/prof_$TAG.ncu-rep + csv.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${CFG:-C4}
TAG=${TAG:-$CFG}
SHORT="env NLSP_LOOP=host $EXTRA_ENV python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --profile-iters 2"
timeout 300 $SHORT > gpurun_out/short_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K:-k_march} -s ${SKIP:-6} -c ${COUNT:-3} \
  -o gpurun_out/prof_$TAG -f $SHORT > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit=$?"
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_$TAG.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv > gpurun_out/prof_$TAG.source.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details > gpurun_out/prof_$TAG.details.txt 2>/dev/null
ls -la gpurun_out/prof_$TAG*
