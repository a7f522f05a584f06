#!/bin/bash
# Development helper under gpurun: bench line, ncu launch list, and full ncu
# captures of the one-pass cycle's kernels for one config. Output: gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${CFG:-C4}
timeout 600 python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench exit=$?"
if [ "${REF:-0}" = "1" ]; then
timeout 600 python bench.py --config $CFG --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$CFG.json 2> gpurun_out/bench_ref_$CFG.err; echo "ref exit=$?"
fi
# ncu cannot profile kernel nodes of graphs with conditional nodes: the
# profiled command runs the same kernels stream-ordered (NLSP_LOOP=host)
SHORT="env NLSP_LOOP=host python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --profile-iters 1"
timeout 300 $SHORT > gpurun_out/short_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$CFG.csv $SHORT > gpurun_out/ncu_list.log 2>&1; echo "ncu list exit=$?"
for K in ${KERNELS:-k_prolong_onepass_tma OpUpdSweep OpSpmvP}; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s ${SKIP:-20} -c 1 -o /tmp/prof_${CFG}_$K -f $SHORT > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu full $K exit=$?"
  # reports with source are large: bring back the raw and details pages only
  ncu -i /tmp/prof_${CFG}_$K.ncu-rep --page raw --csv > gpurun_out/prof_${CFG}_${K}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_${CFG}_$K.ncu-rep --page details --csv > gpurun_out/prof_${CFG}_${K}_details.csv 2>/dev/null
done
