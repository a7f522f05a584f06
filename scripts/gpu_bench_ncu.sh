#!/bin/bash
# Development helper run under gpurun: bench (both arms), ncu launch list and one
# full ncu capture of the dominant kernel. Everything lands in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${CFG:-C4}
if [ "${BENCH:-1}" = "1" ]; then
timeout 600 python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench exit=$?"
timeout 600 python bench.py --config $CFG --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$CFG.json 2> gpurun_out/bench_ref_$CFG.err; echo "ref exit=$?"
fi
# ncu cannot profile kernel nodes of graphs with conditional nodes: the
# profiled command runs the same kernels stream-ordered (NLSP_LOOP=host)
SHORT="env NLSP_LOOP=host python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --profile-iters 1"
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 $SHORT > gpurun_out/short_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$CFG.csv $SHORT > gpurun_out/ncu_list.log 2>&1; echo "ncu list exit=$?"
  for K in ${KERNELS:-k_update_restrict k_prolong}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-20} -c 1 -o gpurun_out/prof_${CFG}_$K -f $SHORT > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu full $K exit=$?"
    # exports only (gpurun brings back at most 64 MiB)
    ncu -i gpurun_out/prof_${CFG}_$K.ncu-rep --page raw --csv > gpurun_out/prof_${CFG}_$K.raw.csv 2>/dev/null
    ncu -i gpurun_out/prof_${CFG}_$K.ncu-rep --page details > gpurun_out/prof_${CFG}_$K.details.txt 2>/dev/null
    [ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/prof_${CFG}_$K.ncu-rep
  done
fi
