#!/bin/bash
# Development helper under gpurun: ncu --set full captures of the setup
# contractions at C4 (scripts/setup_probe.py): the DMMA kernels (symmetric Gram
# S^T S, k_gram_dmma for the k = 64 Grams, U_k = S V_k / sigma) and, with
# NLSP_DMMA=0, the register-tiled FFMA kernels they replace. Each profiled
# command first exits 0 without ncu.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python scripts/setup_probe.py ${CFG:-C4} 1"
$CMD > gpurun_out/setup_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_dmma|k_dense_mm_dmma|k_gram_reduce" -c 8 \
  -o gpurun_out/prof_setup_dmma -f $CMD > gpurun_out/ncu_setup_dmma.log 2>&1
echo "ncu dmma exit=$?"
NLSP_DMMA=0 $CMD > gpurun_out/setup_plain_ffma.log 2>&1 && \
NLSP_DMMA=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_partial|k_dense_mm" -c 6 \
  -o gpurun_out/prof_setup_ffma -f env NLSP_DMMA=0 $CMD > gpurun_out/ncu_setup_ffma.log 2>&1
echo "ncu ffma exit=$?"
for t in dmma ffma; do
  ncu -i gpurun_out/prof_setup_$t.ncu-rep --page raw --csv > gpurun_out/prof_setup_$t.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_setup_$t.ncu-rep --page details > gpurun_out/prof_setup_$t.details.txt 2>/dev/null
done
ls -la gpurun_out/prof_setup_*
