#!/bin/bash
# compute-sanitizer over the product path (SURVEY §5 race detection): memcheck,
# racecheck and synccheck on the cluster solver (C1), the stream-ordered
# multi-kernel loop with the diagonal form and the TMA rings (C4, C3 with
# nu = 2/2) and the CSR row tiles (C5). Conditional graph nodes are not
# supported under the sanitizer, so the loop runs stream-ordered
# (NLSP_LOOP=host: the identical kernels). Logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
export NLSP_LOOP=host
for C in ${CASES:-C1 C4 C3 C5}; do
  for T in ${TOOLS:-memcheck racecheck synccheck}; do
    EXTRA=""
    [ "$T" = "racecheck" ] && EXTRA="--racecheck-report hazard"
    timeout ${TMO:-900} compute-sanitizer --tool $T $EXTRA --error-exitcode 7 \
      python scripts/sanitize_driver.py $C ${ITERS:-6} > gpurun_out/sanitizer_${C}_${T}.log 2>&1
    echo "$C $T exit=$? $(tail -1 gpurun_out/sanitizer_${C}_${T}.log)"
  done
done
