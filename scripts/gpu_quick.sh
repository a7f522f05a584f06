#!/bin/bash
# Development helper run under gpurun: the path tests and one bench line per
# config (no CPU baseline). Everything lands in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
if [ "${TESTS:-paths}" = "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit=$?"
elif [ "${TESTS:-paths}" = "paths" ]; then
  timeout 900 python -m pytest tests/test_gpu_paths.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit=$?"
fi
for C in ${CONFIGS:-C4 C3 C2 C5}; do
  timeout 600 python bench.py --config $C --no-cpu-baseline $BENCH_ARGS > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; echo "bench $C exit=$?"
done
