#!/bin/bash
# In place of compute-sanitizer (closed on this pool): the GPU test suite (or a
# subset, $TESTS) against the checked build, whose device-side NLSP_CHECKs
# bound every staged copy and shared-memory window and trap on a violation.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
LIB=paper_2601_20174_b200/variants/libnlsp_gpu_checked.so
[ -f $LIB ] || { echo "build it first: make -C paper_2601_20174_b200 checked"; exit 1; }
NLSP_GPU_LIB=$PWD/$LIB timeout ${TMO:-2400} python -m pytest ${TESTS:-tests -m gpu} -q -p no:cacheprovider \
  > gpurun_out/pytest_checked.log 2>&1
echo "checked pytest exit=$?"; tail -3 gpurun_out/pytest_checked.log
# the march kernels (off by default) under the checks too
NLSP_MARCH=1 NLSP_GPU_LIB=$PWD/$LIB timeout 900 python -m pytest tests/test_gpu_paths.py -q -k "execution or march" \
  > gpurun_out/pytest_checked_march.log 2>&1
echo "checked march pytest exit=$?"; tail -3 gpurun_out/pytest_checked_march.log
