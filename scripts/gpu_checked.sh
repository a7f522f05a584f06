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
# (the march kernels run under the checks too: the forced "march" path of
# test_execution_paths_match_reference and test_march_matches_direct_kernels
# pass NLSP_MARCH to their subprocesses, which inherit NLSP_GPU_LIB)
