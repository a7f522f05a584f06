#!/bin/bash
# Development helper: libnlsp_gpu variants built with extra -D macros for
# solve_kernels.cu. usage: build_defs_variants.sh tag1:"-DA=1 -DB=2" tag2:"..."
set -e
D=$(cd "$(dirname "$0")/.." && pwd)/paper_2601_20174_b200
mkdir -p $D/variants $D/build/variants
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$D/../include -I$D/csrc"
make -s -C $D
for spec in "$@"; do
  tag=${spec%%:*}; defs=${spec#*:}
  $NV $defs -c $D/csrc/solve_kernels.cu -o $D/build/variants/solve_$tag.o &
done
wait
for spec in "$@"; do
  tag=${spec%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/variants/libnlsp_gpu_$tag.so $D/build/variants/solve_$tag.o $D/build/setup_kernels.o $D/build/setup_dmma.o $D/build/mlp.o $D/build/cluster_solve.o $D/build/nlsp_gpu.o -lcudart
done
ls $D/variants
